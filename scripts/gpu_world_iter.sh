mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_world_gpu.py tests/test_vecenv_gpu.py -x -q > gpurun_out/world_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/world_pytest.log; tail -2 gpurun_out/world_pytest.log
for c in world vecenv; do timeout 300 python bench.py --config $c --no-cpu --no-e2e --no-fused > gpurun_out/qb_$c.json 2> gpurun_out/qb_$c.err; python -c "import json;d=json.load(open('gpurun_out/qb_$c.json'));print('$c', round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],4))" || tail -3 gpurun_out/qb_$c.err; done
