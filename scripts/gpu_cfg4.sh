mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_fleet_gpu.py tests/test_chain_gpu.py -x -q > gpurun_out/cfg4_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/cfg4_pytest.log; tail -2 gpurun_out/cfg4_pytest.log
for v in "" "--ncw 20"; do timeout 300 python bench.py --config cfg4 --no-cpu --no-e2e --no-fused $v > gpurun_out/qb.json 2>gpurun_out/qb.err; python -c "import json;d=json.load(open('gpurun_out/qb.json'));print('cfg4 $v', round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],4), d['per_step_launches']['ms_per_step'])" || tail -3 gpurun_out/qb.err; done
