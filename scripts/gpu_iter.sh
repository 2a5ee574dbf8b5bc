# Iteration check after a hot-kernel change: stream-kernel parity tests, then
# quick bench lines (no CPU / e2e legs) for the configs given (default cfg2 cfg3).
mkdir -p gpurun_out
CFGS=${CFGS:-"cfg2 cfg3"}
timeout 600 python -m pytest tests/test_fleet_gpu.py tests/test_parity_gpu.py tests/test_chain_gpu.py -x -q -m gpu > gpurun_out/iter_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/iter_pytest.log
tail -n 2 gpurun_out/iter_pytest.log
for c in $CFGS; do timeout 600 python bench.py --config $c --no-cpu --no-e2e --no-fused $BENCH_ARGS > gpurun_out/qb_$c.json 2> gpurun_out/qb_$c.err; python -c "import json;d=json.load(open('gpurun_out/qb_$c.json'));print('$c', round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],4), 'per-step', round(d.get('per_step_launches',{}).get('ms_per_step',0)*1e3,2))" || tail -3 gpurun_out/qb_$c.err; done
