# reordered output-stage wait: correctness (chain / fleet / fullscale respawn tests) + timing
mkdir -p gpurun_out
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_chain_gpu.py tests/test_fleet_gpu.py tests/test_compat_gpu.py > gpurun_out/pytest_h.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_h.log
python tools/gpu_cfg3_persistent.py > gpurun_out/h_cfg3.txt 2>&1
for c in cfg2 cfg4; do timeout 300 python bench.py --config $c --steps 300 --no-cpu --no-fused --no-e2e --no-north-star > gpurun_out/h_$c.json 2>/dev/null; done
timeout 300 python bench.py --config cfg3 --n 2097152 --steps 300 --no-cpu --no-fused --no-e2e > gpurun_out/h_cfg3_bench.json 2>/dev/null
