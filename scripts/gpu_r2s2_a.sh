# session 2 re-entry: GPU suite + smoke + the headline and north-star bench lines on HEAD
mkdir -p gpurun_out/s2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/s2a/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/s2a/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/s2a/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2a/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/s2a/smoke.txt
timeout 900 python bench.py > gpurun_out/s2a/bench_default.json 2> gpurun_out/s2a/bench_default.err
timeout 600 python tools/gpu_cfg3_persistent.py > gpurun_out/s2a/cfg3_breakdown.txt 2>&1
timeout 900 python bench.py --config forest > gpurun_out/s2a/bench_forest.json 2> gpurun_out/s2a/bench_forest.err
