# forest: full-width listed resets (reset_pose/slot/place kernels); scene + world tests, breakdown, bench, ncu launch list of one steady step
mkdir -p gpurun_out/r2x
timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py tests/test_world_gpu.py tests/test_vecenv_gpu.py tests/test_compat_gpu.py > gpurun_out/r2x/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2x/pytest.log
python tools/gpu_forest_breakdown.py > gpurun_out/r2x/base.json 2>&1
timeout 600 python bench.py --config forest --no-cpu --no-e2e > gpurun_out/r2x/bench_forest.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --launch-skip 1300 --launch-count 14 --csv python tools/gpu_forest_breakdown.py > gpurun_out/r2x/launches_steady.csv 2>/dev/null
