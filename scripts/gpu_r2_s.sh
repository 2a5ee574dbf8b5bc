mkdir -p gpurun_out
timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py tests/test_world_gpu.py tests/test_vecenv_gpu.py > gpurun_out/pytest_s.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_s.log
python tools/gpu_forest_breakdown.py > gpurun_out/s_forest.json 2>&1
timeout 600 python bench.py --config forest --no-cpu --no-e2e > gpurun_out/s_forest_bench.json 2>/dev/null
