# forest: warp-per-env resets (fetch only by warps below the count); with / without instance-pose planes
mkdir -p gpurun_out/r2y
timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py tests/test_world_gpu.py > gpurun_out/r2y/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2y/pytest.log
python tools/gpu_forest_breakdown.py > gpurun_out/r2y/base.json 2>&1
FS_BREAKDOWN_NO_INST_POSE=1 python tools/gpu_forest_breakdown.py > gpurun_out/r2y/nopose.json 2>&1
timeout 600 python bench.py --config forest --no-cpu --no-e2e > gpurun_out/r2y/bench_forest.json 2>/dev/null
