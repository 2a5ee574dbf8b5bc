# forest: instance poses on demand (fs_obstacles_poses), resets skip the pose planes
mkdir -p gpurun_out/r2z
timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py tests/test_world_gpu.py tests/test_vecenv_gpu.py tests/test_compat_gpu.py > gpurun_out/r2z/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2z/pytest.log
python tools/gpu_forest_breakdown.py > gpurun_out/r2z/base.json 2>&1
timeout 600 python bench.py --config forest --no-cpu --no-e2e > gpurun_out/r2z/bench_forest.json 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:world_reset_warp --launch-skip 200 --launch-count 1 -o gpurun_out/r2z/reset python tools/gpu_forest_breakdown.py > gpurun_out/r2z/ncu_reset.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scene_fix --launch-skip 200 --launch-count 1 -o gpurun_out/r2z/fix python tools/gpu_forest_breakdown.py > gpurun_out/r2z/ncu_fix.log 2>&1
