# forest: scene tests, steady-state breakdown, bench, full ncu of the fix + reset kernels at step ~200
mkdir -p gpurun_out/r2t
timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py tests/test_world_gpu.py > gpurun_out/r2t/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2t/pytest.log
python tools/gpu_forest_breakdown.py > gpurun_out/r2t/breakdown.json 2>&1
timeout 600 python bench.py --config forest --no-cpu --no-e2e > gpurun_out/r2t/bench_forest.json 2>/dev/null
for k in scene_fix_kernel world_reset_warp_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 200 --launch-count 1 -o gpurun_out/r2t/$k python tools/gpu_forest_breakdown.py > gpurun_out/r2t/ncu_$k.log 2>&1
done
