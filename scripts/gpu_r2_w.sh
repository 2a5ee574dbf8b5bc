# forest: half-warp deferred collision test; scene tests + steady-state breakdown + bench
mkdir -p gpurun_out/r2w
timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py tests/test_world_gpu.py > gpurun_out/r2w/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2w/pytest.log
python tools/gpu_forest_breakdown.py > gpurun_out/r2w/base.json 2>&1
timeout 600 python bench.py --config forest --no-cpu --no-e2e > gpurun_out/r2w/bench_forest.json 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:world_stream --launch-skip 200 --launch-count 1 -o gpurun_out/r2w/stream python tools/gpu_forest_breakdown.py > gpurun_out/r2w/ncu_stream.log 2>&1
