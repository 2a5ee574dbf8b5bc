mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_scene_gpu.py tests/test_world_gpu.py -x -q > gpurun_out/forest_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/forest_pytest.log; tail -2 gpurun_out/forest_pytest.log
timeout 300 python bench.py --config forest --no-cpu --no-e2e --no-fused 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('forest', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3))"
