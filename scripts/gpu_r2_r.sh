mkdir -p gpurun_out; rm -f gpurun_out/r.txt
timeout 600 python tools/chain_stress.py 2 > gpurun_out/r_stress.txt 2>&1
timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_chain_gpu.py tests/test_fleet_gpu.py tests/test_scene_gpu.py tests/test_world_gpu.py > gpurun_out/pytest_r.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r.log
python tools/gpu_cfg3_persistent.py >> gpurun_out/r.txt 2>&1
python tools/gpu_forest_breakdown.py > gpurun_out/r_forest.json 2>&1
