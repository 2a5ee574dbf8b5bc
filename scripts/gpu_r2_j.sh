mkdir -p gpurun_out; rm -f gpurun_out/j_cfg3.txt
timeout 600 python tools/chain_stress.py 3 > gpurun_out/stress_j.txt 2>&1
timeout 1500 python -m pytest -q -p no:cacheprovider tests/test_chain_gpu.py tests/test_fleet_gpu.py tests/test_scene_gpu.py tests/test_world_gpu.py > gpurun_out/pytest_j.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_j.log
for sw in 0 64 256; do echo "spawn=$sw $(python tools/gpu_cfg3_persistent.py 2 $sw 0 2>&1)" >> gpurun_out/j_cfg3.txt; done
timeout 600 python bench.py --config forest --steps 100 --no-cpu --no-e2e > gpurun_out/j_forest.json 2> gpurun_out/j_forest.err
