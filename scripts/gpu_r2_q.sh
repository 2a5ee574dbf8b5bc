mkdir -p gpurun_out; rm -f gpurun_out/q.txt
timeout 600 python tools/chain_stress.py 3 > gpurun_out/q_stress.txt 2>&1
timeout 1500 python -m pytest -q -x -p no:cacheprovider tests/test_chain_gpu.py tests/test_fleet_gpu.py tests/test_fullscale_gpu.py > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_q.log
python tools/gpu_cfg3_persistent.py >> gpurun_out/q.txt 2>&1
python tools/gpu_cfg3_persistent.py >> gpurun_out/q.txt 2>&1
