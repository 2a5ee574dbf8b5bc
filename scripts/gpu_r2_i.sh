mkdir -p gpurun_out
timeout 900 python tools/chain_stress.py 6 > gpurun_out/stress.txt 2>&1
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_chain_gpu.py tests/test_fleet_gpu.py tests/test_fullscale_gpu.py > gpurun_out/pytest_i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_i.log
for sw in 0 32 64 128; do for cw in 0 32; do echo "spawn=$sw cons=$cw $(python tools/gpu_cfg3_persistent.py 2 $sw $cw 2>&1)" >> gpurun_out/i_cfg3.txt; done; done
