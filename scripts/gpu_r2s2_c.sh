mkdir -p gpurun_out/s2c
timeout 300 python tools/gpu_cfg3_tune.py > gpurun_out/s2c/tune.txt 2>&1
FS_LIB=paper_2305_16510_b200/lib/libfs_ahead0.so timeout 300 python tools/gpu_cfg3_tune.py >> gpurun_out/s2c/tune.txt 2>&1
timeout 300 python tools/gpu_cfg3_tune.py >> gpurun_out/s2c/tune.txt 2>&1
timeout 900 python -m pytest -q -x -m gpu tests/test_chain_gpu.py tests/test_fleet_gpu.py tests/test_fullscale_gpu.py -p no:cacheprovider > gpurun_out/s2c/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s2c/pytest.txt
