mkdir -p gpurun_out/s2e
timeout 900 python -m pytest -q -x -m gpu tests/test_chain_gpu.py -p no:cacheprovider > gpurun_out/s2e/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s2e/pytest.txt
timeout 300 python tools/gpu_cfg3_tune.py > gpurun_out/s2e/tune.txt 2>&1
