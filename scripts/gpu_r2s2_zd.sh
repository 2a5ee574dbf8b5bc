O=gpurun_out/s2zd; mkdir -p $O
timeout 1200 python -m pytest -q -x -m gpu tests/test_chain_gpu.py tests/test_fleet_gpu.py tests/test_fullscale_gpu.py tests/test_bench_gpu.py -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for i in 1 2; do timeout 300 python tools/gpu_cfg3_tune.py >> $O/tune.txt 2>&1; done
