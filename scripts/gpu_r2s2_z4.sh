O=gpurun_out/s2z4; mkdir -p $O
timeout 300 python tools/gpu_cfg3_tune.py > $O/tune.txt 2>&1
for i in 1 2; do timeout 600 python bench.py --no-cpu --no-e2e --no-north-star > $O/bench_$i.json 2>/dev/null; done
timeout 900 python -m pytest -q -x -m gpu tests/test_chain_gpu.py tests/test_fleet_gpu.py -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
