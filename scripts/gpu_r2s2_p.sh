O=gpurun_out/s2p; mkdir -p $O
timeout 1500 python -m pytest -q -x -m gpu tests/test_scene_gpu.py tests/test_world_gpu.py tests/test_vecenv_gpu.py -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
FS_WARM=110 timeout 300 python tools/gpu_forest_breakdown.py > $O/bd110.json 2>/dev/null
FS_WARM=10 timeout 300 python tools/gpu_forest_breakdown.py > $O/bd10.json 2>/dev/null
timeout 600 python bench.py --config forest --no-cpu > $O/bench_forest.json 2> $O/bench_forest.err
