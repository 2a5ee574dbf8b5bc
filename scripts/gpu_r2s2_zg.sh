O=gpurun_out/s2zg; mkdir -p $O
timeout 1200 python -m pytest -q -x -m gpu tests/test_scene_gpu.py tests/test_world_gpu.py tests/test_vecenv_gpu.py -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python bench.py --config forest --no-cpu > $O/bench_forest.json 2> $O/bench_forest.err
FS_WARM=110 timeout 300 python tools/gpu_forest_breakdown.py > $O/bd.json 2>/dev/null
