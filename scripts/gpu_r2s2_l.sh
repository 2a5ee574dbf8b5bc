mkdir -p gpurun_out/s2l
timeout 1200 python -m pytest -q -x -m gpu tests/test_scene_gpu.py tests/test_world_gpu.py -p no:cacheprovider > gpurun_out/s2l/pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/s2l/pytest.txt
timeout 600 python bench.py --config forest > gpurun_out/s2l/bench_forest.json 2> gpurun_out/s2l/bench_forest.err
