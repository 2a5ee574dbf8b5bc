O=gpurun_out/s2s; mkdir -p $O
timeout 1500 python -m pytest -q -x -m gpu tests/test_world_gpu.py tests/test_vecenv_gpu.py tests/test_scene_gpu.py -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python tools/gpu_world_resets.py > $O/resets.json 2>&1
