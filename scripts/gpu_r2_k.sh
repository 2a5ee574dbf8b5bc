mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py tests/test_world_gpu.py tests/test_vecenv_gpu.py > gpurun_out/pytest_k.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_k.log
timeout 600 python bench.py --config forest --steps 100 --no-cpu --no-e2e > gpurun_out/k_forest.json 2> gpurun_out/k_forest.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv python bench.py --config forest --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/k_forest_ncu.csv 2>/dev/null
