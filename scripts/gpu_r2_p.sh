mkdir -p gpurun_out/r2p
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2p/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2p/pytest_gpu.txt
timeout 900 python bench.py --config forest > gpurun_out/r2p/bench_forest.json 2> gpurun_out/r2p/bench_forest.err
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:"world_|scene_fix" --launch-skip 30 --launch-count 30 --csv python bench.py --config forest --steps 20 --warmup 10 --no-cpu --no-e2e > gpurun_out/r2p/forest_launches.csv 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"world_stream|scene_fix|world_reset" --launch-skip 30 --launch-count 3 -o gpurun_out/r2p/forest_full python bench.py --config forest --steps 20 --warmup 10 --no-cpu --no-e2e > gpurun_out/r2p/ncu_forest.log 2>&1
