# round-2 final pass: GPU suite, smoke, every bench config (ours + reference), launch list, ncu
mkdir -p gpurun_out/r2f
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2f/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2f/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2f/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2f/smoke.txt
timeout 900 python bench.py > gpurun_out/r2f/bench_default.json 2> gpurun_out/r2f/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/r2f/bench_ref.json 2> gpurun_out/r2f/bench_ref.err
for c in cfg0 cfg1 cfg3 cfg4 world vecenv forest render; do
  timeout 900 python bench.py --config $c > gpurun_out/r2f/bench_$c.json 2> gpurun_out/r2f/bench_$c.err
done
for c in forest render cfg3; do
  timeout 600 python bench.py --impl reference --config $c > gpurun_out/r2f/bench_ref_$c.json 2> gpurun_out/r2f/bench_ref_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f/launches_cfg2.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-fused --north-star-steps 20 > gpurun_out/r2f/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 3 --launch-count 1 -o gpurun_out/r2f/cfg2_full python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-fused --no-north-star > gpurun_out/r2f/ncu_cfg2.log 2>&1
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for c in world vecenv; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:world_stream --launch-skip 3 --launch-count 1 --csv python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2f/traffic_${c}.csv 2>/dev/null
done
timeout 600 ncu --metrics $M --clock-control none -k regex:"world_|scene_fix" --launch-skip 9 --launch-count 3 --csv python bench.py --config forest --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/r2f/traffic_forest.csv 2>/dev/null
