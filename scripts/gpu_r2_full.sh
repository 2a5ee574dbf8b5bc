# round-2 full pass: GPU suite, smoke, every bench config (ours + reference), launch lists
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2/gpu.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r2/smoke.txt
timeout 900 python bench.py > gpurun_out/r2/bench_default.json 2> gpurun_out/r2/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/r2/bench_ref.json 2> gpurun_out/r2/bench_ref.err
for c in cfg0 cfg1 cfg3 cfg4 world vecenv forest render; do
  timeout 900 python bench.py --config $c > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err
done
for c in forest render cfg3; do
  timeout 600 python bench.py --impl reference --config $c > gpurun_out/r2/bench_ref_$c.json 2> gpurun_out/r2/bench_ref_$c.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2/launches_cfg2.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-fused --north-star-steps 20 > gpurun_out/r2/ncu_launch.log 2>&1
