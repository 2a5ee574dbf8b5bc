# Full round bench: every config (+ CPU baseline), the reference arms, the
# default launch list and one ncu --set full capture of the hot kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" > gpurun_out/lscpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
for c in cfg0 cfg1 cfg3 cfg4 world vecenv forest render; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for c in forest render; do
  timeout 900 python bench.py --config $c --impl reference > gpurun_out/bench_ref_$c.json 2> gpurun_out/bench_ref_$c.err; echo "ref $c rc=$?"
done
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/prof_default $B > gpurun_out/ncu2.log 2>&1
echo "ncu rc=$?"
B="python bench.py --config cfg3 --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/prof_cfg3 $B > gpurun_out/ncu3.log 2>&1
echo "ncu3 rc=$?"
