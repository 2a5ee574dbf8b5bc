mkdir -p gpurun_out
for c in forest render; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
  timeout 900 python bench.py --config $c --impl reference > gpurun_out/bench_ref_$c.json 2> gpurun_out/bench_ref_$c.err; echo "$c ref rc=$?"
done
timeout 600 python bench.py --no-cpu --no-e2e --steps 50 > gpurun_out/bench_cfg2_quick.json 2>&1; echo "cfg2 rc=$?"
