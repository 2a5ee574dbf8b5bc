mkdir -p gpurun_out
for c in forest render; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"
  timeout 900 python bench.py --config $c --impl reference > gpurun_out/bench_ref_$c.json 2> gpurun_out/bench_ref_$c.err; echo "$c ref rc=$?"
done
B="python bench.py --config render --steps 3 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/render_launches.csv $B > gpurun_out/ncu_r1.log 2>&1; echo "rl rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/render_full $B > gpurun_out/ncu_r2.log 2>&1; echo "rf rc=$?"
B="python bench.py --config forest --steps 10 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/forest_launches.csv $B > gpurun_out/ncu_f1.log 2>&1; echo "fl rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_step -s 6 -c 1 -o gpurun_out/forest_full $B > gpurun_out/ncu_f2.log 2>&1; echo "ff rc=$?"
