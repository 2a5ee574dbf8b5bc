mkdir -p gpurun_out
for c in world vecenv forest; do timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?; done
B="python bench.py --config forest --steps 10 --warmup 3 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/forest_launches.csv $B > gpurun_out/ncu1.log 2>&1; echo "l rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_ -s 6 -c 2 -o gpurun_out/forest_prof $B > gpurun_out/ncu2.log 2>&1; echo "f rc=$?"
