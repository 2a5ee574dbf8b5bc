# ncu evidence for the persistent (fs_step_many) bench path: launch list of
# the default bench command and one --set full capture per config of the
# K=20-step persistent launch (the 4th stream_kernel launch, after 3 warm-ups),
# exported on the box (details / raw / source pages) to stay under the
# 64 MiB pull limit; only cfg2's report is kept.
mkdir -p gpurun_out
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 300 $B > gpurun_out/plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1
for c in cfg2 cfg3 cfg1 cfg4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/pers_$c $B --config $c > gpurun_out/ncu_$c.log 2>&1
  echo "$c rc=$?"
  ncu -i gpurun_out/pers_$c.ncu-rep --page details > gpurun_out/pers_${c}_details.txt 2>&1
  ncu -i gpurun_out/pers_$c.ncu-rep --page raw --csv > gpurun_out/pers_${c}_raw.csv 2>&1
  ncu -i gpurun_out/pers_$c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pers_${c}_source.csv 2>&1
  [ "$c" = cfg2 ] || rm -f gpurun_out/pers_$c.ncu-rep
done
du -sh gpurun_out
