# one --set full capture of the persistent launch for the configs in $CFGS
mkdir -p gpurun_out
for c in ${CFGS:-cfg3}; do
  B="python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 3 -c 1 -o gpurun_out/pers_$c $B > gpurun_out/ncu_$c.log 2>&1; echo "$c rc=$?"
  ncu -i gpurun_out/pers_$c.ncu-rep --page details > gpurun_out/pers_${c}_details.txt 2>&1
  ncu -i gpurun_out/pers_$c.ncu-rep --page raw --csv > gpurun_out/pers_${c}_raw.csv 2>&1
  ncu -i gpurun_out/pers_$c.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/pers_${c}_source.csv 2>&1
  rm -f gpurun_out/pers_$c.ncu-rep
done
