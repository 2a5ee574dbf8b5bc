# ncu evidence for the World.step / VecEnvHandle.step streaming kernel
# (one --set full capture each, exported on the box)
mkdir -p gpurun_out
for c in world vecenv; do
  B="python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused"
  timeout 300 $B > gpurun_out/plain_$c.log 2>&1 || exit 1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_stream -s 5 -c 1 -o gpurun_out/${c}_prof $B > gpurun_out/ncu_$c.log 2>&1; echo "$c rc=$?"
  ncu -i gpurun_out/${c}_prof.ncu-rep --page details > gpurun_out/${c}_details.txt 2>&1
  ncu -i gpurun_out/${c}_prof.ncu-rep --page raw --csv > gpurun_out/${c}_raw.csv 2>&1
  ncu -i gpurun_out/${c}_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${c}_source.csv 2>&1
  rm -f gpurun_out/${c}_prof.ncu-rep
done
