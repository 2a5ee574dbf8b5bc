mkdir -p gpurun_out
B="python bench.py --config world --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 300 $B > gpurun_out/plain_world.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:world_stream -s 5 -c 1 -o gpurun_out/world_prof $B > gpurun_out/ncu_world.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/world_prof.ncu-rep --page details > gpurun_out/world_details.txt 2>&1
ncu -i gpurun_out/world_prof.ncu-rep --page raw --csv > gpurun_out/world_raw.csv 2>&1
ncu -i gpurun_out/world_prof.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/world_source.csv 2>&1
rm -f gpurun_out/world_prof.ncu-rep
