mkdir -p gpurun_out
B="python bench.py --config render --steps 3 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/render_p $B > gpurun_out/ncu_render.log 2>&1; echo "rc=$?"
ncu -i gpurun_out/render_p.ncu-rep --page details > gpurun_out/render_details.txt 2>&1
ncu -i gpurun_out/render_p.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/render_source.csv 2>&1
rm -f gpurun_out/render_p.ncu-rep
