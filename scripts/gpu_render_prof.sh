mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:render_kernel -s 3 -c 1 -o gpurun_out/render_prof python tools/gpu_render.py --iters 1 > gpurun_out/render_ncu.log 2>&1; echo "ncu rc=$?"
