mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 5 -c 1 -o gpurun_out/var_plain python tools/gpu_fleet_variant.py position 0 0 > gpurun_out/var1.log 2>&1; echo "a rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 5 -c 1 -o gpurun_out/var_cfg3 python tools/gpu_fleet_variant.py position 0.01 1 > gpurun_out/var2.log 2>&1; echo "b rc=$?"
