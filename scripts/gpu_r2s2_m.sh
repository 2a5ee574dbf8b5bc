mkdir -p gpurun_out/s2m
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:stream_kernel --csv python tools/gpu_cfg4_traffic.py > gpurun_out/s2m/ncu.csv 2> gpurun_out/s2m/ncu.err
