mkdir -p gpurun_out/s2g
timeout 300 python tools/gpu_cfg3_plan.py 0 32 200 > gpurun_out/s2g/plan.txt 2>&1
timeout 300 python tools/gpu_cfg3_tune.py >> gpurun_out/s2g/plan.txt 2>&1
FS_K=40 FS_REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv python tools/gpu_cfg3_plan.py 0 8 > gpurun_out/s2g/ncu.csv 2> gpurun_out/s2g/ncu.err
