mkdir -p gpurun_out/s2j
FS_WARM=10 timeout 300 python tools/gpu_forest_breakdown.py > gpurun_out/s2j/fresh.json 2>&1
FS_WARM=110 timeout 300 python tools/gpu_forest_breakdown.py > gpurun_out/s2j/mid.json 2>&1
