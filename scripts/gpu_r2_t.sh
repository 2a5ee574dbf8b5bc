mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"world_reset|scene_fix" --launch-skip 400 --launch-count 2 -o gpurun_out/t_forest_reset python tools/gpu_forest_breakdown.py > gpurun_out/t_ncu.log 2>&1
