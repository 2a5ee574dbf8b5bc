mkdir -p gpurun_out/s2h
for i in 1 2; do
timeout 300 python tools/gpu_cfg3_plan.py 0 200 >> gpurun_out/s2h/plan.txt 2>&1
FS_LIB=paper_2305_16510_b200/lib/libfs_old.so timeout 300 python tools/gpu_cfg3_plan.py 0 200 >> gpurun_out/s2h/plan.txt 2>&1
done
