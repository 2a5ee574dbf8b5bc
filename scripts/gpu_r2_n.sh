mkdir -p gpurun_out; rm -f gpurun_out/n.txt
for lib in libflocksim_b200 libfs_ost3; do
  echo "$lib $(FS_LIB=paper_2305_16510_b200/lib/$lib.so python tools/gpu_cfg3_persistent.py 2>&1)" >> gpurun_out/n.txt
  FS_LIB=paper_2305_16510_b200/lib/$lib.so timeout 600 python tools/chain_stress.py 2 >> gpurun_out/n.txt 2>&1
done
