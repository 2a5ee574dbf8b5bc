mkdir -p gpurun_out; rm -f gpurun_out/e.txt
for lib in libflocksim_b200 libfs_diag_nospawn libfs_diag_nocfence libfs_diag_both; do
  echo $lib >> gpurun_out/e.txt
  FS_LIB=paper_2305_16510_b200/lib/$lib.so python tools/gpu_cfg3_persistent.py 2 >> gpurun_out/e.txt 2>&1
done
