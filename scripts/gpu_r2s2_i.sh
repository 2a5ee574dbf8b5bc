mkdir -p gpurun_out/s2i
for L in libflocksim_b200 libfs_dec libfs_dec2 libfs_nocf; do
  echo $L >> gpurun_out/s2i/tune.txt
  FS_LIB=paper_2305_16510_b200/lib/$L.so timeout 300 python tools/gpu_cfg3_tune.py >> gpurun_out/s2i/tune.txt 2>&1
done
