O=gpurun_out/s2z2; mkdir -p $O
for L in libflocksim_b200 libfs_sw3 libfs_sw1 libflocksim_b200 libfs_sw3; do
  echo $L >> $O/tune.txt
  FS_LIB=paper_2305_16510_b200/lib/$L.so timeout 300 python tools/gpu_cfg3_tune.py >> $O/tune.txt 2>&1
done
