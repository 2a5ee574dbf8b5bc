O=gpurun_out/s2u; mkdir -p $O
for L in libflocksim_b200 libfs_h1k libfs_h100k libfs_noh libflocksim_b200; do
  echo $L >> $O/tune.txt
  FS_LIB=paper_2305_16510_b200/lib/$L.so timeout 300 python tools/gpu_cfg3_tune.py >> $O/tune.txt 2>&1
done
