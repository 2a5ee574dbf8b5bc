O=gpurun_out/s2w; mkdir -p $O
timeout 900 python -m pytest -q -x -m gpu tests/test_chain_gpu.py tests/test_fleet_gpu.py tests/test_fullscale_gpu.py -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for L in libflocksim_b200 libfs_ip0 libflocksim_b200 libfs_ip0; do
  echo $L >> $O/tune.txt
  FS_LIB=paper_2305_16510_b200/lib/$L.so timeout 300 python tools/gpu_cfg3_tune.py >> $O/tune.txt 2>&1
done
