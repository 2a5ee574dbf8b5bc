O=gpurun_out/s2x; mkdir -p $O
L=paper_2305_16510_b200/lib
for V in libflocksim_b200 libfs_ipall libflocksim_b200 libfs_ipall; do
  echo $V >> $O/tune.txt
  FS_LIB=$L/$V.so timeout 300 python tools/gpu_cfg3_tune.py >> $O/tune.txt 2>&1
done
cp $L/libflocksim_b200.so /tmp/orig.so
for V in orig ipall orig ipall; do
  if [ $V = ipall ]; then cp $L/libfs_ipall.so $L/libflocksim_b200.so; else cp /tmp/orig.so $L/libflocksim_b200.so; fi
  timeout 600 python bench.py --no-cpu --no-e2e --no-north-star > $O/bench_$V.json 2>/dev/null
  python -c "import json; d=json.loads([l for l in open('$O/bench_$V.json') if l.startswith('{')][-1]); print('$V', d['ms_per_step']*1e3, d['roofline']['frac'])" >> $O/bench.txt
done
cp /tmp/orig.so $L/libflocksim_b200.so
