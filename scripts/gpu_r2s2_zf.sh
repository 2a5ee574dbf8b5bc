O=gpurun_out/s2zf; mkdir -p $O
L=paper_2305_16510_b200/lib
cp $L/libflocksim_b200.so /tmp/orig.so
for V in orig w12 w10 orig w12; do
  if [ $V = orig ]; then cp /tmp/orig.so $L/libflocksim_b200.so; else cp $L/libfs_$V.so $L/libflocksim_b200.so; fi
  for c in world vecenv; do
    timeout 600 python bench.py --config $c --no-cpu > $O/${c}_$V.json 2>/dev/null
    python -c "import json; d=json.loads([l for l in open('$O/${c}_$V.json') if l.startswith('{')][-1]); print('$c $V', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3))" >> $O/summary.txt
  done
done
cp /tmp/orig.so $L/libflocksim_b200.so
