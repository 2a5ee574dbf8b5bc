O=gpurun_out/s2zl; mkdir -p $O
for L in libflocksim_b200 libfs_pm5 libfs_pm4 libflocksim_b200 libfs_pm5; do
  echo $L >> $O/bd.txt
  FS_LIB=paper_2305_16510_b200/lib/$L.so FS_WARM=110 timeout 300 python tools/gpu_forest_breakdown.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(json.dumps({k[:28]:(v['us_avg'] if isinstance(v,dict) else v) for k,v in d.items() if 'walk' not in k}))" >> $O/bd.txt
done
