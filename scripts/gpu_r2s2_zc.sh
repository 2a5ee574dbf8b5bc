O=gpurun_out/s2zc; mkdir -p $O
for L in libflocksim_b200 libfs_nopdl libflocksim_b200 libfs_nopdl; do
  echo $L >> $O/bd.txt
  FS_LIB=paper_2305_16510_b200/lib/$L.so FS_WARM=110 timeout 300 python tools/gpu_forest_breakdown.py 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(json.dumps({k[:28]:(v['us_avg'] if isinstance(v,dict) else v) for k,v in d.items()}))" >> $O/bd.txt
done
timeout 1200 python -m pytest -q -x -m gpu tests/test_scene_gpu.py tests/test_vecenv_gpu.py tests/test_world_gpu.py -p no:cacheprovider > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
timeout 600 python bench.py --config forest --no-cpu > $O/bench_forest.json 2>/dev/null
