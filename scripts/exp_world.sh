mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_world_gpu.py tests/test_vecenv_gpu.py -x -q > gpurun_out/world_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/world_pytest.log; tail -2 gpurun_out/world_pytest.log
cp paper_2305_16510_b200/lib/libflocksim_b200.so /tmp/lib16.so
for v in 16 14 12; do
  if [ $v != 16 ]; then cp paper_2305_16510_b200/lib/libexp_w$v.so paper_2305_16510_b200/lib/libflocksim_b200.so; fi
  for c in world vecenv; do python bench.py --config $c --no-cpu --no-e2e --no-fused 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('ncw $v $c', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3))"; done
done
cp /tmp/lib16.so paper_2305_16510_b200/lib/libflocksim_b200.so
