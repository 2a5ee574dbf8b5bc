# forest reset kernel: dynamic list fetch, split pose lanes, slot->primitive table, lane-spread stores; MINB variants
mkdir -p gpurun_out/r2v
L=paper_2305_16510_b200/lib
timeout 1800 python -m pytest -q -p no:cacheprovider tests/test_scene_gpu.py tests/test_world_gpu.py tests/test_vecenv_gpu.py tests/test_compat_gpu.py > gpurun_out/r2v/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2v/pytest.log
python tools/gpu_forest_breakdown.py > gpurun_out/r2v/base.json 2>&1
cp $L/libflocksim_b200.so /tmp/base.so
for v in rs5 rs4; do
  cp $L/var/$v.so $L/libflocksim_b200.so
  timeout 600 python tools/gpu_forest_breakdown.py > gpurun_out/r2v/$v.json 2>&1
done
cp /tmp/base.so $L/libflocksim_b200.so
timeout 600 python bench.py --config forest --no-cpu --no-e2e > gpurun_out/r2v/bench_forest.json 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:world_reset_warp --launch-skip 200 --launch-count 1 -o gpurun_out/r2v/reset python tools/gpu_forest_breakdown.py > gpurun_out/r2v/ncu_reset.log 2>&1
