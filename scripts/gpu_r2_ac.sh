# World.step streaming kernel: consumer-warp count variants (FS_WORLD_NCW, lib/var): forest breakdown + bench, free-space world bench
mkdir -p gpurun_out/r2ac
L=paper_2305_16510_b200/lib
cp $L/libflocksim_b200.so /tmp/base.so
for v in base n10 n12; do
  [ $v != base ] && cp $L/var/$v.so $L/libflocksim_b200.so
  timeout 600 python tools/gpu_forest_breakdown.py > gpurun_out/r2ac/$v.json 2>&1
  timeout 600 python bench.py --config forest --no-cpu --no-e2e > gpurun_out/r2ac/forest_$v.json 2>/dev/null
  timeout 600 python bench.py --config world --no-cpu --no-e2e > gpurun_out/r2ac/world_$v.json 2>/dev/null
  cp /tmp/base.so $L/libflocksim_b200.so
done
