# forest fix kernel: box + primitive loads in flight together, launch-bounds variants (lib/var)
mkdir -p gpurun_out/r2aa
L=paper_2305_16510_b200/lib
cp $L/libflocksim_b200.so /tmp/base.so
python tools/gpu_forest_breakdown.py > gpurun_out/r2aa/base.json 2>&1
for v in f8 f6 f5; do
  cp $L/var/$v.so $L/libflocksim_b200.so
  timeout 600 python tools/gpu_forest_breakdown.py > gpurun_out/r2aa/$v.json 2>&1
done
cp /tmp/base.so $L/libflocksim_b200.so
