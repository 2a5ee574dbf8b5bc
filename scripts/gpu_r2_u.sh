# forest fix / reset kernel launch-bounds variants (developer libs under lib/var), steady-state breakdown each
mkdir -p gpurun_out/r2u
L=paper_2305_16510_b200/lib
cp $L/libflocksim_b200.so /tmp/base.so
python tools/gpu_forest_breakdown.py > gpurun_out/r2u/base.json 2>&1
for v in fix8 flat6 rs5 rs6 combo; do
  cp $L/var/$v.so $L/libflocksim_b200.so
  timeout 600 python tools/gpu_forest_breakdown.py > gpurun_out/r2u/$v.json 2>&1
done
cp /tmp/base.so $L/libflocksim_b200.so
python tools/gpu_forest_breakdown.py > gpurun_out/r2u/base2.json 2>&1
