O=gpurun_out/s2z1; mkdir -p $O
for t in "" "NCW=16" "NCW=12" ""; do
  timeout 300 python tools/gpu_cfg3_tune.py $t >> $O/tune.txt 2>&1
done
