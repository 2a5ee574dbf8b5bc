mkdir -p gpurun_out/s2b
for t in "" "CHAIN_RELEASE=1" "CONS_WAIT_NS=32" "NCW=16"; do
  timeout 300 python tools/gpu_cfg3_tune.py $t >> gpurun_out/s2b/tune.txt 2>&1
done
