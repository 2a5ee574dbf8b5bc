O=gpurun_out/s2z9; mkdir -p $O
for t in "" "CONS_WAIT_NS=64" "CONS_WAIT_NS=256" "CONS_WAIT_NS=1000" "SPAWN_WAIT_NS=128" ""; do
  timeout 300 python tools/gpu_cfg3_tune.py $t >> $O/tune.txt 2>&1
done
