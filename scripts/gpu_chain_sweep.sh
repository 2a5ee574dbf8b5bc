mkdir -p gpurun_out
for c in cfg2; do for k in 1 2 4 8 16 44; do for v in "" "--no-chain"; do n=$((148*640*k)); python bench.py --config $c --n $n --steps 200 --warmup 5 --no-cpu --no-e2e --no-fused $v 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$c', $k, $n, '$v', round(d['ms_per_step']*1e3,2))"; done; done; done > gpurun_out/chain_sweep.txt 2>&1
