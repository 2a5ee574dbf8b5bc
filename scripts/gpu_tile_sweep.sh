mkdir -p gpurun_out
for c in cfg3 cfg2; do for k in 8 16 22 23 32; do n=$((148*640*k)); python bench.py --config $c --n $n --steps 200 --warmup 5 --no-cpu --no-e2e --no-fused 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$c', $k, $n, round(d['ms_per_step']*1e3,2))"; done; done > gpurun_out/sweep.txt 2>&1
