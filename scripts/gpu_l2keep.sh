mkdir -p gpurun_out
for c in cfg2 cfg3; do for mb in 0 32 64 96 112; do timeout 300 python bench.py --config $c --no-cpu --no-e2e --no-fused --l2-keep-mb $mb 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$c keep $mb', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3))"; done; done
