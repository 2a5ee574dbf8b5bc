# Run-to-run spread of the headline lines: five cfg2 and three cfg3 runs
mkdir -p gpurun_out
for r in 1 2 3 4 5; do python bench.py --no-cpu --no-e2e --no-fused 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('cfg2', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
for r in 1 2 3; do python bench.py --config cfg3 --no-cpu --no-e2e --no-fused 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('cfg3', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
