mkdir -p gpurun_out
for c in cfg2 cfg3 cfg1 cfg4; do timeout 600 python bench.py --config $c --no-cpu --no-e2e --no-fused > gpurun_out/qb_$c.json 2> gpurun_out/qb_$c.err; echo $c rc=$?; done
