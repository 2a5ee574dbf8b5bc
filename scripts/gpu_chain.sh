# Chained steps: parity tests, then quick bench lines chained (fast / release) vs unchained.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_chain_gpu.py -q > gpurun_out/chain_pytest.log 2>&1; echo "chain pytest rc=$?" >> gpurun_out/chain_pytest.log
grep -E "passed|failed|FAILED|rc=" gpurun_out/chain_pytest.log | head -20
for c in ${CFGS:-cfg2 cfg3 cfg1 cfg4}; do
  for v in persistent chained steps; do
    timeout 120 python bench.py --config $c --no-cpu --no-e2e --no-fused --launch $v > gpurun_out/qb.json 2> gpurun_out/qb.err
    python -c "import json;d=json.load(open('gpurun_out/qb.json'));print('$c', '$v', round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['frac'],4))" 2>/dev/null || { echo "$c $v FAILED"; tail -n 2 gpurun_out/qb.err; }
  done
done
