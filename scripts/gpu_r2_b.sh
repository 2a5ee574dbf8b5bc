# round 2: full GPU suite, smoke, default bench line, chain-acquire A/B
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
for acq in 0 1 0 1; do
  timeout 300 python bench.py --config cfg2 --no-cpu --no-fused --no-e2e --no-north-star --chain-acquire $acq >> gpurun_out/ab_cfg2.jsonl 2>/dev/null
  timeout 300 python bench.py --config cfg3 --n 2097152 --no-cpu --no-fused --no-e2e --chain-acquire $acq >> gpurun_out/ab_cfg3.jsonl 2>/dev/null
done
