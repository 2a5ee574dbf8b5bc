O=gpurun_out/s2y; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?" >> $O/smoke.txt
for c in cfg1 cfg3 cfg4; do
  timeout 900 python bench.py --config $c --no-cpu --no-e2e > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --no-cpu > $O/bench_default.json 2> $O/bench_default.err
timeout 300 python tools/gpu_cfg3_tune.py > $O/tune.txt 2>&1
