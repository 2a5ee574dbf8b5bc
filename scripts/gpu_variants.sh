mkdir -p gpurun_out
python -m paper_2305_16510_b200.build
timeout 900 python tools/gpu_variants.py > gpurun_out/variants.json 2> gpurun_out/variants.err; echo "rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for c in cfg1 cfg2 cfg3; do timeout 600 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/bench_g_$c.json 2> gpurun_out/bench_g_$c.err; done
