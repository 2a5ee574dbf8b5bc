mkdir -p gpurun_out
python -m paper_2305_16510_b200.build
timeout 600 python bench.py --config world --no-cpu > gpurun_out/bench_world.json 2> gpurun_out/bench_world.err; echo "rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
