#!/bin/bash
# RL bindings round: build, vecenv GPU tests, full GPU suite, world/vecenv bench lines.
set -x
mkdir -p gpurun_out
python -m paper_2305_16510_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_vecenv_gpu.py -x -q -m gpu > gpurun_out/pytest_vecenv.log 2>&1
echo "vecenv rc=$?" >> gpurun_out/pytest_vecenv.log
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
for c in world vecenv; do
  timeout 300 python bench.py --config $c --steps 200 --warmup 5 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
tail -3 gpurun_out/pytest_vecenv.log gpurun_out/pytest.log
cat gpurun_out/bench_world.json gpurun_out/bench_vecenv.json | cut -c1-400
