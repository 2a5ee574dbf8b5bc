#!/bin/bash
mkdir -p gpurun_out
python -m paper_2305_16510_b200.build > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python -m pytest tests/test_fleet_gpu.py -x -q -m gpu > gpurun_out/pytest_fleet.log 2>&1; echo "fleet rc=$?" >> gpurun_out/pytest_fleet.log
tail -n 4 gpurun_out/pytest_fleet.log
timeout 600 python tools/gpu_cfg3.py > gpurun_out/cfg3.json 2> gpurun_out/cfg3.err; echo "rc=$?"
cat gpurun_out/cfg3.json; tail -n 5 gpurun_out/cfg3.err
