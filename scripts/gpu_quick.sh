mkdir -p gpurun_out
python -m paper_2305_16510_b200.build
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python tools/gpu_e2e.py > gpurun_out/e2e_sweep.json 2> gpurun_out/e2e_sweep.err
