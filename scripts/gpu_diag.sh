set -x
mkdir -p gpurun_out
python -m paper_2305_16510_b200.build
timeout 900 python tools/gpu_diag.py > gpurun_out/diag.json 2> gpurun_out/diag.err; echo "diag rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
