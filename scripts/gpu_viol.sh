mkdir -p gpurun_out
python -m paper_2305_16510_b200.build
timeout 600 python tools/gpu_viol.py > gpurun_out/viol.json 2> gpurun_out/viol.err; echo "rc=$?"
