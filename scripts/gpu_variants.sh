mkdir -p gpurun_out
python -m paper_2305_16510_b200.build
timeout 600 python tools/gpu_variants.py > gpurun_out/variants.json 2> gpurun_out/variants.err; echo "rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 300 $B > gpurun_out/plain_v.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 5 -c 1 -o gpurun_out/prof_v $B > gpurun_out/ncu_v.log 2>&1
echo "prof rc=$?"
