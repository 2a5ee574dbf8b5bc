mkdir -p gpurun_out
B="python bench.py --config cfg3 --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 300 $B > gpurun_out/cfg3_plain.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 5 -c 1 -o gpurun_out/cfg3_full $B > gpurun_out/ncu_c3.log 2>&1; echo "c3 rc=$?"
B="python bench.py --config cfg2 --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 5 -c 1 -o gpurun_out/cfg2_full $B > gpurun_out/ncu_c2.log 2>&1; echo "c2 rc=$?"
