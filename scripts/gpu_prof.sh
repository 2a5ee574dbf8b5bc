set -x
mkdir -p gpurun_out
python -m paper_2305_16510_b200.build
timeout 900 python tools/gpu_diag.py > gpurun_out/diag2.json 2> gpurun_out/diag2.err; echo "diag rc=$?"
for P in 0 1 2; do
  B="python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu --no-fused --prec $P"
  timeout 300 $B > gpurun_out/plain_p$P.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:stream_kernel -s 5 -c 1 -o gpurun_out/prof_p$P $B > gpurun_out/ncu_p$P.log 2>&1
  echo "prof p$P rc=$?"
done
