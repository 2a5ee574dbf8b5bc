mkdir -p gpurun_out; rm -f gpurun_out/d.txt
for rep in 1 2; do for acq in 2 3 6; do
  timeout 300 python bench.py --config cfg2 --no-cpu --no-fused --no-e2e --no-north-star --chain-acquire $acq --steps 500 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2 acq', $acq, d['ms_per_step']*1e3)" >> gpurun_out/d.txt
done; done
python tools/gpu_cfg3_persistent.py 2 >> gpurun_out/d.txt 2>&1
FS_LIB=paper_2305_16510_b200/lib/libfs_diag_nospawn.so python tools/gpu_cfg3_persistent.py 2 >> gpurun_out/d.txt 2>&1
