# chain-acquire variants (bit 0 acquire loads, bit 1 proxy fence), cfg2 + cfg3@2^21
mkdir -p gpurun_out
for rep in 1 2; do for acq in 0 1 2 3; do
  timeout 300 python bench.py --config cfg2 --no-cpu --no-fused --no-e2e --no-north-star --chain-acquire $acq --steps 500 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2', $acq, d['ms_per_step']*1e3)" >> gpurun_out/acq.txt
  timeout 300 python bench.py --config cfg3 --n 2097152 --no-cpu --no-fused --no-e2e --chain-acquire $acq --steps 500 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', $acq, d['ms_per_step']*1e3)" >> gpurun_out/acq.txt
done; done
python tools/gpu_cfg3.py > gpurun_out/cfg3_breakdown_r2.json 2>&1
