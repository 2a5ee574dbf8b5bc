mkdir -p gpurun_out
python -m paper_2305_16510_b200.build
timeout 600 python bench.py --steps 200 --no-cpu > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "rc=$?"
timeout 300 python -c "
import torch, time
x = torch.empty(256<<20, dtype=torch.uint8, pin_memory=True); y = torch.empty(256<<20, dtype=torch.uint8, device='cuda')
for _ in range(3): y.copy_(x, non_blocking=True); torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(10): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); h2d=10*256*2**20/(time.perf_counter()-t)/1e9
t=time.perf_counter()
for _ in range(10): x.copy_(y, non_blocking=True)
torch.cuda.synchronize(); d2h=10*256*2**20/(time.perf_counter()-t)/1e9
print('pcie GB/s h2d', h2d, 'd2h', d2h)
" > gpurun_out/pcie.txt 2>&1
