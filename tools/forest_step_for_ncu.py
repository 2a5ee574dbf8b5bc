"""One steady-state forest World.step under the CUDA profiler API (developer
tool): bench.py's forest world (2^21 envs), FS_WARM steps (default 110, the
middle of the bench's timed window), then one step between
cudaProfilerStart/Stop -- run under `ncu --profile-from-start off` to capture
the step's three kernels (reset, streaming step, deferred collision test)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
r = bench.WorldRunner(n, 0, 2024, torch.device("cuda", 0), forest=True)
for _ in range(int(os.environ.get("FS_WARM", "110"))):
    r.step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
r.step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
