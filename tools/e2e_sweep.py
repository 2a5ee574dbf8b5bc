"""e2e pipeline sweep (diagnostics): bench.measure_e2e over chunks x streams."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS["cfg2"], global_n=1 << 22)
out = {}
for chunks in (8, 16, 32, 64, 128):
    for ns in (2, 4, 8):
        r = bench.measure_e2e(cfg, 1 << 22, dev, 10, chunks=chunks, nstreams=ns)
        out[f"{chunks}x{ns}"] = round(r["value"] / 1e8, 3)
print(json.dumps(out))
