"""Sweep the e2e pipeline shape (developer tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
torch.cuda.set_device(0)
dev = torch.device('cuda', 0)
cfg = dict(bench.CONFIGS['cfg2'])
out = {}
for ch, st in ((4, 2), (8, 3), (16, 4), (32, 4), (64, 8)):
    r = bench.measure_e2e(cfg, 1 << 22, dev, 10, chunks=ch, nstreams=st)
    out[f'{ch}x{st}'] = r['value']
print(json.dumps(out, indent=0))
