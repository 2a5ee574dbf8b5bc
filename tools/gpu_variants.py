"""Step time of stream-kernel variants (developer tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200.fleet import Fleet

def timing(mode, n, steps=200):
    f = Fleet(n, mode=mode, dt=0.01, seed=3)
    for _ in range(5): f.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): f.step()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return round(ms * 1e3, 1), round(120 * n / ms / 1e6)

torch.cuda.set_device(0); N.load()
out = {}
for prec in (0, 2):
    N.set_tuning(N.FS_TUNE_PREC, prec)
    for ncw, vpt in ((16, 1), (16, 2)):
        N.set_tuning(N.FS_TUNE_NCW, ncw); N.set_tuning(N.FS_TUNE_VPT, vpt)
        for mode in ('attitude', 'velocity', 'position', 'mixed'):
            out[f'prec{prec}/ncw{ncw}/vpt{vpt}/{mode}'] = timing(mode, 1 << 22)
print(json.dumps(out, indent=0))
