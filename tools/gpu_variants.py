"""Step time of stream-kernel variants (developer tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200.fleet import Fleet

def timing(mode, n, steps=200, **kw):
    f = Fleet(n, mode=mode, dt=0.01, seed=3, **kw)
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
which = sys.argv[1:] or ['prec']
if 'prec' in which:
    for prec in (0, 1, 2):
        N.set_tuning(N.FS_TUNE_PREC, prec)
        for mode in ('attitude', 'velocity', 'position', 'mixed'):
            out[f'prec{prec}/{mode}'] = timing(mode, 1 << 22)
    N.set_tuning(N.FS_TUNE_PREC, -1)
out['cfg3/position+reset+stats'] = timing('position', 1 << 21, reset_prob=0.01, want_stats=True)
out['cfg3/position+stats'] = timing('position', 1 << 21, want_stats=True)
out['cfg3/position'] = timing('position', 1 << 21)
print(json.dumps(out, indent=0))
