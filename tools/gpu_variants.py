"""Step time of stream-kernel variants, interleaved repetitions, min time
(developer tool)."""
import json, os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200.fleet import Fleet

torch.cuda.set_device(0); N.load()
n = 1 << 22
fleets = {m: Fleet(n, mode=m, dt=0.01, seed=3) for m in ('attitude', 'velocity', 'position')}

def once(f, steps=100):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): f.step()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps

variants = list(itertools.product((1, 2), (12, 16, 20), ('attitude', 'velocity', 'position')))
best = {}
for rep in range(4):
    for prec, ncw, mode in variants:
        N.set_tuning(N.FS_TUNE_PREC, prec); N.set_tuning(N.FS_TUNE_NCW, ncw)
        f = fleets[mode]
        for _ in range(3): f.step()
        ms = once(f)
        k = f'prec{prec}/ncw{ncw}/{mode}'
        best[k] = min(best.get(k, 1e9), ms)
N.set_tuning(N.FS_TUNE_PREC, -1); N.set_tuning(N.FS_TUNE_NCW, 0)
out = {k: (round(v * 1e3, 1), round(120 * n / v / 1e6)) for k, v in best.items()}
f3 = Fleet(1 << 21, mode='position', seed=3, reset_prob=0.01, want_stats=True)
for _ in range(3): f3.step()
out['cfg3'] = round(min(once(f3) for _ in range(3)) * 1e3, 1)
print(json.dumps(out, indent=0))
