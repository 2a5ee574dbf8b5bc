"""cfg3 cost breakdown (developer tool): position mode at 2^21, with and
without statistics / Bernoulli re-spawns, interleaved repetitions, min time;
plus per-kernel device durations from the torch profiler (CUPTI)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200.fleet import Fleet

torch.cuda.set_device(0)
N.load()
n = 1 << 21
variants = {
    "velocity": dict(reset_prob=0.0, want_stats=False, mode="velocity"),
    "plain": dict(reset_prob=0.0, want_stats=False),
    "stats": dict(reset_prob=0.0, want_stats=True),
    "reset": dict(reset_prob=0.01, want_stats=False),
    "cfg3": dict(reset_prob=0.01, want_stats=True),
}
fleets = {k: Fleet(n, **dict(dict(mode="position", dt=0.01, seed=3), **v))
          for k, v in variants.items()}


def once(f, steps=100):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        f.step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


best = {}
for rep in range(5):
    for k, f in fleets.items():
        for _ in range(3):
            f.step()
        best[k] = min(best.get(k, 1e9), once(f))
out = {k: round(v * 1e3, 2) for k, v in best.items()}
f = fleets["cfg3"]
for ncw in (12, 16, 20):
    N.set_tuning(N.FS_TUNE_NCW, ncw)
    for _ in range(3):
        f.step()
    out[f"cfg3/ncw{ncw}"] = round(min(once(f) for _ in range(3)) * 1e3, 2)
N.set_tuning(N.FS_TUNE_NCW, 0)

from torch.profiler import ProfilerActivity, profile

kern = {}
for k in ("reset", "cfg3"):
    f = fleets[k]
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(50):
            f.step()
        torch.cuda.synchronize()
    for e in prof.key_averages():
        if e.device_type is not None and "CUDA" in str(e.device_type) and e.count >= 50:
            kern[f"{k}:{e.key[:60]}"] = (e.count, round(e.device_time / 1.0, 2))
out["kernels_us_avg"] = kern
print(json.dumps(out, indent=1))
