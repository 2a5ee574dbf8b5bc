"""Fixed cost of one persistent fs_step_many launch (developer tool): cfg2
(velocity, 2^22) graph replays of K steps for several K; the intercept of
time = a + b K is the per-launch cost (launch, tile-counter reset, ramp, drain)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_16510_b200.fleet import Fleet

torch.cuda.set_device(0)
n = 1 << 22
f = Fleet(n, mode="velocity", dt=0.01, seed=3)
out = {}
for K in (1, 2, 5, 20, 100, 400):
    g = f.capture(K, persistent=True)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[K] = round(best * 1e3, 1)
ks = sorted(out)
b = (out[400] - out[100]) / 300
a = out[100] - 100 * b
print(json.dumps({"us_total": out, "us_per_step_slope": round(b, 2), "us_intercept": round(a, 1)}))
