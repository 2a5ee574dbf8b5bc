"""cfg3 variants under process tunings (developer tool): position mode at
2^21, K = 200 steps in one fs_step_many launch; argv: KEY=VALUE tunings
(FS_TUNE_* names without the prefix), applied to every variant."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200.fleet import Fleet

torch.cuda.set_device(0)
N.load(os.environ.get("FS_LIB", N.LIB_PATH))
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    N.set_tuning(getattr(N, "FS_TUNE_" + k), int(v))
n, K = 1 << 21, int(os.environ.get("FS_K", "200"))
variants = {
    "velocity": dict(mode="velocity"),
    "plain": dict(),
    "stats": dict(want_stats=True),
    "reset": dict(reset_prob=0.01),
    "cfg3": dict(reset_prob=0.01, want_stats=True),
}
fleets = {k: Fleet(n, **dict(dict(mode="position", dt=0.01, seed=3), **v))
          for k, v in variants.items()}
graphs = {k: f.capture(K, persistent=True) for k, f in fleets.items()}


def once(g):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K


best = {}
for rep in range(4):
    for k, g in graphs.items():
        best[k] = min(best.get(k, 1e9), once(g))
out = {k: round(v * 1e3, 2) for k, v in best.items()}
out["frac_cfg3"] = round(121 * n / (best["cfg3"] * 1e-3) / 1e9 / 6545.3, 4)
out["tunings"] = sys.argv[1:]
print(json.dumps(out))
