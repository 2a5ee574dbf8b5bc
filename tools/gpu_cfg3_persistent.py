"""cfg3 cost breakdown on the persistent launch (developer tool): position
mode at 2^21 vehicles, K = 200 steps in one fs_step_many launch, with and
without statistics / Bernoulli re-spawns; interleaved repetitions, min time.
Optional argv: FS_TUNE_CHAIN_ACQUIRE, FS_TUNE_SPAWN_WAIT_NS, FS_TUNE_CONS_WAIT_NS."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200.fleet import Fleet

torch.cuda.set_device(0)
N.load(os.environ.get("FS_LIB", N.LIB_PATH))
for key, val in zip((N.FS_TUNE_CHAIN_ACQUIRE, N.FS_TUNE_SPAWN_WAIT_NS, N.FS_TUNE_CONS_WAIT_NS),
                    sys.argv[1:]):
    N.set_tuning(key, int(val))
n, K = 1 << 21, 200
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
print(json.dumps(out))
