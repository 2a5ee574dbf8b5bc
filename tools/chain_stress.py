"""Stress the persistent K-step launch against K single steps (developer
tool): repeats the flags_outputs / position-respawn cases per chain-acquire
setting and counts bitwise mismatches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200.fleet import Fleet

N.load(os.environ.get("FS_LIB", N.LIB_PATH))
cases = {
    "flags_outputs": dict(mode="velocity", want_flags=True, reset_prob=0.02),
    "position_respawn_stats": dict(mode="position", reset_prob=0.01, want_stats=True),
    "velocity": dict(mode="velocity"),
}
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for acq in (2, 3):
    N.set_tuning(N.FS_TUNE_CHAIN_ACQUIRE, acq)
    for name, kw in cases.items():
        for n in (1 << 17, 300001):
            bad = []
            for r in range(reps):
                a, b = Fleet(n, seed=13 + r, **kw), Fleet(n, seed=13 + r, **kw)
                for _ in range(9):
                    a.step()
                b.rollout(9, persistent=True)
                torch.cuda.synchronize()
                d = (a.state[:, :n] != b.state[:, :n]).any(0)
                dc = (a.cmd[:, :n] != b.cmd[:, :n]).any(0)
                if bool(d.any()) or bool(dc.any()):
                    idx = torch.nonzero(d | dc)[:5, 0].tolist()
                    bad.append((r, int(d.sum()), int(dc.sum()), idx))
            print(f"acq={acq} {name} n={n}: {len(bad)}/{reps} mismatching {bad[:3]}", flush=True)
