"""Bitwise stress of the in-place streaming ring at bench sizes (developer
tool): for several configs, K steps in one persistent launch against K
per-step launches, repeated with fresh seeds; counts mismatching vehicles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_16510_b200.allocation import HEXAROTOR, QUAD_X
from paper_2305_16510_b200.fleet import Fleet

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cases = {
    "cfg2_velocity_2^22": (1 << 22, dict(mode="velocity"), 50),
    "cfg3_position_respawn_stats_2^21": (1 << 21, dict(mode="position", reset_prob=0.01,
                                                       want_stats=True), 50),
    "cfg4_hetero_rotors_2^21": (1 << 21, dict(mode="position", hetero=True,
                                              airframes=(QUAD_X, HEXAROTOR),
                                              airframe_split=1 << 20, rotor_dynamics=True), 30),
    "mixed_2^20": (1 << 20, dict(mode="mixed"), 30),
}
for name, (n, kw, K) in cases.items():
    bad = 0
    for r in range(reps):
        a, b = Fleet(n, seed=100 + r, **kw), Fleet(n, seed=100 + r, **kw)
        if kw.get("mode") == "mixed":
            m = (torch.arange(n, device=a.device) % 3 == 0).to(torch.uint8)
            a.mode_plane[:n].copy_(m)
            b.mode_plane[:n].copy_(m)
        for _ in range(K):
            a.step()
        b.rollout(K, persistent=True)
        torch.cuda.synchronize()
        ok = torch.equal(a.state[:, :n], b.state[:, :n]) and torch.equal(a.cmd[:, :n], b.cmd[:, :n])
        if a.stats_slots is not None:
            ok = ok and torch.equal(a.stats_local(), b.stats_local())
        bad += 0 if ok else 1
        del a, b
        torch.cuda.empty_cache()
    print(f"{name}: {bad}/{reps} mismatching", flush=True)
