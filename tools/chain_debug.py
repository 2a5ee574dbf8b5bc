"""Debug helper: run one chain case step by step with blocking launches and
report which launch fails (python tools/chain_debug.py CASE N MODE)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2305_16510_b200.allocation import HEXAROTOR, QUAD_X  # noqa: E402
from paper_2305_16510_b200.fleet import Fleet  # noqa: E402

CASES = {
    "velocity": dict(mode="velocity"),
    "position_respawn_stats": dict(mode="position", reset_prob=0.01, want_stats=True),
    "flags_outputs": dict(mode="velocity", want_flags=True, reset_prob=0.02),
    "flags_only": dict(mode="velocity", want_flags=True),
    "stats_only": dict(mode="position", want_stats=True),
    "respawn_only": dict(mode="position", reset_prob=0.01),
    "hetero_rotors": dict(mode="position", hetero=True, airframes=(QUAD_X, HEXAROTOR),
                          rotor_dynamics=True),
}
case, n, how = sys.argv[1], int(sys.argv[2]), sys.argv[3]
f = Fleet(n, seed=11, **CASES[case])
torch.cuda.synchronize()
print("init ok", flush=True)
try:
    if how == "steps":
        for k in range(4):
            f.step()
            torch.cuda.synchronize()
            print("step", k, "ok", flush=True)
    elif how == "chained":
        f._chain_start(None)
        for k in range(4):
            f.step(chain=k)
            torch.cuda.synchronize()
            ts = f.tile_sync[:f.lib.fs_tile_sync_len(n)]
            print("chained step", k, "ok", ts[:12].tolist(), "min", int(ts.min()), "max",
                  int(ts.max()), "count==k+1", int((ts == k + 1).sum()), "of", ts.numel(), flush=True)
    else:
        f.step_many(4)
        torch.cuda.synchronize()
        print("step_many ok", flush=True)
except Exception as e:  # noqa: BLE001
    print("FAILED:", str(e).splitlines()[0], flush=True)
