"""Free-space World.step bench worlds (developer tool): auto-reset rate per
step and step time, with the bench's commands / actions and with all-zero
commands (hover: no crashes, no resets) -- the cost of the inline resets."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2305_16510_b200 import _native as N

torch.cuda.set_device(0)
n = 1 << 22
out = {}
for name, kw in (("world", {}), ("vecenv", dict(actions=True))):
    for zero in (False, True):
        r = bench.WorldRunner(n, 0, 2024, torch.device("cuda", 0), **kw)
        if zero:
            if r.actions is not None:
                r.actions.zero_()
            else:
                r.cmds.buf.zero_()
        for _ in range(10):
            r.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        resets = 0
        e0.record()
        K = 200
        for _ in range(K):
            r.step()
        e1.record()
        torch.cuda.synchronize()
        resets = int(((r.world._info[:n] & N.FS_INFO_AUTORESET) != 0).sum())
        out[name + ("_zero" if zero else "")] = {"ms": round(e0.elapsed_time(e1) / K, 4),
                                                 "reset_frac_last_step": resets / n}
        del r
        torch.cuda.empty_cache()
print(json.dumps(out))
