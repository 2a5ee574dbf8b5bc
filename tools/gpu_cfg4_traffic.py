"""DRAM bytes per vehicle-step of fs_step_many (K = 20) for config-4-like
fleets with and without each feature (developer tool; run under ncu with
--metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:stream_kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_16510_b200.allocation import HEXAROTOR, QUAD_X
from paper_2305_16510_b200.fleet import Fleet

torch.cuda.set_device(0)
n = 1 << 23
variants = [
    ("cfg4", dict(hetero=True, airframes=(QUAD_X, HEXAROTOR), airframe_split=n // 2,
                  rotor_dynamics=True)),
    ("hetero_only", dict(hetero=True)),
    ("frames_no_rdyn", dict(hetero=True, airframes=(QUAD_X, HEXAROTOR), airframe_split=n // 2)),
    ("plain", dict()),
]
for name, kw in variants:
    f = Fleet(n, mode="position", dt=0.005, seed=1, **kw)
    f.step_many(20)
    torch.cuda.synchronize()
    print(name, flush=True)
    del f
    torch.cuda.empty_cache()
