"""Run one Fleet variant for profiling (developer tool).
python tools/gpu_fleet_variant.py MODE RESET_PROB STATS [steps] [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200.fleet import Fleet

mode, p, stats = sys.argv[1], float(sys.argv[2]), sys.argv[3] == "1"
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
n = int(sys.argv[5]) if len(sys.argv) > 5 else 1 << 21
torch.cuda.set_device(0)
N.load()
f = Fleet(n, mode=mode, dt=0.01, seed=3, reset_prob=p, want_stats=stats)
for _ in range(steps):
    f.step()
torch.cuda.synchronize()
print("ok")
