"""Forest World.step breakdown in steady state (developer tool): bench.py's
forest world at 2^21 envs, 200 warm-up steps, then 20 profiled steps;
per-kernel device time from the torch profiler (CUPTI) against the step's
event-timed wall time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile

from paper_2305_16510_b200 import _native as N
N.load(os.environ.get("FS_LIB", N.LIB_PATH))
import bench

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 21
r = bench.WorldRunner(n, 0, 2024, torch.device("cuda", 0), forest=True)
if os.environ.get("FS_BREAKDOWN_NO_INST_POSE"):
    r.world._ob.inst_pose = None      # experiment: resets skip the instance-pose planes
for _ in range(int(os.environ.get("FS_WARM", "200"))):
    r.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    r.step()
e1.record()
torch.cuda.synchronize()
wall = e0.elapsed_time(e1) / 20
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(20):
        r.step()
    torch.cuda.synchronize()
out = {"ms_per_step_events": wall}
for ev in prof.key_averages():
    if ev.device_type is not None and "CUDA" in str(ev.device_type):
        out[ev.key[:60]] = {"count": ev.count, "us_avg": round(ev.device_time / 1.0, 1)}
wl = r.world._worklist
out["worklist_total"] = int(wl[2].item())
out["autoreset_last_step"] = int(((r.world._info[:n] & 32) != 0).sum().item())
ws = getattr(r.world, "_walk_slots", None)
if ws is not None:
    v = int(ws.item())
    out["walk_slots_counter"] = v
    out["walk_slots_hi32"] = v >> 32
print(json.dumps(out, indent=1))
