"""Per-step time of long persistent launches (developer tool): cfg2 at 2^22,
1000 steps as one fs_step_many launch vs 5 x 200 and 10 x 100 launches in
one CUDA graph, interleaved, each timed 3 times."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2305_16510_b200.fleet import Fleet

torch.cuda.set_device(0)
n = 1 << 22
f = Fleet(n, mode="velocity", dt=0.01, seed=3)


def graph(chunk, total=1000):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    import ctypes as C
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(total // chunk):
                f.step_many(chunk, C.c_void_p(s.cuda_stream))
    torch.cuda.current_stream().wait_stream(s)
    return g


gs = {c: graph(c) for c in (1000, 200, 100)}
res = {c: [] for c in gs}
for rep in range(3):
    for c, g in gs.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[c].append(round(e0.elapsed_time(e1), 3))
print(json.dumps({f"{c}-step launches: us/step": [round(x, 2) for x in v] for c, v in res.items()}))
