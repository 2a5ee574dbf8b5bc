"""PCIe probe (diagnostics): H2D alone, D2H alone, both at once (two streams),
1D vs 2D (13-plane chunk) copies.  Prints GB/s."""
import json
import torch

torch.cuda.set_device(0)
N = 256 << 20
a = torch.empty(N, dtype=torch.uint8, pin_memory=True)
b = torch.empty(N, dtype=torch.uint8, pin_memory=True)
da = torch.empty(N, dtype=torch.uint8, device="cuda")
db = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


def h2d():
    with torch.cuda.stream(s1):
        da.copy_(a, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        b.copy_(db, non_blocking=True)


def both():
    h2d()
    d2h()


out = {}
out["h2d_GBs"] = N / timed(h2d) / 1e9
out["d2h_GBs"] = N / timed(d2h) / 1e9
out["duplex_GBs_total"] = 2 * N / timed(both) / 1e9
# chunked: 8 chunks alternating on 4 streams each way
streams = [torch.cuda.Stream() for _ in range(8)]


def chunked():
    c = N // 8
    for k in range(8):
        with torch.cuda.stream(streams[k]):
            da[k * c:(k + 1) * c].copy_(a[k * c:(k + 1) * c], non_blocking=True)
            b[k * c:(k + 1) * c].copy_(db[k * c:(k + 1) * c], non_blocking=True)


out["chunked_duplex_GBs_total"] = 2 * N / timed(chunked) / 1e9
print(json.dumps(out))
