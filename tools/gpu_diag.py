"""GPU diagnostics: parity violation rates vs the float64 oracle and step
timing, per kernel variant (developer tool; writes JSON to stdout)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_16510_b200 as fs
from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200.fleet import Fleet
from oracle import flocksim_oracle as O
from oracle.workload import config_batch

def parity(mode, n, seed=11):
    s, m, att, vel, pos = config_batch(mode, n, seed)
    if mode == 'mixed':
        m = (np.arange(n) % 2).astype(np.uint8)
    st = fs.RigidStateBatch(p=s[0:3].T, q=s[3:7].T, v=s[7:10].T, omega=s[10:13].T)
    A = fs.AttitudeCommands(*att, validate=False)
    V = fs.VelocityCommands(v=vel[0:3].T, yaw_rate=vel[3], validate=False)
    if mode == 'attitude': cmds = fs.CommandBatch.all_attitude(A)
    elif mode == 'velocity': cmds = fs.CommandBatch.all_velocity(V)
    else: cmds = fs.CommandBatch(mode=m, attitude=A, velocity=V)
    w = fs.WrenchBatch.empty(n)
    out, flags = fs.fused_step(st, cmds, fs.ControlGains(), fs.RobotParams(), 0.01, wrench=w)
    got = out.numpy(); gw = w.buf[:, :n].double().cpu().numpy()
    ref, info = O.step(s, m, att, vel, O.Gains(), O.Robot(), 0.01)
    rw = np.concatenate([info['thrust'][None], np.stack(info['moment'])])
    r20 = np.abs(2*(s[4]*s[6]-s[3]*s[5])); ok = r20 < 0.99
    res = {}
    for name, g, r in [('p', got[0:3], ref[0:3]), ('q', got[3:7], ref[3:7]), ('v', got[7:10], ref[7:10]),
                       ('w', got[10:13], ref[10:13]), ('wrench', gw, rw)]:
        d = np.abs(g - r)
        ratio = d / (1e-6 + 1e-5*np.abs(r))
        bad = (ratio > 1).any(axis=0)
        res[name] = dict(viol_out=int((bad & ok).sum()), viol_band=int((bad & ~ok).sum()),
                         max_abs=float(d[:, ok].max()), max_ratio=float(ratio[:, ok].max()),
                         p9999_ratio=float(np.percentile(ratio[:, ok].max(axis=0), 99.99)))
    res['n_out'] = int(ok.sum())
    return res, got

def timing(mode, n, steps=200, kernel=0):
    f = Fleet(n, mode=mode, dt=0.01, seed=3)
    for _ in range(5): f.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps): f.step()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    return dict(ms_per_step=ms, GBps=120*n/ms/1e6, vsteps=n/ms*1e3)

torch.cuda.set_device(0)
N.load()
out = {}
for prec in (0, 1, 2):
    N.set_tuning(N.FS_TUNE_PREC, prec)
    for mode in ('attitude', 'velocity', 'mixed'):
        res, _ = parity(mode, 1 << 21, seed=23)
        out[f'parity/prec{prec}/{mode}'] = res
N.set_tuning(N.FS_TUNE_PREC, -1)
print(json.dumps(out, indent=1))
