"""Dump the velocity-mode rows that violate the bar (developer tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2305_16510_b200 as fs
from paper_2305_16510_b200 import _native as N
from oracle import flocksim_oracle as O
from oracle.workload import config_batch
torch.cuda.set_device(0); N.load()
res = {}
for prec in (2,):
    N.set_tuning(N.FS_TUNE_PREC, prec)
    for mode in ('velocity', 'attitude'):
        n = 1 << 20
        s, m, att, vel, _ = config_batch(mode, n, 11)
        st = fs.RigidStateBatch(p=s[0:3].T, q=s[3:7].T, v=s[7:10].T, omega=s[10:13].T)
        cmds = (fs.CommandBatch.all_velocity(fs.VelocityCommands(v=vel[0:3].T, yaw_rate=vel[3], validate=False))
                if mode == 'velocity' else fs.CommandBatch.all_attitude(fs.AttitudeCommands(*att, validate=False)))
        w = fs.WrenchBatch.empty(n)
        out, _ = fs.fused_step(st, cmds, fs.ControlGains(), fs.RobotParams(), 0.01, wrench=w)
        got = out.numpy(); gw = w.buf[:, :n].double().cpu().numpy()
        ref, info = O.step(s, m, att, vel, O.Gains(), O.Robot(), 0.01)
        rw = np.concatenate([info['thrust'][None], np.stack(info['moment'])])
        ok = np.abs(2*(s[4]*s[6]-s[3]*s[5])) < 0.99
        bad = ((np.abs(gw-rw) > 1e-6+1e-5*np.abs(rw)).any(0) | (np.abs(got-ref) > 1e-6+1e-5*np.abs(ref)).any(0)) & ok
        idx = np.nonzero(bad)[0]
        res[f'{mode}/prec{prec}'] = [dict(i=int(i), state=s[:, i].tolist(), att=att[:, i].tolist(), vel=vel[:, i].tolist(),
                                   got_w=gw[:, i].tolist(), ref_w=rw[:, i].tolist(), got_s=got[:, i].tolist(), ref_s=ref[:, i].tolist()) for i in idx[:10]]
print(json.dumps(res))
