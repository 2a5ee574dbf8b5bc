"""Which controller stage must be wider than fp32 to meet 1e-5 rel / 1e-6 abs?"""
import numpy as np, sys
sys.path.insert(0, '.')
from oracle import flocksim_oracle as O
from oracle.workload import config_batch

def run(s, cmd, mode, T_R, T_V, T_A, T_M):
    """T_* = dtype for: R/yaw, velocity loop, attitude core, moment law."""
    c = lambda x, T: np.asarray(x).astype(T)
    q = [c(x, T_R) for x in s[3:7]]; qw,qx,qy,qz = q
    two, one = T_R(2), T_R(1)
    R = [[one-two*(qy*qy+qz*qz), two*(qx*qy-qw*qz), two*(qx*qz+qw*qy)],
         [two*(qx*qy+qw*qz), one-two*(qx*qx+qz*qz), two*(qy*qz-qw*qx)],
         [two*(qx*qz-qw*qy), two*(qy*qz+qw*qx), one-two*(qx*qx+qy*qy)]]
    ir = one/np.sqrt(R[0][0]**2+R[1][0]**2); cy, sy = R[0][0]*ir, R[1][0]*ir
    g = T_V(9.81)
    if mode == 'velocity':
        V = lambda x: c(x, T_V)
        vc = [V(x) for x in cmd[0:3]]; yr = cmd[3]
        vn2 = vc[0]*vc[0]+vc[1]*vc[1]+vc[2]*vc[2]
        scl = np.where(vn2 > T_V(25), T_V(5)/np.sqrt(vn2), T_V(1))
        vc = [x*scl for x in vc]
        cyv, syv = V(cy), V(sy); v = [V(x) for x in s[7:10]]
        vvx = cyv*v[0]+syv*v[1]; vvy = -syv*v[0]+cyv*v[1]
        ax = T_V(3)*(vc[0]-vvx); ay = T_V(3)*(vc[1]-vvy); az = T_V(3)*(vc[2]-v[2])+g
        R02, R12, R22 = V(R[0][2]), V(R[1][2]), V(R[2][2])
        thrust = ax*(cyv*R02+syv*R12)+ay*(-syv*R02+cyv*R12)+az*R22
        hxz2 = ax*ax+az*az; a2 = ay*ay+hxz2; ih = T_V(1)/np.sqrt(hxz2)
        ct, st = az*ih, ax*ih; hxz = hxz2*ih
        ctm, stm = T_V(np.cos(0.6)), T_V(np.sin(0.6))
        m = ct < ctm; ct = np.where(m, ctm, ct); st = np.where(m, np.copysign(stm, ax), st)
        ia = T_V(1)/np.sqrt(a2); cr, sr = hxz*ia, -ay*ia
        m = cr < ctm; cr = np.where(m, ctm, cr); sr = np.where(m, np.copysign(stm, -ay), sr)
    else:
        roll, pitch, yr, thrust = cmd
        sr, cr, st, ct = np.sin(roll), np.cos(roll), np.sin(pitch), np.cos(pitch)
    A_ = lambda x: c(x, T_A)
    cyA, syA = A_(cy), A_(sy); RA = [[A_(x) for x in row] for row in R]
    ct, st, cr, sr = A_(ct), A_(st), A_(cr), A_(sr)
    P0 = [cyA*RA[0][j]+syA*RA[1][j] for j in range(3)]
    P1 = [cyA*RA[1][j]-syA*RA[0][j] for j in range(3)]
    A21 = st*cr*P0[1] - sr*P1[1] + ct*cr*RA[2][1]
    A12 = st*sr*P0[2] + cr*P1[2] + ct*sr*RA[2][2]
    A02 = ct*P0[2] - st*RA[2][2]
    A20 = st*cr*P0[0] - sr*P1[0] + ct*cr*RA[2][0]
    A10 = st*sr*P0[0] + cr*P1[0] + ct*sr*RA[2][0]
    A01 = ct*P0[1] - st*RA[2][1]
    eR = [T_A(0.5)*(A21-A12), T_A(0.5)*(A02-A20), T_A(0.5)*(A10-A01)]
    Mt = lambda x: c(x, T_M)
    w = [Mt(x) for x in s[10:13]]; yrm = Mt(yr)
    eW = [w[i]-yrm*Mt(RA[2][i]) for i in range(3)]
    J = [T_M(0.01), T_M(0.01), T_M(0.02)]
    jw = [J[i]*w[i] for i in range(3)]
    gy = [w[1]*jw[2]-w[2]*jw[1], w[2]*jw[0]-w[0]*jw[2], w[0]*jw[1]-w[1]*jw[0]]
    kR = [8,8,2]; kW=[1.2,1.2,0.6]; Mm=[2,2,1]
    M = [np.clip(-T_M(kR[i])*Mt(eR[i])-T_M(kW[i])*eW[i]+gy[i], -Mm[i], Mm[i]) for i in range(3)]
    return np.clip(np.asarray(thrust, np.float64), 0, 25), [np.asarray(x, np.float64) for x in M]

F, D = np.float32, np.float64
for mode in ('velocity', 'attitude'):
    s, m, att, vel, _ = config_batch(mode, 1<<17, seed=7)
    cmd = vel if mode=='velocity' else att
    th, mo, _, _ = O.control(s, m, att, vel, O.Gains(), O.Robot())
    ok = np.abs(2*(s[4]*s[6]-s[3]*s[5])) < 0.99
    for combo in [(F,F,F,F),(D,F,F,F),(F,D,F,F),(D,D,F,F),(D,D,D,F),(D,D,F,D),(F,F,D,D),(D,D,D,D)]:
        f, M = run(s, cmd, mode, *combo)
        v = np.zeros(s.shape[1], bool)
        for got, ref in [(f, th)] + list(zip(M, mo)):
            v |= np.abs(got-ref) > 1e-6 + 1e-5*np.abs(ref)
        print(mode, ''.join('D' if t is D else 'F' for t in combo), f"viol={(v&ok).sum()} / {ok.sum()}")

print("---- DDDD violators detail")
mode='velocity'
s, m, att, vel, _ = config_batch(mode, 1<<17, seed=7)
th, mo, _, _ = O.control(s, m, att, vel, O.Gains(), O.Robot())
f, M = run(s, vel, mode, D, D, D, D)
for name, got, ref in [('f', f, th)] + [(f'M{i}', a, b) for i,(a,b) in enumerate(zip(M, mo))]:
    bad = np.nonzero(np.abs(got-ref) > 1e-6 + 1e-5*np.abs(ref))[0]
    for i in bad:
        r20 = abs(2*(s[4,i]*s[6,i]-s[3,i]*s[5,i]))
        print(name, i, got[i], ref[i], 'r20=', r20, 'ratt=', O.velocity_control(s[:, i:i+1], tuple(vel[0:3, i:i+1]), vel[3, i:i+1], O.Gains(), O.Robot(), O.Limits())[:2])
