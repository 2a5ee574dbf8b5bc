"""float32 numpy emulation of the fused kernel (velocity / attitude modes) to
study the fp32 error budget against the float64 oracle (developer tool)."""
import numpy as np, sys
sys.path.insert(0, '.')
from oracle import flocksim_oracle as O
from oracle.workload import config_batch

F = np.float32

def kernel_f32(s, cmd, mode, dt=0.01, robust=False):
    s = s.astype(F)
    p, q, v, w = s[0:3], s[3:7], s[7:10], s[10:13]
    qw, qx, qy, qz = q
    two = F(2); one = F(1)
    R00 = one - two*(qy*qy+qz*qz); R01 = two*(qx*qy-qw*qz); R02 = two*(qx*qz+qw*qy)
    R10 = two*(qx*qy+qw*qz); R11 = one - two*(qx*qx+qz*qz); R12 = two*(qy*qz-qw*qx)
    R20 = two*(qx*qz-qw*qy); R21 = two*(qy*qz+qw*qx); R22 = one - two*(qx*qx+qy*qy)
    rho2 = R00*R00 + R10*R10
    ir = F(1)/np.sqrt(rho2)
    cy, sy = R00*ir, R10*ir
    g = F(9.81)
    if mode == 'velocity':
        vc = cmd[0:3].astype(F); yr = cmd[3].astype(F)
        vn2 = vc[0]**2+vc[1]**2+vc[2]**2
        sc = np.where(vn2 > F(25), F(5)/np.sqrt(vn2), F(1)).astype(F)
        vc = vc*sc
        vvx = cy*v[0]+sy*v[1]; vvy = -sy*v[0]+cy*v[1]
        ax = F(3)*(vc[0]-vvx); ay = F(3)*(vc[1]-vvy); az = F(3)*(vc[2]-v[2])+g
        vb3x = cy*R02+sy*R12; vb3y = -sy*R02+cy*R12
        thrust = ax*vb3x+ay*vb3y+az*R22
        hxz2 = ax*ax+az*az; a2 = ay*ay+hxz2
        ih = F(1)/np.sqrt(hxz2)
        ct, st = az*ih, ax*ih; hxz = hxz2*ih
        ctm, stm = F(np.cos(0.6)), F(np.sin(0.6))
        m = ct < ctm; ct = np.where(m, ctm, ct); st = np.where(m, np.copysign(stm, ax), st)
        ia = F(1)/np.sqrt(a2); cr, sr = hxz*ia, -ay*ia
        m = cr < ctm; cr = np.where(m, ctm, cr); sr = np.where(m, np.copysign(stm, -ay), sr)
    else:
        roll, pitch, yr, thrust = [cmd[k].astype(F) for k in range(4)]
        sr, cr = np.sin(roll.astype(np.float64)).astype(F), np.cos(roll.astype(np.float64)).astype(F)
        st, ct = np.sin(pitch.astype(np.float64)).astype(F), np.cos(pitch.astype(np.float64)).astype(F)
    if robust:
        # fp64 core for the attitude error
        D = np.float64
        Rm = [[D(x) for x in row] for row in ((R00,R01,R02),(R10,R11,R12),(R20,R21,R22))]
        qd = [D(x) for x in (qw,qx,qy,qz)]
        w_,x_,y_,z_ = qd
        Rm = [[1-2*(y_*y_+z_*z_), 2*(x_*y_-w_*z_), 2*(x_*z_+w_*y_)],[2*(x_*y_+w_*z_), 1-2*(x_*x_+z_*z_), 2*(y_*z_-w_*x_)],[2*(x_*z_-w_*y_), 2*(y_*z_+w_*x_), 1-2*(x_*x_+y_*y_)]]
        cyd, syd = D(cy), D(sy); n = np.sqrt(cyd*cyd+syd*syd); cyd/=n; syd/=n
        ctd, std, crd, srd = D(ct), D(st), D(cr), D(sr)
        P00 = cyd*Rm[0][0]+syd*Rm[1][0]; P01 = cyd*Rm[0][1]+syd*Rm[1][1]; P02 = cyd*Rm[0][2]+syd*Rm[1][2]
        P10 = cyd*Rm[1][0]-syd*Rm[0][0]; P11 = cyd*Rm[1][1]-syd*Rm[0][1]; P12 = cyd*Rm[1][2]-syd*Rm[0][2]
        A21 = std*crd*P01 - srd*P11 + ctd*crd*Rm[2][1]
        A12 = std*srd*P02 + crd*P12 + ctd*srd*Rm[2][2]
        A02 = ctd*P02 - std*Rm[2][2]
        A20 = std*crd*P00 - srd*P10 + ctd*crd*Rm[2][0]
        A10 = std*srd*P00 + crd*P10 + ctd*srd*Rm[2][0]
        A01 = ctd*P01 - std*Rm[2][1]
        eR = [F(0.5*(A21-A12)), F(0.5*(A02-A20)), F(0.5*(A10-A01))]
    else:
        P00 = cy*R00+sy*R10; P01 = cy*R01+sy*R11; P02 = cy*R02+sy*R12
        P10 = cy*R10-sy*R00; P11 = cy*R11-sy*R01; P12 = cy*R12-sy*R02
        stsr, stcr, ctsr, ctcr = st*sr, st*cr, ct*sr, ct*cr
        A21 = stcr*P01 - sr*P11 + ctcr*R21
        A12 = stsr*P02 + cr*P12 + ctsr*R22
        A02 = ct*P02 - st*R22
        A20 = stcr*P00 - sr*P10 + ctcr*R20
        A10 = stsr*P00 + cr*P10 + ctsr*R20
        A01 = ct*P01 - st*R21
        eR = [F(0.5)*(A21-A12), F(0.5)*(A02-A20), F(0.5)*(A10-A01)]
    eW = [w[0]-yr*R20, w[1]-yr*R21, w[2]-yr*R22]
    J = [F(0.01), F(0.01), F(0.02)]
    jw = [J[0]*w[0], J[1]*w[1], J[2]*w[2]]
    gy = [w[1]*jw[2]-w[2]*jw[1], w[2]*jw[0]-w[0]*jw[2], w[0]*jw[1]-w[1]*jw[0]]
    kR = [F(8),F(8),F(2)]; kW=[F(1.2),F(1.2),F(0.6)]; Mm=[F(2),F(2),F(1)]
    M = [np.clip(-kR[i]*eR[i]-kW[i]*eW[i]+gy[i], -Mm[i], Mm[i]).astype(F) for i in range(3)]
    f = np.clip(thrust, F(0), F(25)).astype(F)
    return f, M, eR

def compare(mode, n=1<<16, robust=False):
    s, m, att, vel, _ = config_batch(mode, n, seed=7)
    cmd = vel if mode=='velocity' else att
    f, M, eR = kernel_f32(s, cmd, mode, robust=robust)
    th, mo, _, _ = O.control(s, m, att, vel, O.Gains(), O.Robot())
    q = tuple(s[3:7]); yaw,_ = O.yaw_of(q)
    r20 = np.abs(2*(s[4]*s[6]-s[3]*s[5])); ok = r20 < 0.99
    for name, got, ref in [('thrust', f, th)] + [(f'M{i}', M[i], mo[i]) for i in range(3)]:
        d = np.abs(got.astype(np.float64)-ref)[ok]
        viol = (d > 1e-6 + 1e-5*np.abs(ref[ok])).mean()
        print(f"{mode:9s} robust={robust} {name}: max|d|={d.max():.2e} p99={np.percentile(d,99):.2e} viol={viol:.4%}")

for mode in ('velocity','attitude'):
    compare(mode)
    compare(mode, robust=True)
