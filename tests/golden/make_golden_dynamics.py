"""Golden vectors for the scalar / saturation drop-ins, from the UNMODIFIED
reference (flocksim.dynamics).  Run in the build container:

    python tests/golden/make_golden_dynamics.py

Writes tests/golden/dynamics.npz:

sat_in / sat_out    saturate_batch (dynamics.py:214-218) on 2048 wrenches
                    spanning every clamp (thrust < 0, > thrust_max, moments
                    beyond +-moment_max), float32-representable inputs
sat1_in / sat1_out  the scalar saturate (dynamics.py:221-226) row by row
step_state / step_wrench / step_out
                    the scalar step (dynamics.py:344-358) on 64 random robots
                    (test_dynamics.py random_batch-style ranges), one row at a
                    time, dt = 0.01
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def main():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from flocksim import dynamics as D
    from flocksim import se3

    rng = np.random.default_rng(2305)
    params = D.RobotParams()
    n = 2048
    thrust = f32(rng.uniform(-10.0, 40.0, n))
    moment = f32(rng.uniform(-5.0, 5.0, (n, 3)))
    thrust[:4] = [0.0, 25.0, -0.0, 24.999998]
    moment[:4] = [[2.0, -2.0, 1.0], [-2.0, 2.0, -1.0], [0.0, 0.0, 0.0], [1.9999999, 0.5, -0.25]]
    thrust, moment = f32(thrust), f32(moment)     # (the hand rows too: both sides see them)
    sat = D.saturate_batch(D.WrenchBatch(thrust=thrust, moment=moment), params)
    sat_in = np.concatenate([thrust[None], moment.T])
    sat_out = np.concatenate([sat.thrust[None], sat.moment.T])

    m1 = 16
    sat1_out = np.zeros((4, m1))
    for i in range(m1):
        w = D.saturate(D.Wrench(thrust=thrust[i], moment=moment[i]), params)
        sat1_out[:, i] = [w.thrust, *w.moment]

    k = 64
    p = f32(rng.uniform(-5.0, 5.0, (k, 3)))
    q = f32(se3.quat_normalize(rng.normal(size=(k, 4))))
    q = f32(q / np.linalg.norm(q, axis=1, keepdims=True))
    v = f32(rng.uniform(-4.0, 4.0, (k, 3)))
    w = f32(rng.uniform(-3.0, 3.0, (k, 3)))
    ft = f32(rng.uniform(0.0, params.thrust_max, k))
    fm = f32(rng.uniform(-1.0, 1.0, (k, 3)) * params.moment_max)
    out = np.zeros((13, k))
    for i in range(k):
        s1 = D.step(D.RigidState(p=p[i], q=q[i], v=v[i], omega=w[i]), params,
                    D.Wrench(thrust=ft[i], moment=fm[i]), 0.01)
        out[:, i] = np.concatenate([s1.p, s1.q, s1.v, s1.omega])
    np.savez_compressed(
        os.path.join(HERE, "dynamics.npz"), sat_in=sat_in, sat_out=sat_out,
        sat1_in=sat_in[:, :m1], sat1_out=sat1_out,
        step_state=np.concatenate([p.T, q.T, v.T, w.T]),
        step_wrench=np.concatenate([ft[None], fm.T]), step_out=out)
    print("wrote dynamics.npz")


if __name__ == "__main__":
    main()
