"""Generate golden vectors by running the UNMODIFIED reference (flocksim).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports ``flocksim`` from /root/reference/pkg/src (read-only; nothing is
copied), feeds it seeded inputs that are exactly representable in float32
(so the same values can be fed to the fp32 CUDA kernels), and stores the
reference's own float64 outputs in ``tests/golden/*.npz``.  Those fixtures
travel to the GPU box; /root/reference does not.

Cases
-----
att      config-1 distributions (attitude mode), N=1024, one pipeline step
vel      config-2 distributions (velocity mode), N=1024, one pipeline step
mixed    per-row mode, wide command ranges (test_control.py:271-294 style)
diag     desired_attitude / attitude_errors / velocity_control / yaw_of
edge     hand-made rows: hover, clamps, saturation, gimbal lock, NaN/inf
traj_att 100 attitude-mode steps, N=128 (checkpoints 1, 10, 100)
traj_vel 1000 velocity-mode steps, N=128 (checkpoints 1, 10, 100, 1000)
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import flocksim  # noqa: F401
    from flocksim import control, dynamics, se3
    return control, dynamics, se3


def f32(x):
    """Round to float32 and back: values both sides can represent exactly."""
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def shoemake(u1, u2, u3):
    """Uniform unit quaternion on S^3 from three U[0,1) draws (w first)."""
    a, b = np.sqrt(1.0 - u1), np.sqrt(u1)
    t1, t2 = 2 * np.pi * u2, 2 * np.pi * u3
    return np.stack([b * np.cos(t2), a * np.sin(t1), a * np.cos(t1), b * np.sin(t2)], axis=-1)


def cfg_states(rng, n):
    """Initial-state distributions of BASELINE.json config 0."""
    p = rng.uniform(-5.0, 5.0, (n, 3))
    q = shoemake(rng.random(n), rng.random(n), rng.random(n))
    q = f32(q)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)   # renormalize, then round again
    v = rng.normal(0.0, 1.0, (n, 3))
    w = rng.normal(0.0, 0.5, (n, 3))
    return f32(p), f32(q), f32(v), f32(w)


def planar(p, q, v, w):
    return np.concatenate([p.T, q.T, v.T, w.T], axis=0)


def run_pipeline(control, dynamics, p, q, v, w, mode, att, vel, dt):
    st = dynamics.RigidStateBatch(p=p, q=q, v=v, omega=w)
    cmds = control.CommandBatch(
        mode=mode,
        attitude=control.AttitudeCommands(roll=att[0], pitch=att[1], yaw_rate=att[2],
                                          thrust=att[3]),
        velocity=control.VelocityCommands(v=vel[0:3].T, yaw_rate=vel[3]))
    params, gains, limits = dynamics.RobotParams(), control.ControlGains(), control.ControlLimits()
    wrench, cflags = control.control_batch(st, cmds, gains, params, limits)
    out, sflags = dynamics.step_batch(st, params, wrench, dt)
    return dict(
        thrust=wrench.thrust, moment=wrench.moment.T,
        gimbal=cflags.gimbal_degenerate, degenerate=cflags.degenerate_acceleration,
        state_out=planar(out.p, out.q, out.v, out.omega),
        clamped=sflags.clamped, nonfinite=sflags.nonfinite)


def case_single(control, dynamics, name, seed, n, kind):
    rng = np.random.default_rng(seed)
    p, q, v, w = cfg_states(rng, n)
    mg = 9.81
    att = np.stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n),
                    rng.uniform(-1.0, 1.0, n), rng.uniform(0.5, 1.5, n) * mg])
    vel = np.concatenate([rng.normal(0.0, 1.0, (3, n)), rng.uniform(-1.0, 1.0, (1, n))])
    att, vel = f32(att), f32(vel)
    if kind == "att":
        mode = np.zeros(n, np.uint8)
        vel = np.zeros_like(vel)
    elif kind == "vel":
        mode = np.ones(n, np.uint8)
        att = np.zeros_like(att)
    else:
        raise ValueError(kind)
    res = run_pipeline(control, dynamics, p, q, v, w, mode, att, vel, 0.01)
    return dict(state_in=planar(p, q, v, w), mode=mode, att_cmd=att, vel_cmd=vel,
                dt=np.float64(0.01), **res)


def case_mixed(control, dynamics, seed=33, n=1024):
    """Wide ranges as in test_control.py:26-37 / 271-294 (incl. speed clamp)."""
    _, _, se3 = _import_reference()
    rng = np.random.default_rng(seed)
    ang = np.stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-1.2, 1.2, n),
                    rng.uniform(-math.pi, math.pi, n)])
    q = f32(se3.rot_zyx(ang[0], ang[1], ang[2]))
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    p = f32(rng.uniform(-5, 5, (n, 3)))
    v = f32(rng.uniform(-4, 4, (n, 3)))
    w = f32(rng.uniform(-3, 3, (n, 3)))
    q = f32(q)
    mode = rng.integers(0, 2, n).astype(np.uint8)
    att = f32(np.stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n),
                        rng.uniform(-1, 1, n), rng.uniform(0, 20, n)]))
    vel = f32(np.concatenate([rng.uniform(-6, 6, (3, n)), rng.uniform(-1, 1, (1, n))]))
    res = run_pipeline(control, dynamics, p, q, v, w, mode, att, vel, 0.01)
    return dict(state_in=planar(p, q, v, w), mode=mode, att_cmd=att, vel_cmd=vel,
                dt=np.float64(0.01), **res)


def case_diag(control, dynamics, se3, seed=99, n=512):
    """The four controller operations the reference's oracle test covers
    (test_control.py:304-362)."""
    rng = np.random.default_rng(seed)
    ang = np.stack([rng.uniform(-1.2, 1.2, n), rng.uniform(-1.2, 1.2, n),
                    rng.uniform(-math.pi, math.pi, n)])
    q = f32(se3.rot_zyx(ang[0], ang[1], ang[2]))
    q = f32(q / np.linalg.norm(q, axis=1, keepdims=True))
    p = f32(rng.uniform(-5, 5, (n, 3)))
    v = f32(rng.uniform(-4, 4, (n, 3)))
    w = f32(rng.uniform(-3, 3, (n, 3)))
    roll = f32(rng.uniform(-1.0, 1.0, n))
    pitch = f32(rng.uniform(-1.0, 1.0, n))
    yaw_rate = f32(rng.uniform(-2, 2, n))
    thrust = f32(rng.uniform(0, 24, n))
    v_cmd = f32(rng.uniform(-4, 4, (n, 3)))
    st = dynamics.RigidStateBatch(p=p, q=q, v=v, omega=w)
    params, gains, limits = dynamics.RobotParams(), control.ControlGains(), control.ControlLimits()
    att = control.AttitudeCommands(roll=roll, pitch=pitch, yaw_rate=yaw_rate, thrust=thrust)
    yaw, gimbal = se3.yaw_of(q)
    q_d, omega_d = control.desired_attitude(yaw, att)
    err = control.attitude_errors(q, w, q_d, omega_d)
    wrench = control.attitude_control(st, att, gains, params)
    att_out, degen = control.velocity_control(
        st, control.VelocityCommands(v=v_cmd, yaw_rate=yaw_rate), gains, params, limits)
    return dict(state_in=planar(p, q, v, w), roll=roll, pitch=pitch, yaw_rate=yaw_rate,
                thrust=thrust, v_cmd=v_cmd.T, yaw=yaw, gimbal=gimbal, q_d=q_d.T,
                omega_d=omega_d.T, e_rot=err.rotation.T, e_rate=err.rate.T,
                att_thrust=wrench.thrust, att_moment=wrench.moment.T,
                vel_roll=att_out.roll, vel_pitch=att_out.pitch,
                vel_yaw_rate=att_out.yaw_rate, vel_thrust=att_out.thrust,
                vel_degenerate=degen)


def case_edge(control, dynamics, se3):
    """Hand-made rows covering the reference's flag and clamp semantics
    (test_dynamics.py:65-177, 232-238; test_control.py:176-234)."""
    rows = []   # (p, q, v, w, mode, att(4), vel(4))
    I = [1.0, 0.0, 0.0, 0.0]
    mg = 9.81
    rows.append(([1, 2, 3], I, [0, 0, 0], [0, 0, 0], 0, [0, 0, 0, mg], [0] * 4))        # hover, att
    rows.append(([1, -2, 3], I, [0, 0, 0], [0, 0, 0], 1, [0] * 4, [0, 0, 0, 0]))        # hover, vel
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 0], 1, [0] * 4, [0, 0, -mg / 3, 0]))   # degenerate accel
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 0], 1, [0] * 4, [40, 0, 0, 0]))       # speed-cmd clamp
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 0], 1, [0] * 4, [5, 0, 0, 0]))        # tilt clamp
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 0], 1, [0] * 4, [1, 0, 0, 0.3]))      # forward pitch
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 0], 1, [0] * 4, [0, 1, 0, 0]))        # side roll
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 0], 0, [0.3, 0, 0, mg], [0] * 4))      # roll 0.3 hand case
    rows.append(([0, 0, 0], I, [1, 0, 0], [0, 0, 0], 0, [0, 0, 0, 0], [0] * 4))         # ballistic
    rows.append(([0, 0, 0], I, [30, 30, 30], [0, 0, 0], 0, [0, 0, 0, 25], [0] * 4))     # v clamp (|v|>50)
    rows.append(([0, 0, 0], I, [0, 0, 0], [80, 80, 0], 0, [0, 0, 0, mg], [0] * 4))     # omega clamp
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 3], 0, [0, 0, 0, 0], [0] * 4))         # principal spin
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 0], 0, [0, 0, 0, -2], [0] * 4))        # thrust < 0
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 0], 0, [0, 0, 0, 100], [0] * 4))       # thrust > max
    rows.append(([0, 0, 0], I, [0, 0, 0], [0, 0, 0], 0, [1.4, -1.4, 2.0, mg], [0] * 4))  # moment sat
    gl = se3.rot_zyx(0.2, math.pi / 2, 0.5)
    rows.append(([0, 0, 0], list(gl), [0, 0, 0], [0.1, 0.2, 0.3], 0, [0.1, 0.1, 0.1, mg], [0] * 4))  # gimbal
    rows.append(([0, 0, 0], list(se3.rot_zyx(0.0, 0.0, math.pi)), [0.5, 0.5, 0], [0, 0, 0], 1,
                 [0] * 4, [1, 1, 0, 0]))                                                    # yaw = pi
    rows.append(([0, 0, 0], list(se3.rot_zyx(0.0, 0.0, 0.4)), [0, 0, 0], [0, 0, 0], 0,
                 [0, 0, 0.7, mg], [0] * 4))                                                # yaw 0.4
    rows.append(([np.nan, 0, 0], I, [0, 0, 0], [0, 0, 0], 0, [0, 0, 0, 0], [0] * 4))   # NaN state
    rows.append(([np.inf, 0, 0], I, [0, 0, 0], [0, 0, 0], 0, [0, 0, 0, 0], [0] * 4))   # inf state
    rows.append(([0, 0, 0], I, [0, 0, 0], [1e-9, -2e-9, 3e-9], 0, [0, 0, 0, mg], [0] * 4))  # Taylor branch
    rows.append(([0, 0, 0], [-1.0, 0, 0, 0], [0, 0, 0], [0, 0, 0], 1, [0] * 4, [0.5, 0, 0, 0]))  # w<0 identity
    n = len(rows)
    p = f32(np.array([r[0] for r in rows], dtype=np.float64))
    q = np.array([r[1] for r in rows], dtype=np.float64)
    q = f32(f32(q) / np.linalg.norm(f32(q), axis=1, keepdims=True))
    v = f32(np.array([r[2] for r in rows], dtype=np.float64))
    w = f32(np.array([r[3] for r in rows], dtype=np.float64))
    mode = np.array([r[4] for r in rows], dtype=np.uint8)
    att = f32(np.array([r[5] for r in rows], dtype=np.float64).T)
    vel = f32(np.array([r[6] for r in rows], dtype=np.float64).T)
    res = run_pipeline(control, dynamics, p, q, v, w, mode, att, vel, 0.01)
    return dict(state_in=planar(p, q, v, w), mode=mode, att_cmd=att, vel_cmd=vel,
                dt=np.float64(0.01), **res)


def case_traj(control, dynamics, kind, steps, checkpoints, seed, n=128):
    rng = np.random.default_rng(seed)
    p, q, v, w = cfg_states(rng, n)
    mg = 9.81
    if kind == "att":
        att = f32(np.stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n),
                            rng.uniform(-1.0, 1.0, n), rng.uniform(0.5, 1.5, n) * mg]))
        vel = np.zeros((4, n))
        mode = np.zeros(n, np.uint8)
    else:
        vel = f32(np.concatenate([rng.normal(0.0, 1.0, (3, n)), rng.uniform(-1.0, 1.0, (1, n))]))
        att = np.zeros((4, n))
        mode = np.ones(n, np.uint8)
    params, gains, limits = dynamics.RobotParams(), control.ControlGains(), control.ControlLimits()
    cmds = control.CommandBatch(
        mode=mode,
        attitude=control.AttitudeCommands(roll=att[0], pitch=att[1], yaw_rate=att[2], thrust=att[3]),
        velocity=control.VelocityCommands(v=vel[0:3].T, yaw_rate=vel[3]))
    st = dynamics.RigidStateBatch(p=p, q=q, v=v, omega=w)
    out = dict(state_in=planar(p, q, v, w), mode=mode, att_cmd=att, vel_cmd=vel,
               dt=np.float64(0.01), checkpoints=np.array(checkpoints))
    for k in range(1, steps + 1):
        wrench, _ = control.control_batch(st, cmds, gains, params, limits)
        st, _ = dynamics.step_batch(st, params, wrench, 0.01)
        if k in checkpoints:
            out[f"state_{k}"] = planar(st.p, st.q, st.v, st.omega)
    return out


def main():
    control, dynamics, se3 = _import_reference()
    cases = {
        "att": case_single(control, dynamics, "att", 101, 1024, "att"),
        "vel": case_single(control, dynamics, "vel", 202, 1024, "vel"),
        "mixed": case_mixed(control, dynamics),
        "diag": case_diag(control, dynamics, se3),
        "edge": case_edge(control, dynamics, se3),
        "traj_att": case_traj(control, dynamics, "att", 100, (1, 10, 100), 303),
        "traj_vel": case_traj(control, dynamics, "vel", 1000, (1, 10, 100, 1000), 404),
    }
    for name, arrays in cases.items():
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **arrays)
        print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
