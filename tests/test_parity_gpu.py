"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden
vectors and the pinned CPU oracle, on identical fp32-representable inputs.

Tolerance (north_star): 1e-5 relative / 1e-6 absolute per step for every
vehicle outside the gimbal conditioning band (tests/fs_parity.py).
"""

import numpy as np
import pytest
import torch

from oracle import flocksim_oracle as O
from fs_parity import assert_drift, assert_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fs():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2305_16510_b200 as fs
    fs._native.load()
    return fs


def _batch(fs, planar):
    s = np.asarray(planar, dtype=np.float32)
    return fs.RigidStateBatch(p=s[0:3].T, q=s[3:7].T, v=s[7:10].T, omega=s[10:13].T)


def _cmds(fs, g):
    n = g["mode"].shape[0]
    att = fs.AttitudeCommands(*[g["att_cmd"][k].astype(np.float32) for k in range(4)],
                              validate=False)
    vel = fs.VelocityCommands(v=g["vel_cmd"][0:3].T.astype(np.float32),
                              yaw_rate=g["vel_cmd"][3].astype(np.float32), validate=False)
    modes = np.unique(g["mode"])
    if len(modes) == 1 and modes[0] == 0:
        return fs.CommandBatch.all_attitude(att)
    if len(modes) == 1 and modes[0] == 1:
        return fs.CommandBatch.all_velocity(vel)
    return fs.CommandBatch(mode=g["mode"], attitude=att, velocity=vel)


def _oracle_fn(g, what):
    """The pinned oracle as a function of (state columns, column ids)."""
    def fn(s, cols):
        with np.errstate(invalid="ignore"):
            out, info = O.step(s, g["mode"][cols], g["att_cmd"][:, cols], g["vel_cmd"][:, cols],
                               O.Gains(), O.Robot(), 0.01)
        if what == "state":
            return out
        return np.concatenate([info["thrust"][None], np.stack(info["moment"])])
    return fn


@pytest.mark.parametrize("case", ["att", "vel", "mixed", "edge"])
def test_control_batch_matches_golden(fs, golden, case):
    g = golden(case)
    st = _batch(fs, g["state_in"])
    wrench, flags = fs.control_batch(st, _cmds(fs, g), fs.ControlGains(), fs.RobotParams())
    got = wrench.buf[:, :st.n].double().cpu().numpy()
    ref = np.concatenate([g["thrust"][None], g["moment"]])
    assert_parity(got, ref, g["state_in"], f"{case}: wrench", _oracle_fn(g, "wrench"))
    np.testing.assert_array_equal(flags.gimbal_degenerate.cpu().numpy(), g["gimbal"])
    np.testing.assert_array_equal(flags.degenerate_acceleration.cpu().numpy(), g["degenerate"])


@pytest.mark.parametrize("case", ["att", "vel", "mixed", "edge"])
def test_fused_step_matches_golden(fs, golden, case):
    g = golden(case)
    st = _batch(fs, g["state_in"])
    out, flags = fs.fused_step(st, _cmds(fs, g), fs.ControlGains(), fs.RobotParams(), 0.01)
    got = out.numpy()
    assert_parity(got, g["state_out"], g["state_in"], f"{case}: state", _oracle_fn(g, "state"))
    np.testing.assert_array_equal(flags.clamped.cpu().numpy(), g["clamped"])
    np.testing.assert_array_equal(flags.nonfinite.cpu().numpy(), g["nonfinite"])


@pytest.mark.parametrize("case", ["att", "vel", "mixed", "edge"])
def test_unfused_pipeline_matches_golden(fs, golden, case):
    """control_batch -> step_batch through the two drop-in entry points."""
    g = golden(case)
    st = _batch(fs, g["state_in"])
    params = fs.RobotParams()
    wrench, _ = fs.control_batch(st, _cmds(fs, g), fs.ControlGains(), params)
    out, flags = fs.step_batch(st, params, wrench, 0.01)
    assert_parity(out.numpy(), g["state_out"], g["state_in"], f"{case}: state (unfused)",
                  _oracle_fn(g, "state"))
    np.testing.assert_array_equal(flags.nonfinite.cpu().numpy(), g["nonfinite"])


def test_diag_operations_match_golden(fs, golden):
    g = golden("diag")
    s = g["state_in"]
    st = _batch(fs, s)
    yaw, gimbal = fs.yaw_of(st.q)
    band = np.abs(2.0 * (s[4] * s[6] - s[3] * s[5]))
    ok = band < 0.99
    np.testing.assert_allclose(yaw.double().cpu().numpy()[ok], g["yaw"][ok], rtol=1e-5, atol=2e-6)
    np.testing.assert_array_equal(gimbal.cpu().numpy(), g["gimbal"])
    att = fs.AttitudeCommands(g["roll"].astype(np.float32), g["pitch"].astype(np.float32),
                              g["yaw_rate"].astype(np.float32), g["thrust"].astype(np.float32))
    qd, wd = fs.desired_attitude(g["yaw"].astype(np.float32), att)
    assert_parity(qd.T.double().cpu().numpy(), g["q_d"], s, "q_d")
    assert_parity(wd.T.double().cpu().numpy(), g["omega_d"], s, "omega_d")
    err = fs.attitude_errors(st.q, st.omega, g["q_d"].T.astype(np.float32),
                             g["omega_d"].T.astype(np.float32))
    assert_parity(err.rotation.T.double().cpu().numpy(), g["e_rot"], s, "e_R")
    assert_parity(err.rate.T.double().cpu().numpy(), g["e_rate"], s, "e_W")
    w = fs.attitude_control(st, att, fs.ControlGains(), fs.RobotParams())
    assert_parity(w.buf[:, :st.n].double().cpu().numpy(),
                  np.concatenate([g["att_thrust"][None], g["att_moment"]]), s, "attitude_control")
    vel = fs.VelocityCommands(v=g["v_cmd"].T.astype(np.float32),
                              yaw_rate=g["yaw_rate"].astype(np.float32))
    ac, dg = fs.velocity_control(st, vel, fs.ControlGains(), fs.RobotParams())
    got = ac.buf[:, :st.n].double().cpu().numpy()
    ref = np.stack([g["vel_roll"], g["vel_pitch"], g["vel_yaw_rate"], g["vel_thrust"]])
    assert_parity(got, ref, s, "velocity_control")
    np.testing.assert_array_equal(dg.cpu().numpy(), g["vel_degenerate"])


@pytest.mark.parametrize("case", ["traj_att", "traj_vel"])
def test_trajectory_drift_bound(fs, golden, case):
    """K-step drift vs the pure float64 reference, bounded by a multiple of
    the fp32-storage floor (float64 math, state rounded to fp32 each step;
    SURVEY.md Appendix C.6)."""
    g = golden(case)
    st = _batch(fs, g["state_in"])
    cmds = _cmds(fs, g)
    gains, params = fs.ControlGains(), fs.RobotParams()
    mode, att, vel = g["mode"], g["att_cmd"], g["vel_cmd"]
    floor_state = g["state_in"].copy()
    last = int(g["checkpoints"].max())
    for k in range(1, last + 1):
        st, _ = fs.fused_step(st, cmds, gains, params, 0.01, out=st)
        floor_state, _ = O.step(floor_state, mode, att, vel, O.Gains(), O.Robot(), 0.01)
        floor_state = floor_state.astype(np.float32).astype(np.float64)
        if f"state_{k}" in g:
            assert_drift(st.numpy(), g[f"state_{k}"], floor_state, f"{case} step {k}")


def test_known_answers(fs):
    """Reference hand cases through the GPU API (test_control.py:176-234)."""
    params, gains = fs.RobotParams(), fs.ControlGains(velocity=[1.0, 1.0, 1.0])
    st = fs.RigidStateBatch.rest(1)
    att, dg = fs.velocity_control(st, fs.VelocityCommands.single([1.0, 0.0, 0.0], 0.0), gains,
                                  params)
    assert att.pitch.item() == pytest.approx(np.arctan2(1.0, 9.81), abs=1e-6)
    assert att.roll.item() == 0.0
    assert att.thrust.item() == pytest.approx(9.81, rel=1e-6)
    att, dg = fs.velocity_control(st, fs.VelocityCommands.single([0.0, 0.0, -9.81 / 3.0], 0.0),
                                  fs.ControlGains(), params)
    assert bool(dg[0]) and att.roll.item() == 0.0 and att.thrust.item() == pytest.approx(9.81)


def test_hover_fixed_point_1000_steps(fs):
    """test_control_closed_loop.py:91-103 in fp32: the rest state is an
    exact fixed point of the fused step."""
    st = fs.RigidStateBatch.rest(8, p=np.tile([1.0, -2.0, 3.0], (8, 1)))
    ref = st.numpy()
    cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=np.zeros((8, 3)),
                                                            yaw_rate=np.zeros(8)))
    for _ in range(1000):
        st, _ = fs.fused_step(st, cmds, fs.ControlGains(), fs.RobotParams(), 0.01, out=st)
    assert np.array_equal(st.numpy(), ref)
