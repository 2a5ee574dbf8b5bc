"""Pin the CPU oracle to the reference: golden vectors + known answers.

The golden vectors were produced by the unmodified reference
(tests/golden/make_golden.py).  The oracle must reproduce them to 1e-12
relative (the reference's own oracle tolerance, test_control.py:337-362).
Known-answer cases restate the reference's hand tests
(test_control.py:63-234, test_dynamics.py:65-177, test_se3.py:76-188).
"""

import math

import numpy as np
import pytest

from oracle import flocksim_oracle as O

TOL = dict(rtol=1e-12, atol=1e-12)


def _cmds(g):
    return g["mode"], g["att_cmd"], g["vel_cmd"]


@pytest.mark.parametrize("case", ["att", "vel", "mixed", "edge"])
def test_pipeline_matches_reference_golden(golden, case):
    g = golden(case)
    s = g["state_in"]
    mode, att, vel = _cmds(g)
    with np.errstate(invalid="ignore"):
        out, info = O.step(s, mode, att, vel, O.Gains(), O.Robot(), float(g["dt"]))
    np.testing.assert_allclose(info["thrust"], g["thrust"], **TOL)
    np.testing.assert_allclose(np.stack(info["moment"]), g["moment"], **TOL)
    np.testing.assert_array_equal(info["gimbal"], g["gimbal"])
    np.testing.assert_array_equal(info["degenerate"], g["degenerate"])
    np.testing.assert_allclose(out, g["state_out"], equal_nan=True, **TOL)
    np.testing.assert_array_equal(info["clamped"], g["clamped"])
    np.testing.assert_array_equal(info["nonfinite"], g["nonfinite"])


def test_pipeline_golden_is_bitwise_for_regular_rows(golden):
    """Same expression order as the reference => identical float64 bits."""
    g = golden("att")
    out, info = O.step(g["state_in"], *_cmds(g), O.Gains(), O.Robot(), 0.01)
    assert np.array_equal(out, g["state_out"])
    assert np.array_equal(info["thrust"], g["thrust"])


def test_diag_operations_match_reference(golden):
    g = golden("diag")
    s = g["state_in"]
    q = tuple(s[3:7])
    w = tuple(s[10:13])
    yaw, gimbal = O.yaw_of(q)
    np.testing.assert_allclose(yaw, g["yaw"], **TOL)
    np.testing.assert_array_equal(gimbal, g["gimbal"])
    q_d, w_d = O.desired_attitude(yaw, g["roll"], g["pitch"], g["yaw_rate"])
    np.testing.assert_allclose(np.stack(q_d), g["q_d"], **TOL)
    np.testing.assert_allclose(np.stack(w_d), g["omega_d"], **TOL)
    e_r, e_w = O.attitude_errors(q, w, q_d, w_d)
    np.testing.assert_allclose(np.stack(e_r), g["e_rot"], **TOL)
    np.testing.assert_allclose(np.stack(e_w), g["e_rate"], **TOL)
    f, m = O.attitude_control(s, g["roll"], g["pitch"], g["yaw_rate"], g["thrust"],
                              O.Gains(), O.Robot())
    np.testing.assert_allclose(f, g["att_thrust"], **TOL)
    np.testing.assert_allclose(np.stack(m), g["att_moment"], **TOL)
    r, p, yr, th, dg = O.velocity_control(s, tuple(g["v_cmd"]), g["yaw_rate"], O.Gains(),
                                          O.Robot(), O.Limits())
    np.testing.assert_allclose(r, g["vel_roll"], **TOL)
    np.testing.assert_allclose(p, g["vel_pitch"], **TOL)
    np.testing.assert_allclose(yr, g["vel_yaw_rate"], **TOL)
    np.testing.assert_allclose(th, g["vel_thrust"], **TOL)
    np.testing.assert_array_equal(dg, g["vel_degenerate"])


@pytest.mark.parametrize("case", ["traj_att", "traj_vel"])
def test_trajectory_matches_reference(golden, case):
    g = golden(case)
    s = g["state_in"]
    mode, att, vel = _cmds(g)
    last = int(g["checkpoints"].max())
    for k in range(1, last + 1):
        s, _ = O.step(s, mode, att, vel, O.Gains(), O.Robot(), 0.01)
        if f"state_{k}" in g:
            np.testing.assert_allclose(s, g[f"state_{k}"], rtol=1e-10, atol=1e-10)


# --- known answers (reference hand cases) -------------------------------------

def _rest(n=1, p=(0.0, 0.0, 0.0)):
    s = np.zeros((13, n))
    s[0:3] = np.asarray(p, dtype=np.float64)[:, None]
    s[3] = 1.0
    return s


def test_known_forward_command_pitch():
    """test_control.py:186-196: pitch = atan2(1, 9.81) with unit gains."""
    gains = O.Gains(velocity=np.array([1.0, 1.0, 1.0]))
    r, p, _, f, _ = O.velocity_control(_rest(), (np.array([1.0]), np.zeros(1), np.zeros(1)),
                                       np.zeros(1), gains, O.Robot(), O.Limits())
    assert p[0] == pytest.approx(math.atan2(1.0, 9.81), abs=1e-15)
    assert r[0] == 0.0
    assert f[0] == pytest.approx(9.81, rel=1e-15)


def test_known_yaw_offset_error():
    """test_control.py:92-98: e_R = (0, 0, sin 0.4)."""
    q = O.rot_zyx(np.zeros(1), np.zeros(1), np.full(1, 0.4))
    one, zero = np.ones(1), np.zeros(1)
    e_r, _ = O.attitude_errors(q, (zero, zero, zero), (one, zero, zero, zero), (zero, zero, zero))
    np.testing.assert_allclose(np.stack(e_r)[:, 0], [0.0, 0.0, math.sin(0.4)], atol=1e-15)


def test_known_hover_fixed_point_velocity_mode():
    """test_control_closed_loop.py:91-103 (1000 steps, 1e-12)."""
    s0 = _rest(1, (1.0, -2.0, 3.0))
    s = s0.copy()
    for _ in range(1000):
        s, _ = O.step(s, np.ones(1, np.uint8), np.zeros((4, 1)), np.zeros((4, 1)),
                      O.Gains(), O.Robot(), 0.01)
    assert np.abs(s - s0).max() < 1e-12


def test_known_ballistic_closed_form():
    """test_dynamics.py:102-118: bitwise against the discrete recursion."""
    s = _rest()
    s[7] = 1.0
    for _ in range(100):
        s, _, _ = O.integrate(s, np.zeros(1), (np.zeros(1),) * 3, O.Robot(), 0.01)
    px, vz, pz = 0.0, 0.0, 0.0
    for _ in range(100):
        vz = vz + 0.01 * (0.0 * 1.0 - 9.81)
        pz = pz + 0.01 * vz
        px = px + 0.01 * 1.0
    assert s[0, 0] == px and s[2, 0] == pz and s[9, 0] == vz


def test_known_principal_spin_bitwise():
    """test_dynamics.py:120-127."""
    robot = O.Robot(inertia=np.diag([1.0, 1.0, 2.0]), moment_max=np.array([5.0, 5.0, 5.0]))
    s = _rest()
    s[12] = 3.0
    for _ in range(200):
        s, _, _ = O.integrate(s, np.zeros(1), (np.zeros(1),) * 3, robot, 0.01)
    assert (s[10, 0], s[11, 0], s[12, 0]) == (0.0, 0.0, 3.0)


def test_dt_validation():
    with pytest.raises(ValueError, match="dt"):
        O.integrate(_rest(), np.zeros(1), (np.zeros(1),) * 3, O.Robot(), 0.2)


# --- extension oracle properties (parity unpinned by the reference) ----------

@pytest.mark.parametrize("frame", [O.QUAD_X, O.HEX])
def test_allocation_pseudoinverse(frame):
    a = frame.matrix()
    np.testing.assert_allclose(a @ frame.pinv(), np.eye(4), atol=1e-12)


def test_allocation_unclamped_rotor_sum_equals_thrust():
    f = np.array([9.81, 12.0])
    m = (np.array([0.1, -0.2]), np.array([0.05, 0.1]), np.array([0.02, -0.03]))
    for frame in (O.QUAD_X, O.HEX):
        t, fr, mr = O.allocate(f, m, frame)
        np.testing.assert_allclose(t.sum(axis=0), f, rtol=1e-12)
        np.testing.assert_allclose(np.stack(mr), np.stack(m), atol=1e-12)


def test_position_hover_fixed_point():
    s = _rest(1, (1.0, 2.0, 3.0))
    pd = (np.ones(1), np.full(1, 2.0), np.full(1, 3.0))
    f, m, dg = O.position_control(s, pd, np.zeros(1), O.Gains(), O.Robot(), O.Limits())
    assert f[0] == 9.81 and all(x[0] == 0.0 for x in m) and not dg[0]


def test_position_controller_converges():
    """Closed loop from a 2 m offset with a yaw setpoint: reaches the goal."""
    robot, gains, lim = O.Robot(), O.Gains(), O.Limits()
    s = _rest(1, (0.0, 0.0, 0.0))
    pd = (np.full(1, 2.0), np.full(1, -1.0), np.full(1, 1.0))
    yaw_d = np.full(1, 0.7)
    for _ in range(1000):
        f, m, _ = O.position_control(s, pd, yaw_d, gains, robot, lim)
        s, _, _ = O.integrate(s, f, m, robot, 0.01)
    err = np.sqrt(sum((s[i] - pd[i]) ** 2 for i in range(3)))
    yaw, _ = O.yaw_of(tuple(s[3:7]))
    assert err[0] < 1e-2
    assert abs(yaw[0] - 0.7) < 1e-2


def test_saturate_and_scalar_step_match_reference_golden(golden):
    """dynamics.npz (make_golden_dynamics.py): saturate_batch, the scalar
    saturate and the scalar step of the unmodified reference."""
    g = golden("dynamics")
    f, m = O.saturate(g["sat_in"][0], tuple(g["sat_in"][1:4]), O.Robot())
    np.testing.assert_array_equal(np.concatenate([np.asarray(f)[None], np.stack(m)]),
                                  g["sat_out"])
    np.testing.assert_array_equal(g["sat1_out"], g["sat_out"][:, :16])
    s, w = g["step_state"], g["step_wrench"]
    out, _, _ = O.integrate(s, w[0], tuple(w[1:4]), O.Robot(), 0.01)
    np.testing.assert_allclose(out, g["step_out"], **TOL)
