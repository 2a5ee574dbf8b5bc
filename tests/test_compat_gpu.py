"""The reference-side drop-in (paper_2305_16510_b200/compat.py) swapped into
the UNMODIFIED reference's own callers (oracle/_ref wheels, built by
oracle/build_ref.py):

* ``World._pipeline`` (world.py:254-257) of a flocksim World: every step of
  a 200-step episode run (auto-resets, truncations, out-of-bounds
  terminations) reproduces the unswapped World's StepResult on identical
  fp32-representable inputs -- observations and rewards at the parity bar,
  every flag equal;
* ``bench._pipeline_step`` (bench.py:146-149): the reference's own
  bench_dynamics runs through it; one step matches at the bar and 100 steps
  stay within the stated drift bound (tests/fs_parity.py);
* ``control_batch`` / ``step_batch`` on the reference's golden inputs
  (mixed per-row modes: fs_step_host_ex's FS_MODE_MIXED path).
"""

import numpy as np
import pytest
import torch

from fs_parity import assert_drift, assert_parity
from oracle import flocksim_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built (python oracle/build_ref.py)")
    return {m: R.flocksim(m) for m in ("world", "config", "bench", "control", "dynamics")}


@pytest.fixture(scope="module")
def compat():
    from paper_2305_16510_b200 import compat
    return compat


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def _round_states(fd, s):
    return fd.RigidStateBatch(p=f32(s.p), q=f32(s.q), v=f32(s.v), omega=f32(s.omega))


def _round_cmds(fc, c):
    return fc.CommandBatch(
        mode=c.mode,
        attitude=fc.AttitudeCommands(roll=f32(c.attitude.roll), pitch=f32(c.attitude.pitch),
                                     yaw_rate=f32(c.attitude.yaw_rate),
                                     thrust=f32(c.attitude.thrust)),
        velocity=fc.VelocityCommands(v=f32(c.velocity.v), yaw_rate=f32(c.velocity.yaw_rate)))


def _planar(s):
    return np.concatenate([s.p.T, s.q.T, s.v.T, s.omega.T])


def test_world_pipeline_swap_reproduces_reference_world(ref, compat):
    fw, fcfg, fb, fc, fd = (ref[k] for k in ("world", "config", "bench", "control", "dynamics"))
    cfg = fcfg.SimConfig(env=fcfg.EnvConfig(num_envs=64, seed=5, episode_max_steps=120))
    a = fw.World.create(cfg)
    b = fw.World.create(cfg)
    b._pipeline = compat.world_pipeline(b)
    rng = np.random.default_rng(0)
    # half the robots fly a fixed per-env velocity (they leave the box:
    # out of bounds = collision -> terminated), half follow the goal policy
    drift = rng.normal(0.0, 3.0, (a.num_envs, 3))
    drift[::2] = 0.0
    seen = {"autoreset": 0, "terminated": 0, "truncated": 0}
    for step in range(200):
        # identical fp32-representable inputs on both sides
        a.states = _round_states(fd, a.states)
        b.states = a.states.copy()
        np.testing.assert_array_equal(a.goals, b.goals)
        np.testing.assert_array_equal(a.pending_reset, b.pending_reset)
        goal = fb.goal_policy_commands(a, speed=2.0)
        v = np.where(drift != 0.0, drift, goal.velocity.v)
        cmds = _round_cmds(fc, fc.CommandBatch.all_velocity(fc.VelocityCommands(
            v=v, yaw_rate=rng.uniform(-1, 1, a.num_envs))))
        s_in = _planar(a.states)
        ra, rb = a.step(cmds), b.step(cmds)
        assert_parity(rb.observations.T, ra.observations.T, s_in, f"step {step}: observations")
        assert_parity(rb.reward[None], ra.reward[None], s_in, f"step {step}: reward")
        np.testing.assert_array_equal(rb.terminated, ra.terminated)
        np.testing.assert_array_equal(rb.truncated, ra.truncated)
        for k in ra.info:
            np.testing.assert_array_equal(rb.info[k], ra.info[k], err_msg=k)
        seen["autoreset"] += int(ra.info["autoreset"].sum())
        seen["terminated"] += int(ra.terminated.sum())
        seen["truncated"] += int(ra.truncated.sum())
    assert all(v > 0 for v in seen.values()), seen


@pytest.mark.parametrize("mode", ["attitude", "velocity"])
def test_bench_pipeline_step_swap(ref, compat, mode, monkeypatch):
    fb, fc, fd = ref["bench"], ref["control"], ref["dynamics"]
    calls = []

    def counted(*a, **k):
        calls.append(1)
        return compat.pipeline_step(*a, **k)
    monkeypatch.setattr(fb, "_pipeline_step", counted)
    rep = fb.bench_dynamics(num_envs=4096, steps=20, mode=mode, warmup=5)
    assert len(calls) == 25 and rep.steps_per_second > 0 and rep.num_envs == 4096
    monkeypatch.undo()
    # one step at the bar, then 100 steps within the drift bound
    params, gains, limits = fd.RobotParams(), fc.ControlGains(), fc.ControlLimits()
    states, cmds = fb.make_bench_batch(2048, 1, mode, params)
    states, cmds = _round_states(fd, states), _round_cmds(fc, cmds)
    one_ref = fb._pipeline_step(states, cmds, gains, params, limits, 0.01, 1)
    one = compat.pipeline_step(states, cmds, gains, params, limits, 0.01)
    assert type(one) is type(one_ref)
    assert_parity(_planar(one), _planar(one_ref), _planar(states), f"{mode}: one step")
    pure, floor, gpu = states, states, states
    for _ in range(100):
        pure = fb._pipeline_step(pure, cmds, gains, params, limits, 0.01, 1)
        floor = _round_states(fd, fb._pipeline_step(floor, cmds, gains, params, limits, 0.01, 1))
        gpu = compat.pipeline_step(gpu, cmds, gains, params, limits, 0.01)
    assert_drift(_planar(gpu), _planar(pure), _planar(floor), f"{mode}: 100 steps")


def test_control_and_step_batch_adapters_on_reference_golden(ref, compat, golden):
    fc, fd = ref["control"], ref["dynamics"]
    g = golden("mixed")
    s = g["state_in"]
    states = fd.RigidStateBatch(p=s[0:3].T, q=s[3:7].T, v=s[7:10].T, omega=s[10:13].T)
    att, vel = g["att_cmd"], g["vel_cmd"]
    cmds = fc.CommandBatch(mode=g["mode"],
                           attitude=fc.AttitudeCommands(roll=att[0], pitch=att[1],
                                                        yaw_rate=att[2], thrust=att[3]),
                           velocity=fc.VelocityCommands(v=vel[0:3].T, yaw_rate=vel[3]))
    params, gains = fd.RobotParams(), fc.ControlGains()
    wrench, flags = compat.control_batch(states, cmds, gains, params)
    assert type(wrench) is fd.WrenchBatch and type(flags) is fc.ControlFlags

    def spread(st, cols):
        with np.errstate(invalid="ignore"):
            _, info = O.step(st, g["mode"][cols], att[:, cols], vel[:, cols], O.Gains(),
                             O.Robot(), 0.01)
        return np.concatenate([info["thrust"][None], np.stack(info["moment"])])
    got = np.concatenate([wrench.thrust[None], wrench.moment.T])
    assert_parity(got, np.concatenate([g["thrust"][None], g["moment"]]), s, "compat wrench",
                  spread)
    np.testing.assert_array_equal(flags.gimbal_degenerate, g["gimbal"])
    np.testing.assert_array_equal(flags.degenerate_acceleration, g["degenerate"])
    ref_w = fd.WrenchBatch(thrust=f32(g["thrust"]), moment=f32(g["moment"].T))
    out, sf = compat.step_batch(states, params, ref_w, 0.01)
    exp, ef = fd.step_batch(states, params, ref_w, 0.01)
    assert type(out) is fd.RigidStateBatch and type(sf) is fd.StepFlags
    assert_parity(_planar(out), _planar(exp), s, "compat step_batch", band=2.0)
    np.testing.assert_array_equal(sf.nonfinite, ef.nonfinite)
    np.testing.assert_array_equal(sf.clamped, ef.clamped)
    # the fused pipeline on the same mixed batch (FS_MODE_MIXED through
    # fs_step_host_ex) against the reference's pair
    fused, ff = compat.pipeline(states, cmds, gains, params, fc.ControlLimits(), 0.01)
    exp2, ef2 = fd.step_batch(states, params, fc.control_batch(states, cmds, gains, params)[0],
                              0.01)
    assert_parity(_planar(fused), _planar(exp2), s, "compat fused pipeline",
                  lambda st, cols: O.step(st, g["mode"][cols], att[:, cols], vel[:, cols],
                                          O.Gains(), O.Robot(), 0.01)[0])
    np.testing.assert_array_equal(ff.nonfinite, ef2.nonfinite)
    with pytest.raises(ValueError, match="dt"):
        compat.pipeline(states, cmds, gains, params, None, 0.5)
    with pytest.raises(ValueError, match="command batch length"):
        compat.control_batch(states.slice(slice(0, 3)), cmds, gains, params)
