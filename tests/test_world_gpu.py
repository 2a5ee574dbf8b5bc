"""GPU tests of the device World.

The device World is compared with the pinned float64 world oracle
(oracle/world_oracle.py, itself pinned to the reference World in
tests/test_world_oracle.py) on IDENTICAL fp32 inputs: the reference's
recorded trajectory (tests/golden/world.npz) is replayed step by step, the
device re-spawn points (its own Philox stream) are fed to the oracle for
the envs that auto-reset.  Bar: 1e-5 rel / 1e-6 abs on state, observation
and reward; flags and counters exact.
"""

import numpy as np
import pytest
import torch

from fs_parity import assert_parity
from oracle import flocksim_oracle as O
from oracle import rng_twin as R
from oracle import world_oracle as WO

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fsw():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2305_16510_b200 as fs
    from paper_2305_16510_b200 import world
    fs._native.load()
    return fs, world


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def test_creation_placement_matches_twin(fsw):
    fs, W = fsw
    cfg = W.SimConfig(env=W.EnvConfig(num_envs=5000, seed=11))
    world = W.World.create(cfg)
    gid = np.arange(5000, dtype=np.uint64)
    e = cfg.env
    sp, ok1 = R.world_place(11, gid, 0, False, e.spawn_min, e.spawn_max, e.bounds, 0.2)
    gl, ok2 = R.world_place(11, gid, 0, True, e.goal_min, e.goal_max, e.bounds, 0.2)
    assert ok1.all() and ok2.all()
    st = world.states.numpy()
    assert np.array_equal(st[0:3], sp)
    assert np.array_equal(world.goals.T.double().cpu().numpy(), gl)
    assert np.array_equal(st[3], np.ones(5000)) and not st[4:].any() and not st[7:].any()
    obs = world.observations().T.double().cpu().numpy()
    np.testing.assert_allclose(obs, WO.observations(st, gl), rtol=1e-6, atol=1e-6)


def test_world_step_matches_oracle_on_reference_trajectory(fsw, golden):
    fs, W = fsw
    g = golden("world")
    E = g["state"].shape[2]
    env = W.EnvConfig(num_envs=E, seed=5, episode_max_steps=int(g["episode_max_steps"]))
    world = W.World.create(W.SimConfig(env=env))
    ocfg = WO.EnvCfg(bounds=g["bounds"], episode_max_steps=int(g["episode_max_steps"]))
    ones, zeros4 = np.ones(E, np.uint8), np.zeros((4, E))
    n_reset = 0
    for k in range(g["vel_cmd"].shape[0]):
        s_in, goal_in = _f32(g["state"][k]), _f32(g["goal"][k])
        world.load(state=s_in, goals=goal_in, pending=g["pending"][k], steps=g["steps"][k])
        vel = _f32(g["vel_cmd"][k])
        cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=vel[0:3].T, yaw_rate=vel[3],
                                                                validate=False))
        res = world.step(cmds)
        got_state = world.states.numpy()
        got_goal = world.goals.T.double().cpu().numpy()
        spawn = lambda idx: (got_state[0:3][:, idx], got_goal[:, idx])
        ref = WO.world_step(s_in, goal_in, g["pending"][k], g["steps"][k], ones, zeros4, vel,
                            O.Robot(), O.Gains(), O.Limits(), ocfg, WO.RewardCfg(), spawn)
        assert_parity(got_state, ref["state"], s_in, f"world state step {k}")
        assert_parity(res.observations.T.double().cpu().numpy(), ref["obs"], s_in,
                      f"world obs step {k}")
        assert_parity(res.reward.double().cpu().numpy(), ref["reward"], s_in,
                      f"world reward step {k}")
        for key, got in (("terminated", res.terminated), ("truncated", res.truncated),
                         ("collision", res.info["collision"]), ("oob", res.info["out_of_bounds"]),
                         ("nonfinite", res.info["nonfinite"]),
                         ("autoreset", res.info["autoreset"])):
            np.testing.assert_array_equal(got.cpu().numpy(), ref[key], err_msg=f"{key} {k}")
        np.testing.assert_array_equal(world.steps_in_episode.cpu().numpy(), ref["steps"])
        np.testing.assert_array_equal(world.pending_reset.cpu().numpy(), ref["pending"])
        n_reset += int(ref["autoreset"].sum())
    assert n_reset > 0


def test_reset_env_isolation_and_counter(fsw):
    fs, W = fsw
    world = W.World.create(W.SimConfig(env=W.EnvConfig(num_envs=6, seed=31)))
    before = world.states.numpy().copy()
    goals_before = world.goals.cpu().numpy().copy()
    world.reset_env(3)
    after = world.states.numpy()
    for e in range(6):
        if e != 3:
            assert np.array_equal(before[:, e], after[:, e])
            assert np.array_equal(goals_before[e], world.goals.cpu().numpy()[e])
    assert world.reset_counter.cpu().tolist() == [0, 0, 0, 1, 0, 0]
    e = world.env
    sp, _ = R.world_place(31, np.array([3], np.uint64), 1, False, e.spawn_min, e.spawn_max,
                          e.bounds, 0.2)
    assert np.array_equal(after[0:3, 3:4], sp)


def test_goal_reaching_velocity_policy(fsw):
    """test_world.py:320-345 / acceptance criterion 'end-to-end demo': a 3 m
    goal is reached within 6 s by a velocity policy toward the goal."""
    fs, W = fsw
    env = W.EnvConfig(num_envs=1, seed=0, bounds=[8.0, 8.0, 4.0],
                      spawn_min=[0.25, 0.5, 0.5], spawn_max=[0.25, 0.5, 0.5],
                      goal_min=[0.625, 0.5, 0.5], goal_max=[0.625, 0.5, 0.5])
    world = W.World.create(W.SimConfig(env=env))
    d0 = float(torch.linalg.norm(world.goals[0] - world.states.p[0]))
    assert abs(d0 - 3.0) < 1e-5
    reached = None
    for k in range(600):
        obs = world.observations()
        gv = obs[:, 13:16]
        dist = torch.linalg.norm(gv, dim=1)
        if float(dist[0]) < 0.2:
            reached = k * 0.01
            break
        scale = torch.clamp(dist, max=1.0) / torch.clamp(dist, min=1e-9)
        cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=gv * scale[:, None],
                                                                yaw_rate=torch.zeros(1, device=gv.device),
                                                                validate=False))
        world.step(cmds)
    assert reached is not None and reached <= 6.0


def test_step_length_check(fsw):
    fs, W = fsw
    world = W.World.create(W.SimConfig(env=W.EnvConfig(num_envs=4)))
    cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=np.zeros((3, 3)),
                                                            yaw_rate=np.zeros(3)))
    with pytest.raises(ValueError, match="expected 4 commands"):
        world.step(cmds)


@pytest.mark.parametrize("mode", ["velocity", "attitude"])
def test_streaming_kernel_matches_thread_kernel(fsw, mode):
    """The streaming World.step (TMA ring, batches >= 2^15) and the
    thread-per-env kernel run the same per-env code (world_env_step): forced
    on two identical worlds of 2^15 + 37 envs (a partial last tile whose
    counter / flag bytes are read from global memory) with commands violent
    enough to crash, auto-reset and truncate, they agree bit for bit."""
    fs, W = fsw
    from paper_2305_16510_b200 import _native as N
    n = (1 << 15) + 37
    env = W.EnvConfig(num_envs=n, seed=4, episode_max_steps=40, control_mode=mode)
    a, b = W.World.create(W.SimConfig(env=env)), W.World.create(W.SimConfig(env=env))
    rng = np.random.default_rng(12)
    resets = 0
    try:
        for k in range(120):
            if mode == "velocity":
                v = np.asarray(rng.normal(0.0, 4.0, (n, 3)), np.float32)
                cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(
                    v=v, yaw_rate=np.asarray(rng.uniform(-1, 1, n), np.float32), validate=False))
            else:
                cmds = fs.CommandBatch.all_attitude(fs.AttitudeCommands(
                    roll=np.asarray(rng.uniform(-0.5, 0.5, n), np.float32),
                    pitch=np.asarray(rng.uniform(-0.5, 0.5, n), np.float32),
                    yaw_rate=np.asarray(rng.uniform(-1, 1, n), np.float32),
                    thrust=np.asarray(rng.uniform(5, 15, n), np.float32), validate=False))
            N.set_tuning(N.FS_TUNE_WORLD_KERNEL, 1)
            ra = a.step(cmds)
            N.set_tuning(N.FS_TUNE_WORLD_KERNEL, 2)
            rb = b.step(cmds)
            assert torch.equal(a.states.buf[:, :n], b.states.buf[:, :n]), f"state {k}"
            assert torch.equal(ra.observations, rb.observations), f"obs {k}"
            assert torch.equal(ra.reward, rb.reward), f"reward {k}"
            for key in ra.info:
                assert torch.equal(ra.info[key], rb.info[key]), f"{key} {k}"
            assert torch.equal(a.steps_in_episode, b.steps_in_episode)
            assert torch.equal(a.goals, b.goals) and torch.equal(a.reset_counter, b.reset_counter)
            resets += int(ra.info["autoreset"].sum())
    finally:
        N.set_tuning(N.FS_TUNE_WORLD_KERNEL, 0)
    assert resets > 0
