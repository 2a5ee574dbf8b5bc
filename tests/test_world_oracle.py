"""Pin the free-space World.step oracle to the reference's own World
(tests/golden/world.npz from make_golden_world.py).  Re-spawn points are
taken from the recorded post-step state of the envs that reset (the
reference's NumPy Philox draws)."""

import numpy as np

from oracle import flocksim_oracle as O
from oracle import world_oracle as W


def test_world_step_matches_reference_golden(golden):
    g = golden("world")
    env = W.EnvCfg(bounds=g["bounds"], episode_max_steps=int(g["episode_max_steps"]),
                   dt=float(g["dt"]))
    E = g["state"].shape[2]
    ones = np.ones(E, np.uint8)
    zeros4 = np.zeros((4, E))
    for k in range(g["vel_cmd"].shape[0]):
        post = g["state"][k + 1]
        spawn = lambda idx: (post[0:3][:, idx], g["goal"][k + 1][:, idx])
        out = W.world_step(g["state"][k], g["goal"][k], g["pending"][k], g["steps"][k], ones,
                           zeros4, g["vel_cmd"][k], O.Robot(), O.Gains(), O.Limits(), env,
                           W.RewardCfg(), spawn)
        tol = dict(rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(out["state"], post, **tol)
        np.testing.assert_allclose(out["obs"], g["obs"][k], **tol)
        np.testing.assert_allclose(out["reward"], g["reward"][k], **tol)
        for key in ("terminated", "truncated", "collision", "oob", "nonfinite", "autoreset"):
            np.testing.assert_array_equal(out[key], g[key][k], err_msg=f"{key} step {k}")
        np.testing.assert_array_equal(out["steps"], g["steps"][k + 1])
        np.testing.assert_array_equal(out["pending"], g["pending"][k + 1])
    assert g["terminated"].sum() > 0 and g["truncated"].sum() > 0 and g["autoreset"].sum() > 0


def test_reward_known_answers():
    """test_world.py:154-172 restated: at goal and at rest -> c_success - c_step."""
    cfg = W.RewardCfg()
    z = np.zeros((3, 1))
    r = W.reward_goal_reaching(z, z, z, np.zeros(1, bool), cfg)
    assert r[0] == cfg.c_success - cfg.c_step
    crashed = W.reward_goal_reaching(z, z, z, np.ones(1, bool), cfg)
    assert crashed[0] == r[0] - cfg.c_crash


def _vecenv_env(g):
    return W.EnvCfg(bounds=g["bounds"], episode_max_steps=int(g["episode_max_steps"]))


def test_action_denormalization_matches_reference_bindings(golden):
    """commands_from_actions == the reference handle's own
    _commands_from_actions (vec_env.py:85-104), bitwise, in both modes."""
    for mode in ("velocity", "attitude"):
        g = golden(f"vecenv_{mode}")
        for k in range(g["actions"].shape[0]):
            m, att, vel = W.commands_from_actions(g["actions"][k], mode, O.Robot(), O.Limits())
            got = att if mode == "attitude" else vel
            assert np.array_equal(got, g["cmd"][k]), (mode, k)
        assert (np.abs(g["actions"]) > 1.0).any() and np.isinf(g["actions"]).any()


def test_vecenv_step_matches_reference_bindings(golden):
    """The oracle's action path (denormalization + World.step) reproduces
    the reference flocksim_rl handle's step outputs at 1e-12."""
    for mode in ("velocity", "attitude"):
        g = golden(f"vecenv_{mode}")
        env = _vecenv_env(g)
        for k in range(g["actions"].shape[0]):
            post = g["state"][k + 1]
            spawn = lambda idx: (post[0:3][:, idx], g["goal"][k + 1][:, idx])
            m, att, vel = W.commands_from_actions(g["actions"][k], mode, O.Robot(), O.Limits())
            out = W.world_step(g["state"][k], g["goal"][k], g["pending"][k], g["steps"][k], m,
                               att, vel, O.Robot(), O.Gains(), O.Limits(), env, W.RewardCfg(),
                               spawn)
            tol = dict(rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(out["state"], post, **tol)
            np.testing.assert_allclose(out["obs"], g["obs"][k], **tol)
            np.testing.assert_allclose(out["reward"], g["reward"][k], **tol)
            for key in ("terminated", "truncated", "collision", "oob", "nonfinite", "autoreset"):
                np.testing.assert_array_equal(out[key], g[key][k], err_msg=f"{mode} {key} {k}")
            np.testing.assert_array_equal(out["steps"], g["steps"][k + 1])
            np.testing.assert_array_equal(out["pending"], g["pending"][k + 1])
        assert g["autoreset"].sum() > 0
