"""GPU tests of the RL bindings: the action clip +
denormalization fused into the World.step kernel (fs_vecenv_step).

* Golden replay: the reference flocksim_rl handle's recorded trajectory
  (tests/golden/vecenv_*.npz, make_golden_vecenv.py) is replayed step by step
  through VecEnvHandle.step with float32 and float64 actions, against the
  pinned oracle (world_oracle.commands_from_actions + world_step, itself
  pinned to the same fixture at 1e-12).  Bar: 1e-5 rel / 1e-6 abs on state,
  observation and reward; flags and counters exact.
* Transparency (test_bindings.py:108-127): with limits and actions chosen
  so the denormalized commands are exactly representable in fp32, stepping
  through the handle equals stepping the World with the host-denormalized
  CommandBatch BITWISE for 500 steps, in both modes.
* The reference's behavioural tests: clip (7.0 == 1.0), shape mismatch,
  NaN, closed handle, same seed -> same reset, reset == fresh world.
"""

import numpy as np
import pytest
import torch

from fs_parity import assert_parity
from oracle import flocksim_oracle as O
from oracle import world_oracle as WO

pytestmark = pytest.mark.gpu

BASE_YAML = """
version: 1
env:
  num_envs: {n}
  seed: {seed}
  control_mode: {mode}
  bounds: [10.0, 10.0, 5.0]
  episode_max_steps: 120
  wall_enabled: true
"""


@pytest.fixture(scope="module")
def fsr():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2305_16510_b200 as fs
    from paper_2305_16510_b200 import rl, world
    fs._native.load()
    return fs, rl, world


def write_cfg(tmp_path, n=4, seed=3, mode="velocity", extra=""):
    p = tmp_path / f"sim_{mode}_{n}_{seed}.yaml"
    p.write_text(BASE_YAML.format(n=n, seed=seed, mode=mode) + extra)
    return p


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


@pytest.mark.parametrize("mode", ["velocity", "attitude"])
@pytest.mark.parametrize("adtype", [torch.float32, torch.float64])
def test_golden_replay_matches_oracle(fsr, golden, tmp_path, mode, adtype):
    fs, rl, W = fsr
    g = golden(f"vecenv_{mode}")
    E = g["actions"].shape[1]
    h = rl.make(write_cfg(tmp_path, n=E, seed=int(g["seed"]), mode=mode))
    world = h.world
    env = WO.EnvCfg(bounds=g["bounds"], episode_max_steps=int(g["episode_max_steps"]))
    n_reset = 0
    for k in range(g["actions"].shape[0]):
        s_in, goal_in = _f32(g["state"][k]), _f32(g["goal"][k])
        world.load(state=s_in, goals=goal_in, pending=g["pending"][k], steps=g["steps"][k])
        acts = torch.tensor(g["actions"][k], dtype=adtype, device="cuda")
        obs, rew, term, trunc, info = h.step(acts)
        got_state = world.states.numpy()
        got_goal = world.goals.T.double().cpu().numpy()
        spawn = lambda idx: (got_state[0:3][:, idx], got_goal[:, idx])
        m, att, vel = WO.commands_from_actions(g["actions"][k], mode, O.Robot(), O.Limits())
        ref = WO.world_step(s_in, goal_in, g["pending"][k], g["steps"][k], m, att, vel,
                            O.Robot(), O.Gains(), O.Limits(), env, WO.RewardCfg(), spawn)
        assert_parity(got_state, ref["state"], s_in, f"{mode} state step {k}")
        assert_parity(obs.T.double().cpu().numpy(), ref["obs"], s_in, f"{mode} obs step {k}")
        assert_parity(rew.double().cpu().numpy(), ref["reward"], s_in, f"{mode} reward {k}")
        for key, got in (("terminated", term), ("truncated", trunc),
                         ("collision", info["collision"]), ("oob", info["out_of_bounds"]),
                         ("nonfinite", info["nonfinite"]), ("autoreset", info["autoreset"])):
            np.testing.assert_array_equal(got.cpu().numpy(), ref[key], err_msg=f"{key} {k}")
        np.testing.assert_array_equal(world.steps_in_episode.cpu().numpy(), ref["steps"])
        np.testing.assert_array_equal(world.pending_reset.cpu().numpy(), ref["pending"])
        n_reset += int(ref["autoreset"].sum())
    assert n_reset > 0


EXACT_LIMITS = """
robot: {thrust_max: 32.0}
limits: {max_tilt: 0.5, max_speed_cmd: 4.0, max_yaw_rate: 2.0}
"""


def _native_commands(fs, world, a):
    """test_bindings.py:46-57: the documented denormalization on the host."""
    a = np.clip(np.asarray(a, dtype=np.float64), -1.0, 1.0)
    lim = world.limits
    if world.env.control_mode == "attitude":
        return fs.CommandBatch.all_attitude(fs.AttitudeCommands(
            roll=a[:, 0] * lim.max_tilt, pitch=a[:, 1] * lim.max_tilt,
            yaw_rate=a[:, 2] * lim.max_yaw_rate,
            thrust=(a[:, 3] + 1.0) / 2.0 * world.robot.thrust_max))
    return fs.CommandBatch.all_velocity(fs.VelocityCommands(
        v=a[:, 0:3] * lim.max_speed_cmd, yaw_rate=a[:, 3] * lim.max_yaw_rate))


@pytest.mark.parametrize("mode,n,steps", [("velocity", 64, 500), ("attitude", 64, 500),
                                          ("velocity", 40000, 150), ("attitude", 40000, 150)])
def test_transparency_500_steps_bitwise(fsr, tmp_path, mode, n, steps):
    """n = 40000 takes the streaming World.step kernel (>= 2^15 envs)."""
    fs, rl, W = fsr
    from paper_2305_16510_b200.config import load_config
    path = write_cfg(tmp_path, n=n, seed=17, mode=mode, extra=EXACT_LIMITS)
    h = rl.make(path)
    native = W.World.create(load_config(path))
    rng = np.random.default_rng(88)
    n_reset = 0
    for k in range(steps):
        # multiples of 1/64 in [-1.25, 1.25]: every denormalized command is an
        # exact fp32 value, so both paths feed the controller identical numbers
        actions = np.round(rng.uniform(-1.25, 1.25, (n, 4)) * 64.0) / 64.0
        obs_b, rew_b, term_b, trunc_b, info_b = h.step(actions)
        res = native.step(_native_commands(fs, native, actions))
        assert torch.equal(obs_b, res.observations), f"step {k}"
        assert torch.equal(rew_b, res.reward)
        assert torch.equal(term_b, res.terminated)
        assert torch.equal(trunc_b, res.truncated)
        for key in res.info:
            assert torch.equal(info_b[key], res.info[key]), key
        n_reset += int(res.info["autoreset"].sum())
    assert n_reset > 0


def test_actions_clipped(fsr, tmp_path):
    fs, rl, W = fsr
    h1 = rl.make(write_cfg(tmp_path, seed=5))
    h2 = rl.make(write_cfg(tmp_path, seed=5))
    o1 = h1.step(np.full((4, 4), 7.0))[0]
    o2 = h2.step(np.ones((4, 4)))[0]
    assert torch.equal(o1, o2)
    o1 = h1.step(torch.full((4, 4), -np.inf, device="cuda"))[0]
    o2 = h2.step(-torch.ones((4, 4), device="cuda"))[0]
    assert torch.equal(o1, o2)


def test_float32_and_float64_actions_agree(fsr, tmp_path):
    fs, rl, W = fsr
    h1 = rl.make(write_cfg(tmp_path, n=257, seed=8, mode="attitude"))
    h2 = rl.make(write_cfg(tmp_path, n=257, seed=8, mode="attitude"))
    rng = np.random.default_rng(3)
    for _ in range(50):
        a = rng.uniform(-1.1, 1.1, (257, 4)).astype(np.float32)
        o1 = h1.step(torch.from_numpy(a).cuda())[0]
        o2 = h2.step(torch.from_numpy(a.astype(np.float64)).cuda())[0]
        assert torch.equal(o1, o2)


def test_strided_and_host_actions(fsr, tmp_path):
    """A column-sliced (non-contiguous) device tensor, a row-offset view and a
    host NumPy array all give the contiguous result."""
    fs, rl, W = fsr
    hs = [rl.make(write_cfg(tmp_path, n=33, seed=4)) for _ in range(4)]
    rng = np.random.default_rng(5)
    for _ in range(10):
        a = torch.tensor(rng.uniform(-1, 1, (34, 6)), dtype=torch.float32, device="cuda")
        ref = hs[0].step(a[1:, 1:5].contiguous())[0].clone()
        assert torch.equal(hs[1].step(a[1:, 1:5])[0], ref)
        flat = torch.zeros(33 * 4 + 2, dtype=torch.float32, device="cuda")
        b = flat[2:].view(33, 4)                                  # 8-B misaligned view
        b.copy_(a[1:, 1:5])
        assert b.data_ptr() % 16 == 8
        assert torch.equal(hs[2].step(b)[0], ref)
        assert torch.equal(hs[3].step(a[1:, 1:5].cpu().numpy())[0], ref)


def test_spaces_reset_and_errors(fsr, tmp_path):
    fs, rl, W = fsr
    from paper_2305_16510_b200.config import load_config
    h = rl.make(write_cfg(tmp_path, n=4))
    assert h.observation_space.shape == (4, 16) and h.action_space.shape == (4, 4)
    assert h.observations().shape == (4, 16)
    with pytest.raises(rl.ShapeMismatchError):
        h.step(np.zeros((3, 4)))
    a = torch.zeros((4, 4), device="cuda")
    a[1, 2] = float("nan")
    with pytest.raises(fs.InvalidCommandError):
        h.step(a)
    with pytest.raises(rl.CameraDisabledError):
        h.render_depth()
    # same seed -> same initial observations; reset == a fresh world's reset_all
    a1 = rl.make(write_cfg(tmp_path, seed=9))
    b1 = rl.make(write_cfg(tmp_path, seed=9))
    assert torch.equal(a1.observations(), b1.observations())
    path = write_cfg(tmp_path, n=2, seed=23)
    h2 = rl.make(path)
    native = W.World.create(load_config(path))
    assert torch.equal(h2.reset(), native.reset_all())
    h2.close()
    with pytest.raises(rl.ClosedHandleError):
        h2.step(np.zeros((2, 4)))


def test_graph_captured_action_steps(fsr, tmp_path):
    """step_async under CUDA-graph capture replays the same trajectory as
    eager steps (the RL rollout loop of bench.py's vecenv config)."""
    fs, rl, W = fsr
    n = 4096
    h1 = rl.make(write_cfg(tmp_path, n=n, seed=12, mode="velocity"))
    h2 = rl.make(write_cfg(tmp_path, n=n, seed=12, mode="velocity"))
    acts = torch.empty((n, 4), dtype=torch.float32, device="cuda")
    gen = torch.Generator(device="cuda").manual_seed(0)
    seq = [torch.rand((n, 4), generator=gen, device="cuda") * 2.4 - 1.2 for _ in range(20)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        acts.copy_(seq[0])
        h2.step_async(acts)                         # warm-up outside capture
    torch.cuda.synchronize()
    h2.reset()
    h1.reset()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        h2.step_async(acts, stream=s.cuda_stream)
    for k in range(20):
        h1.step(seq[k])
        acts.copy_(seq[k])
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(h1.observations(), h2.observations()), k
