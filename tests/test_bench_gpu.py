"""GPU tests of the benchmark-harness mirror, after the reference's own
(pkg/tests/test_bench.py:20-77): bookkeeping, the rate identity, checksum
reproducibility and worker invariance, timing that does not alter results,
both modes, JSON reports, render frame accounting -- plus parity of the
benchmark batch and of one benched step against the float64 oracle."""

import json

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2305_16510_b200 import bench
    return bench


def test_bookkeeping(B):
    r = B.bench_dynamics(num_envs=1, steps=100, warmup=5)
    assert r.num_envs == 1 and r.total_steps == 100
    assert r.steps_per_second > 0 and r.wall_seconds > 0
    assert r.dt == 0.01
    assert r.sim_to_real_ratio == pytest.approx(r.steps_per_second * 0.01)


@pytest.mark.parametrize("n", [32, 1 << 16])
def test_rate_identity(B, n):
    r = B.bench_dynamics(num_envs=n, steps=50, warmup=5)
    assert r.steps_per_second == pytest.approx(r.total_steps * r.num_envs / r.wall_seconds)


@pytest.mark.parametrize("n", [64, 1 << 16])
def test_checksum_reproducible(B, n):
    a = B.bench_dynamics(num_envs=n, steps=40, seed=3, warmup=10)
    b = B.bench_dynamics(num_envs=n, steps=40, seed=3, warmup=10)
    assert a.checksum == b.checksum
    c = B.bench_dynamics(num_envs=n, steps=40, seed=4, warmup=10)
    assert a.checksum != c.checksum


def test_checksum_worker_invariant(B):
    a = B.bench_dynamics(num_envs=128, steps=30, seed=1, warmup=5, workers=1)
    b = B.bench_dynamics(num_envs=128, steps=30, seed=1, warmup=5, workers=4)
    assert a.checksum == b.checksum


@pytest.mark.parametrize("n", [64, 1 << 16])
def test_timing_does_not_alter_results(B, n):
    """The same pipeline without the harness: fused_step launches, one per step."""
    from paper_2305_16510_b200.control import ControlGains, ControlLimits
    from paper_2305_16510_b200.dynamics import RobotParams
    params, gains, limits = RobotParams(), ControlGains(), ControlLimits()
    states, cmds = B.make_bench_batch(n, 7, "velocity", params)
    for _ in range(15 + 25):
        states = B._pipeline_step(states, cmds, gains, params, limits, 0.01)
    r = B.bench_dynamics(num_envs=n, steps=25, mode="velocity", seed=7, warmup=15)
    assert r.checksum == B.state_checksum(states)


def test_both_modes_run(B):
    for mode in ("attitude", "velocity"):
        assert B.bench_dynamics(num_envs=8, steps=10, mode=mode, warmup=2).mode == mode


def test_json_report(B, tmp_path):
    r = B.bench_dynamics(num_envs=4, steps=10, warmup=2)
    path = tmp_path / "report.json"
    r.write_json(path)
    data = json.loads(path.read_text())
    assert data["num_envs"] == 4 and data["checksum"] == r.checksum


@pytest.mark.parametrize("mode", ["attitude", "velocity"])
def test_bench_batch_and_step_match_oracle(B, mode):
    """make_bench_batch draws the reference's NumPy sequence (bench.py:123-143);
    one benched step matches the float64 oracle on the fp32-rounded batch."""
    from oracle import flocksim_oracle as O
    from paper_2305_16510_b200.dynamics import RobotParams
    n = 4096
    states, cmds = B.make_bench_batch(n, 11, mode, RobotParams())
    rng = np.random.default_rng(11)
    p = rng.uniform(-1.0, 1.0, (n, 3))
    rot = rng.uniform(-0.1, 0.1, (n, 3))
    v = rng.uniform(-0.2, 0.2, (n, 3))
    w = rng.uniform(-0.1, 0.1, (n, 3))
    q = np.stack(O.exp_so3(rot[:, 0], rot[:, 1], rot[:, 2]))
    s = states.buf[:, :n].double().cpu().numpy()
    assert np.array_equal(s[0:3], p.T.astype(np.float32))
    assert np.array_equal(s[7:10], v.T.astype(np.float32))
    assert np.array_equal(s[10:13], w.T.astype(np.float32))
    np.testing.assert_allclose(s[3:7], q, rtol=0, atol=1e-7)
    r = B.bench_dynamics(num_envs=n, steps=1, mode=mode, seed=11, warmup=0)
    assert r.total_steps == 1
    out = B._pipeline_step(states, cmds, *_defaults(), 0.01)
    got = out.buf[:, :n].double().cpu().numpy()
    m = np.full(n, 0 if mode == "attitude" else 1, dtype=np.uint8)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    att = f32(np.stack([np.full(n, 0.05), np.full(n, -0.05), np.full(n, 0.2), np.full(n, 9.81)]))
    vel = f32(np.stack([np.full(n, 0.5), np.full(n, 0.3), np.full(n, 0.1), np.full(n, 0.2)]))
    ref, _ = O.step(s, m, att, vel, O.Gains(), O.Robot(), 0.01)
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-6)
    assert B.state_checksum(out) == r.checksum


def _defaults():
    from paper_2305_16510_b200.control import ControlGains, ControlLimits
    from paper_2305_16510_b200.dynamics import RobotParams
    return ControlGains(), RobotParams(), ControlLimits()


def test_render_frame_accounting(B):
    from paper_2305_16510_b200.camera import CameraConfig
    r = B.bench_render(num_envs=4, frames=10, cam_cfg=CameraConfig(width=48, height=32,
                                                                      hfov=1.3), seed=2)
    assert r.total_steps * r.num_envs == 40
    assert r.frames_per_second > 0 and r.resolution == (48, 32)
    again = B.bench_render(num_envs=4, frames=1, cam_cfg=CameraConfig(width=48, height=32,
                                                                         hfov=1.3), seed=2)
    assert again.checksum == r.checksum
