"""Full-size GPU parity (BASELINE sizes) through size-independent checks.

The oracle is elementwise, so a seeded subsample of vehicles (including
every 1/2/4/8-GPU shard boundary) is exact to check.
"""

import numpy as np
import pytest
import torch

from fs_parity import assert_drift, assert_parity
from oracle import flocksim_oracle as O
from oracle import rng_twin as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fs():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2305_16510_b200 as fs
    fs._native.load()
    return fs


def _sample(n, k=4096, seed=0):
    rng = np.random.default_rng(seed)
    bounds = [(n * r) // w for w in (2, 4, 8) for r in range(1, w)]
    edges = np.unique(np.clip(np.concatenate([[0, 1, n - 1], bounds, np.array(bounds) - 1]), 0, n - 1))
    idx = np.unique(np.concatenate([edges, rng.choice(n, k, replace=False)]))
    return torch.from_numpy(idx).long()


def test_one_step_at_2pow24_velocity(fs):
    """2^24 vehicles (config 3's total size; 872 MB of state) in one launch."""
    from paper_2305_16510_b200.fleet import Fleet
    n = 1 << 24
    f = Fleet(n, mode="velocity", seed=42)
    idx = _sample(n).to(f.device)
    s0 = f.state[:, idx].double().cpu().numpy()
    c0 = f.cmd[:, idx].double().cpu().numpy()
    # the sampled inputs are the device RNG's spawns: bit-exact uniforms vs the twin
    st, _ = R.spawn(42, idx.cpu().numpy().astype(np.uint64), R.INIT_STEP, "velocity")
    assert np.array_equal(s0[0:3], st[0:3])
    f.step()
    got = f.state[:, idx].double().cpu().numpy()
    k = idx.numel()
    ref, _ = O.step(s0, np.ones(k, np.uint8), np.zeros((4, k)), c0, O.Gains(), O.Robot(), 0.01)
    assert_parity(got, ref, s0, "2^24 velocity step (subsample)")
    del f
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode,steps", [("velocity", 1000), ("attitude", 100)])
def test_rollout_drift_at_full_size(fs, mode, steps):
    """cfg2 (2^22, 1000 velocity steps) and cfg1 (2^20, 100 attitude steps):
    the subsample's K-step drift against the pure float64 oracle stays within
    16x the fp32-storage floor per component group + 1e-5."""
    from paper_2305_16510_b200.fleet import Fleet
    n = (1 << 22) if mode == "velocity" else (1 << 20)
    f = Fleet(n, mode=mode, seed=7)
    idx = _sample(n, k=2048, seed=1).to(f.device)
    s = f.state[:, idx].double().cpu().numpy()
    c = f.cmd[:, idx].double().cpu().numpy()
    k = idx.numel()
    m = np.full(k, 1 if mode == "velocity" else 0, np.uint8)
    att, vel = (np.zeros((4, k)), c) if mode == "velocity" else (c, np.zeros((4, k)))
    g = f.capture(steps)
    g.replay()
    torch.cuda.synchronize()
    got = f.state[:, idx].double().cpu().numpy()
    ref, floor = s.copy(), s.copy()
    for _ in range(steps):
        ref, _ = O.step(ref, m, att, vel, O.Gains(), O.Robot(), 0.01)
        floor, _ = O.step(floor, m, att, vel, O.Gains(), O.Robot(), 0.01)
        floor = floor.astype(np.float32).astype(np.float64)
    assert_drift(got, ref, floor, f"{mode} x{steps} at n={n}")
    assert np.isfinite(got).all()
