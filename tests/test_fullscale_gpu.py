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


def _pos_step(s, pos, dt=0.01, frame=None, mass=None, jdiag=None, rotor_dynamics=False):
    """One extension-oracle position step (parity unpinned)."""
    f, m, _ = O.position_control(s, pos[0:3], pos[3], O.Gains(), O.Robot(), O.Limits(),
                                 mass=mass, inertia_diag=jdiag)
    if frame is not None:
        _, fr, mr = O.allocate(f, m, frame)
        if rotor_dynamics:
            f, m = fr, mr
    out, _, _ = O.integrate(s, f, m, O.Robot(), dt, mass=mass, inertia_diag=jdiag)
    return out


def test_cfg3_full_size_persistent(fs):
    """Config 3 per GPU (2^21, position, Bernoulli(0.01) re-spawns, statistics)
    as one persistent fs_step_many launch of 50 steps: the sample count equals
    n K minus the twin's re-spawn count (every draw of every vehicle and step
    checked), vehicles re-spawned at the last step hold the twin's spawn, and
    never re-spawned vehicles stay within the drift bound of the extension
    oracle."""
    from paper_2305_16510_b200.fleet import Fleet
    n, k, seed, p = 1 << 21, 50, 5, 0.01
    f = Fleet(n, mode="position", seed=seed, reset_prob=p, want_stats=True)
    idx = _sample(n, k=2048, seed=2).to(f.device)
    s0 = f.state[:, idx].double().cpu().numpy()
    c0 = f.cmd[:, idx].double().cpu().numpy()
    f.rollout(k, persistent=True)
    torch.cuda.synchronize()
    tot = f.stats_local().cpu().numpy()
    gid = np.arange(n, dtype=np.uint64)
    masks = [R.reset_mask(seed, gid, step, p) for step in range(k)]
    assert int(tot[2]) == n * k - sum(int(m.sum()) for m in masks)
    assert int(tot[1]) == 0
    # re-spawned at the last step: the twin's spawn (uniform draws bit-exact)
    last = np.nonzero(masks[-1])[0][:512]
    st, _ = R.spawn(seed, last.astype(np.uint64), k - 1, "position")
    got_last = f.state[:, torch.from_numpy(last).to(f.device)].double().cpu().numpy()
    assert np.array_equal(got_last[0:3], st[0:3])
    # never re-spawned: K-step drift against the float64 extension oracle
    ever = np.zeros(n, bool)
    for m in masks:
        ever |= m
    keep = ~ever[idx.cpu().numpy()]
    assert keep.sum() > 1000
    got = f.state[:, idx].double().cpu().numpy()[:, keep]
    ref, floor = s0[:, keep].copy(), s0[:, keep].copy()
    pos = c0[:, keep]
    for _ in range(k):
        ref = _pos_step(ref, pos)
        floor = _pos_step(floor, pos).astype(np.float32).astype(np.float64)
    assert_drift(got, ref, floor, f"cfg3 position x{k} at n={n}")


def test_cfg4_full_size_persistent(fs):
    """Config 4 (2^23: X-quads then hexarotors, per-vehicle mass / inertia,
    position control, realized rotor wrench, dt = 0.005, 500 steps) as one
    persistent launch: a subsample (both airframes, the split) stays within
    the drift bound of the extension oracle; rotor thrusts stay in bounds."""
    from paper_2305_16510_b200.allocation import HEXAROTOR, QUAD_X
    from paper_2305_16510_b200.fleet import Fleet
    n, k = 1 << 23, 500
    f = Fleet(n, mode="position", dt=0.005, seed=9, hetero=True,
              airframes=(QUAD_X, HEXAROTOR), airframe_split=n // 2, rotor_dynamics=True)
    idx = _sample(n, k=2048, seed=3).to(f.device)
    s0 = f.state[:, idx].double().cpu().numpy()
    c0 = f.cmd[:, idx].double().cpu().numpy()
    vp = f.vparams[:, idx].double().cpu().numpy()
    f.rollout(k, persistent=True)
    torch.cuda.synchronize()
    got = f.state[:, idx].double().cpu().numpy()
    rot = f.rotors[:, idx].double().cpu().numpy()
    hexa = idx.cpu().numpy() >= n // 2
    for sel, frame, nr, rmax in ((~hexa, O.QUAD_X, 4, QUAD_X.rotor_max),
                                 (hexa, O.HEX, 6, HEXAROTOR.rotor_max)):
        ref, floor = s0[:, sel].copy(), s0[:, sel].copy()
        kw = dict(dt=0.005, frame=frame, mass=vp[0, sel], jdiag=vp[1:4, sel],
                  rotor_dynamics=True)
        for _ in range(k):
            ref = _pos_step(ref, c0[:, sel], **kw)
            floor = _pos_step(floor, c0[:, sel], **kw).astype(np.float32).astype(np.float64)
        assert_drift(got[:, sel], ref, floor, f"cfg4 {nr}-rotor x{k} at n={n}")
        assert np.all((rot[:nr, sel] >= 0.0) & (rot[:nr, sel] <= rmax * (1 + 1e-6)))
        assert np.all(rot[nr:, sel] == 0.0)
    del f
    torch.cuda.empty_cache()
