"""GPU tests of the fleet engine and the EXTENSION rows (BASELINE configs 0,
3, 4): position controller, rotor allocation, heterogeneous fleets, the
device RNG against its CPU twin, per-step re-spawns, episode statistics,
shard invariance, fused rollouts and CUDA-graph replay.

Parity of the extensions is against the builder's float64 extension oracle
(oracle/flocksim_oracle.py: position_control, allocate, integrate with
per-vehicle parameters) -- "parity unpinned" by the reference, which has no
such code -- at the same 1e-5 rel / 1e-6 abs bar.
"""

import numpy as np
import pytest
import torch

from fs_parity import assert_parity
from oracle import flocksim_oracle as O
from oracle import rng_twin as R
from oracle.workload import config_batch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fs():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2305_16510_b200 as fs
    fs._native.load()
    return fs


def _fleet(fs, n, mode, **kw):
    from paper_2305_16510_b200.fleet import Fleet
    return Fleet(n, mode=mode, **kw)


def _load(fleet, s, cmd):
    fleet.state[:, :fleet.n].copy_(torch.from_numpy(np.asarray(s, np.float32)))
    fleet.cmd[:cmd.shape[0], :fleet.n].copy_(torch.from_numpy(np.asarray(cmd, np.float32)))


def _np(t, n):
    return t[:, :n].double().cpu().numpy()


# --- device RNG vs CPU twin ---------------------------------------------------

@pytest.mark.parametrize("mode", ["attitude", "velocity", "position", "mixed"])
def test_init_fleet_matches_cpu_twin(fs, mode):
    n, first, seed = 5000, 123456789, 77
    f = _fleet(fs, n, mode, seed=seed, first_id=first)
    gid = np.arange(first, first + n, dtype=np.uint64)
    st, cmd = R.spawn(seed, gid, R.INIT_STEP, mode)
    got = _np(f.state, n)
    # uniforms are bit-exact; transcendental draws (q, normals) within 2e-6
    assert np.array_equal(got[0:3], st[0:3])
    np.testing.assert_allclose(got[3:], st[3:], rtol=2e-6, atol=2e-6)
    gc = _np(f.cmd, n)
    np.testing.assert_allclose(gc, cmd, rtol=2e-6, atol=2e-6)
    if mode in ("attitude", "position"):
        exact = [0, 1, 2, 3] if mode == "position" else [0, 1, 2]
        assert np.array_equal(gc[exact], cmd[exact])


def test_reset_mask_and_respawn_bit_exact(fs):
    n, seed, p = 20000, 5, 0.05
    f = _fleet(fs, n, "position", seed=seed, reset_prob=p, want_flags=True)
    for k in range(3):
        before = _np(f.state, n)
        f.step()
        flags = f.flags[:n].cpu().numpy()
        gid = np.arange(n, dtype=np.uint64)
        mask = R.reset_mask(seed, gid, k, p)
        assert np.array_equal((flags & fs._native.FS_FLAG_RESET) != 0, mask)
        st, cmd = R.spawn(seed, gid[mask], k, "position")
        got = _np(f.state, n)[:, mask]
        assert np.array_equal(got[0:3], st[0:3])
        np.testing.assert_allclose(got[3:], st[3:], rtol=2e-6, atol=2e-6)
        assert np.array_equal(_np(f.cmd, n)[:, mask], cmd)
        assert not np.array_equal(before[:, ~mask], _np(f.state, n)[:, ~mask])


@pytest.mark.parametrize("n,p,want_flags", [
    (1 << 17, 0.05, False),      # stream kernel, statistics + re-spawns (cfg3 path)
    (1 << 17, 0.05, True),       # stream kernel with every optional output
    (1 << 20, 0.5, False),       # > 2048 re-spawns per CTA: the shared list overflows
])
def test_stream_path_respawns_bit_exact(fs, n, p, want_flags):
    """The stream kernel queues re-spawns in a per-CTA shared list and draws
    them after its last tile: re-spawned vehicles equal the CPU twin's draws;
    every other vehicle is the oracle's position step at the parity bar (and
    agrees with the kernel variant without re-spawns to fp32 rounding: the
    FEAT instantiations may contract FMAs differently)."""
    seed = 9
    f = _fleet(fs, n, "position", seed=seed, reset_prob=p, want_flags=want_flags,
               want_stats=True)
    g = _fleet(fs, n, "position", seed=seed)
    gid = np.arange(n, dtype=np.uint64)
    for k in range(2):
        g.state.copy_(f.state)
        g.cmd.copy_(f.cmd)
        s_in, pos_in = _np(f.state, n), _np(f.cmd, n)
        f.step()
        g.step()
        mask = R.reset_mask(seed, gid, k, p)
        if want_flags:
            flags = f.flags[:n].cpu().numpy()
            assert np.array_equal((flags & fs._native.FS_FLAG_RESET) != 0, mask)
        st, cmd = R.spawn(seed, gid[mask], k, "position")
        got = _np(f.state, n)
        assert np.array_equal(got[0:3, mask], st[0:3])
        np.testing.assert_allclose(got[3:, mask], st[3:], rtol=2e-6, atol=2e-6)
        assert np.array_equal(_np(f.cmd, n)[:, mask], cmd)
        keep = ~mask
        _, _, _, out = _pos_oracle(s_in[:, keep], pos_in[:, keep])
        assert_parity(got[:, keep], out, s_in[:, keep], f"stream re-spawn step {k}", band=2.0)
        np.testing.assert_allclose(got[:, keep], _np(g.state, n)[:, keep], rtol=1e-6, atol=1e-6)
        assert np.array_equal(_np(f.cmd, n)[:, keep], pos_in[:, keep])
    stats = f.stats_local()
    assert int(stats[2]) == 2 * n - int(R.reset_mask(seed, gid, 0, p).sum()) - \
        int(R.reset_mask(seed, gid, 1, p).sum())


# --- position controller / allocation (configs 0, 3) --------------------------

def _pos_oracle(s, pos, frame=None, mass=None, jdiag=None, integrate=True, rotor_dynamics=False):
    f, m, _ = O.position_control(s, pos[0:3], pos[3], O.Gains(), O.Robot(), O.Limits(),
                                 mass=mass, inertia_diag=jdiag)
    rot = None
    if frame is not None:
        rot, fr, mr = O.allocate(f, m, frame)
        if rotor_dynamics:
            f, m = fr, mr
    out = None
    if integrate:
        out, _, _ = O.integrate(s, f, m, O.Robot(), 0.01, mass=mass, inertia_diag=jdiag)
    return f, m, rot, out


def test_position_control_and_step_parity(fs):
    n = 1 << 16
    s, _, _, _, pos = config_batch("position", n, seed=3)
    f = _fleet(fs, n, "position", want_wrench=True)
    _load(f, s, pos)
    f.control()
    thr, mom, _, out = _pos_oracle(s, pos)
    assert_parity(_np(f.wrench, n), np.concatenate([thr[None], np.stack(mom)]), s,
                  "position: wrench", band=2.0)
    f.step()
    assert_parity(_np(f.state, n), out, s, "position: state", band=2.0)


def test_config0_quad_rotor_thrusts(fs):
    """BASELINE config 0: position controller, one step, 1024 quads, X-quad
    allocation -> 4 rotor thrusts."""
    from paper_2305_16510_b200.allocation import QUAD_X
    n = 1024
    s, _, _, _, pos = config_batch("position", n, seed=0)
    f = _fleet(fs, n, "position", airframes=(QUAD_X, QUAD_X))
    _load(f, s, pos)
    f.control()
    _, _, rot, _ = _pos_oracle(s, pos, frame=O.QUAD_X, integrate=False)
    got = _np(f.rotors, n)
    assert np.all(got[4:] == 0.0)
    assert_parity(got[:4], rot, s, "cfg0 rotor thrusts", band=2.0)
    assert np.all((got[:4] >= 0.0) & (got[:4] <= QUAD_X.rotor_max))


def test_config4_heterogeneous_fleet_step(fs):
    """BASELINE config 4 in miniature: half X-quads, half hexarotors,
    per-vehicle mass/inertia, position control, realized rotor wrench."""
    from paper_2305_16510_b200.allocation import HEXAROTOR, QUAD_X
    n = 4096
    f = _fleet(fs, n, "position", seed=11, hetero=True, airframes=(QUAD_X, HEXAROTOR),
               airframe_split=n // 2, rotor_dynamics=True)
    s = _np(f.state, n)
    pos = _np(f.cmd, n)
    vp = _np(f.vparams, n)
    np.testing.assert_allclose(vp, R.spawn_vparams(11, np.arange(n, dtype=np.uint64)),
                               rtol=1e-7)
    assert np.all((vp[0] >= 0.8 - 1e-6) & (vp[0] <= 1.2 + 1e-6))
    f.step()
    got_s, got_r = _np(f.state, n), _np(f.rotors, n)
    for lo, hi, frame, nr in ((0, n // 2, O.QUAD_X, 4), (n // 2, n, O.HEX, 6)):
        sl = slice(lo, hi)
        _, _, rot, out = _pos_oracle(s[:, sl], pos[:, sl], frame=frame, mass=vp[0, sl],
                                     jdiag=vp[1:4, sl], rotor_dynamics=True)
        assert_parity(got_r[:nr, sl], rot, s[:, sl], f"cfg4 rotors {frame.angles_deg}", band=2.0)
        assert_parity(got_s[:, sl], out, s[:, sl], f"cfg4 state {nr}-rotor", band=2.0)


# --- fleet engine properties ---------------------------------------------------

def test_shard_invariance_bitwise(fs):
    """1 shard vs 4 shards (first_id offsets, the dynamics.py:269 bounds):
    bitwise-identical vehicles and integer statistics."""
    from paper_2305_16510_b200.parallel import shard_bounds
    n, seed, k = 10000, 3, 25
    whole = _fleet(fs, n, "position", seed=seed, reset_prob=0.02, want_stats=True)
    for _ in range(k):
        whole.step()
    ref_state = _np(whole.state, n)
    ref_stats = whole.stats_local().cpu()
    parts, tot = [], torch.zeros(3, dtype=torch.int64)
    for r in range(4):
        lo, hi = shard_bounds(n, 4, r)
        f = _fleet(fs, hi - lo, "position", seed=seed, first_id=lo, reset_prob=0.02,
                   want_stats=True)
        for _ in range(k):
            f.step()
        parts.append(_np(f.state, hi - lo))
        tot += f.stats_local().cpu()
    assert np.array_equal(np.concatenate(parts, axis=1), ref_state)
    assert torch.equal(tot, ref_stats)
    assert int(ref_stats[2]) > 0


def test_stats_match_host_recomputation(fs):
    n, seed = 8192, 9
    f = _fleet(fs, n, "position", seed=seed, want_stats=True)
    f.step()
    st = _np(f.state, n).astype(np.float32)
    cmd = _np(f.cmd, n).astype(np.float32)
    err = np.sqrt(((st[0:3] - cmd[0:3]) ** 2).sum(axis=0, dtype=np.float32))
    tot = f.stats_local().cpu().numpy()
    assert tot[2] == n and tot[1] == 0
    np.testing.assert_allclose(tot[0] / 2.0 ** 20, err.astype(np.float64).sum(), rtol=1e-6)


@pytest.mark.parametrize("mode", ["attitude", "velocity", "position"])
def test_fused_rollout_matches_per_step_launches(fs, mode):
    n, k = 20000, 50
    a = _fleet(fs, n, mode, seed=4)
    b = _fleet(fs, n, mode, seed=4)
    for _ in range(k):
        a.step()
    b.rollout(k, fused=True)
    np.testing.assert_allclose(_np(b.state, n), _np(a.state, n), rtol=1e-5, atol=2e-5)


def test_cuda_graph_replay_matches_eager(fs):
    n, k = 50000, 10
    a = _fleet(fs, n, "velocity", seed=8)
    b = _fleet(fs, n, "velocity", seed=8)
    g = b.capture(k)
    g.replay()
    torch.cuda.synchronize()
    for _ in range(k):
        a.step()
    assert np.array_equal(_np(a.state, n), _np(b.state, n))


@pytest.mark.parametrize("n", [1, 3, 255, 257, 4097, 70001])
def test_ragged_sizes_and_kernel_paths_agree(fs, n):
    """Tail handling: the TMA stream kernel and the register kernel agree for
    sizes that are not multiples of the tile or vector width."""
    from paper_2305_16510_b200 import _native as N
    res = []
    for kern in (1, 2):
        N.set_tuning(N.FS_TUNE_KERNEL, kern)
        try:
            f = _fleet(fs, n, "velocity", seed=12)
            f.step()
            res.append(_np(f.state, n))
        finally:
            N.set_tuning(N.FS_TUNE_KERNEL, 0)
    np.testing.assert_allclose(res[0], res[1], rtol=1e-6, atol=1e-6)
    f0 = _fleet(fs, n, "velocity", seed=12)
    s, cmd = _np(f0.state, n), _np(f0.cmd, n)
    ref, _ = O.step(s, np.ones(n, np.uint8), np.zeros((4, n)), cmd, O.Gains(), O.Robot(), 0.01)
    assert_parity(res[1], ref, s, f"ragged n={n}")


def test_empty_batch_is_noop(fs):
    st = fs.RigidStateBatch.rest(0)
    cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=np.zeros((0, 3)),
                                                            yaw_rate=np.zeros(0)))
    out, flags = fs.fused_step(st, cmds, fs.ControlGains(), fs.RobotParams(), 0.01)
    assert out.n == 0 and flags.clamped.numel() == 0


@pytest.mark.parametrize("prec", [0, 1, 2])
def test_precision_variants_meet_bar_on_goldens(fs, golden, prec):
    """Every precision variant passes the golden vectors; the default (1)
    and the float64 controller (2) also pass at 1M vehicles (tools/gpu_diag.py)."""
    from paper_2305_16510_b200 import _native as N
    g = golden("mixed")
    N.set_tuning(N.FS_TUNE_PREC, prec)
    try:
        s = g["state_in"]
        st = fs.RigidStateBatch(p=s[0:3].T, q=s[3:7].T, v=s[7:10].T, omega=s[10:13].T)
        att = fs.AttitudeCommands(*g["att_cmd"], validate=False)
        vel = fs.VelocityCommands(v=g["vel_cmd"][0:3].T, yaw_rate=g["vel_cmd"][3],
                                  validate=False)
        out, _ = fs.fused_step(st, fs.CommandBatch(mode=g["mode"], attitude=att, velocity=vel),
                               fs.ControlGains(), fs.RobotParams(), 0.01)
        if prec > 0:
            assert_parity(out.numpy(), g["state_out"], s, f"prec {prec}")
        else:
            np.testing.assert_allclose(out.numpy(), g["state_out"], rtol=1e-5, atol=1e-5)
    finally:
        N.set_tuning(N.FS_TUNE_PREC, -1)


@pytest.mark.parametrize("n", [70001, 65537])
def test_stream_kernel_writes_nothing_past_n(fs, n):
    """A slice view of a larger buffer: the TMA-store tail must not touch the
    vehicles after the slice (out-of-place and in-place)."""
    from paper_2305_16510_b200 import _native as N
    big = n + 7
    s, _, _, vel, _ = config_batch("velocity", big, seed=5)
    full = fs.RigidStateBatch(p=s[0:3].T, q=s[3:7].T, v=s[7:10].T, omega=s[10:13].T)
    cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=vel[0:3].T, yaw_rate=vel[3],
                                                            validate=False))
    out_full = fs.RigidStateBatch.rest(big)
    before_out = out_full.numpy().copy()
    before_in = full.numpy().copy()
    N.set_tuning(N.FS_TUNE_KERNEL, 2)
    try:
        fs.fused_step(full.slice(slice(0, n)), cmds.slice(slice(0, n)), fs.ControlGains(),
                      fs.RobotParams(), 0.01, out=out_full.slice(slice(0, n)), want_flags=False)
        torch.cuda.synchronize()
        assert np.array_equal(out_full.numpy()[:, n:], before_out[:, n:])
        fs.fused_step(full.slice(slice(0, n)), cmds.slice(slice(0, n)), fs.ControlGains(),
                      fs.RobotParams(), 0.01, out=full.slice(slice(0, n)), want_flags=False)
        torch.cuda.synchronize()
        assert np.array_equal(full.numpy()[:, n:], before_in[:, n:])
        assert not np.array_equal(full.numpy()[:, :n], before_in[:, :n])
    finally:
        N.set_tuning(N.FS_TUNE_KERNEL, 0)


def test_step_host_matches_device_path(fs):
    """fs_step_host (host-resident state/commands, chunked over streams) gives
    the same bits as the device-resident fused step."""
    import ctypes as C
    from paper_2305_16510_b200 import _native as N
    from paper_2305_16510_b200._tensors import alloc_planes, stride0
    n = 300001
    f = _fleet(fs, n, "velocity", seed=21)
    host_state = torch.empty(f.state.shape, dtype=torch.float32, pin_memory=True)
    host_cmd = torch.empty(f.cmd.shape, dtype=torch.float32, pin_memory=True)
    host_state.copy_(f.state)
    host_cmd.copy_(f.cmd)
    dev_state, dev_cmd = alloc_planes(13, n), alloc_planes(4, n)
    streams = [torch.cuda.Stream() for _ in range(3)]
    handles = (C.c_void_p * 3)(*[s.cuda_stream for s in streams])
    d = N.fs_step_desc()
    d.n = n
    d.state_in = d.state_out = C.c_void_p(host_state.data_ptr())
    d.state_in_stride = d.state_out_stride = stride0(host_state)
    d.mode, d.integrate, d.dt = N.FS_MODE_VELOCITY, 1, 0.01
    d.cmd = C.c_void_p(host_cmd.data_ptr())
    d.cmd_stride = stride0(host_cmd)
    lib = N.load()
    N.check(lib.fs_step_host(C.byref(d), fs.RobotParams().native(), fs.ControlGains().native(),
                             fs.ControlLimits().native(), None, C.c_void_p(dev_state.data_ptr()),
                             C.c_void_p(dev_cmd.data_ptr()), stride0(dev_state), 7, handles, 3),
            "fs_step_host")
    torch.cuda.synchronize()
    f.step()
    torch.cuda.synchronize()
    np.testing.assert_allclose(host_state[:, :n].double().numpy(), _np(f.state, n),
                               rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("case", ["wrench", "rotors_flags", "respawn_wrench"])
def test_control_only_many_tiles_per_cta(fs, case):
    """Control-only calls (the controller objects, control_batch) at 2^20
    vehicles: the streaming kernel runs ~11 tiles per CTA, more than its
    ring holds, so every ring slot is reused -- the register kernel
    (FS_TUNE_KERNEL = 1) gives bitwise the same wrench / rotor thrusts /
    flags (and re-spawned commands)."""
    from paper_2305_16510_b200 import _native as N
    from paper_2305_16510_b200.allocation import QUAD_X, HEXAROTOR
    n = 1 << 20
    kw = {"wrench": dict(mode="position", want_wrench=True),
          "rotors_flags": dict(mode="position", airframes=(QUAD_X, HEXAROTOR),
                               airframe_split=n // 2, want_flags=True),
          "respawn_wrench": dict(mode="velocity", want_wrench=True, reset_prob=0.02)}[case]
    outs = []
    for kern in (1, 2):
        N.set_tuning(N.FS_TUNE_KERNEL, kern)
        try:
            m = dict(kw)
            f = _fleet(fs, n, m.pop("mode"), seed=31, **m)
            f.control()
            torch.cuda.synchronize()
            outs.append(f)
        finally:
            N.set_tuning(N.FS_TUNE_KERNEL, 0)
    a, b = outs
    assert torch.equal(a.state[:, :n], b.state[:, :n])
    assert torch.equal(a.cmd[:, :n], b.cmd[:, :n])
    if a.wrench is not None:
        assert torch.equal(a.wrench[:, :n], b.wrench[:, :n])
    if a.rotors is not None:
        assert torch.equal(a.rotors[:, :n], b.rotors[:, :n])
    if a.flags is not None:
        assert torch.equal(a.flags[:n], b.flags[:n])
