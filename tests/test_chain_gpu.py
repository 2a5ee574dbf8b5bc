"""GPU tests of chained steps (fs_step_desc.tile_sync): consecutive in-place
steps launched as programmatic dependents, each tile of step k+1 loaded only
once step k has published it.  Chaining is a scheduling change only, so a
chained rollout must be BITWISE identical to the same steps launched one
after another (states, commands rewritten by re-spawns, flags and the
integer episode statistics), for every streaming-kernel variant, for ragged
sizes, inside CUDA graphs replayed more than once, and at the bench size.
"""

import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fs():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2305_16510_b200 as fs
    fs._native.load()
    return fs


def _pair(n, mode, **kw):
    from paper_2305_16510_b200.fleet import Fleet
    return Fleet(n, mode=mode, **kw), Fleet(n, mode=mode, **kw)


def _same(a, b, n):
    assert torch.equal(a.state[:, :n], b.state[:, :n])
    assert torch.equal(a.cmd[:, :n], b.cmd[:, :n])
    if a.stats_slots is not None:
        assert torch.equal(a.stats_local(), b.stats_local())
    if a.flags is not None:
        assert torch.equal(a.flags[:n], b.flags[:n])
    if a.rotors is not None:
        assert torch.equal(a.rotors[:, :n], b.rotors[:, :n])


def _frames():
    from paper_2305_16510_b200.allocation import HEXAROTOR, QUAD_X
    return QUAD_X, HEXAROTOR


CASES = {
    "velocity": dict(mode="velocity"),
    "attitude": dict(mode="attitude"),
    "position_respawn_stats": dict(mode="position", reset_prob=0.01, want_stats=True),
    "stats_only": dict(mode="position", want_stats=True),
    "mixed": dict(mode="mixed"),
    "hetero_rotors": dict(mode="position", hetero=True, airframes="frames",
                          rotor_dynamics=True),
    "flags_outputs": dict(mode="velocity", want_flags=True, reset_prob=0.02),
    "hetero_respawn_stats": dict(mode="position", hetero=True, airframes="frames",
                                 rotor_dynamics=True, reset_prob=0.02, want_stats=True),
    "attitude_stats": dict(mode="attitude", want_stats=True),
}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("n", [1 << 17, 300001])
def test_chained_rollout_bitwise_equals_unchained(fs, case, n):
    kw = dict(CASES[case])
    if kw.get("airframes") == "frames":
        kw["airframes"] = _frames()
        kw["airframe_split"] = n // 2
    a, b = _pair(n, seed=11, **kw)
    if kw["mode"] == "mixed":
        m = (torch.arange(n, device=a.device) % 3 == 0).to(torch.uint8)
        a.mode_plane[:n].copy_(m)
        b.mode_plane[:n].copy_(m)
    k = 12
    for _ in range(k):
        a.step()
    b.rollout(k, chained=True)
    torch.cuda.synchronize()
    assert a.step_index == b.step_index == k
    _same(a, b, n)


def test_chained_graph_replayed_twice(fs):
    """The graph zeroes the counters itself, so a second replay (counters
    left at k by the first) chains correctly too."""
    n, k = 1 << 18, 16
    a, b = _pair(n, "position", seed=5, reset_prob=0.01, want_stats=True)
    g = b.capture(k, chained=True)
    b.stats_slots.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for _ in range(2):          # the graph baked step indices 0..k-1: run them twice
        a.step_index = 0
        for _ in range(k):
            a.step()
    torch.cuda.synchronize()
    _same(a, b, n)


def test_chained_bench_size(fs):
    """cfg2's per-GPU size (2^22, velocity) over 40 chained steps."""
    n, k = 1 << 22, 40
    a, b = _pair(n, "velocity", seed=2024)
    for _ in range(k):
        a.step()
    b.rollout(k, chained=True)
    torch.cuda.synchronize()
    _same(a, b, n)


def test_chain_rejected_off_the_streaming_kernel(fs):
    """Below the streaming kernel's minimum size there is nothing to chain:
    fs_step refuses tile_sync instead of running unsynchronized."""
    from paper_2305_16510_b200 import _native as N
    from paper_2305_16510_b200.fleet import Fleet
    f = Fleet(4096, mode="velocity")
    assert not f.chainable
    sync = torch.zeros(64, dtype=torch.int32, device=f.device)
    d = f._desc(True)
    d.tile_sync = C.c_void_p(sync.data_ptr())
    d.sync_wait, d.sync_post = 1, 2
    rc = f.lib.fs_step(C.byref(d), f._robot, f._gains, f._limits, f._frames,
                       C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == N.FS_EINVAL
    assert "streaming kernel" in f.lib.fs_last_error().decode()
    f.rollout(5)                # chained=True degrades to plain launches here
    torch.cuda.synchronize()
    assert f.step_index == 5


def test_counters_published(fs):
    """After a chain of k steps every counter holds k."""
    n, k = 200003, 7
    from paper_2305_16510_b200.fleet import Fleet
    f = Fleet(n, mode="velocity", seed=1)
    f.rollout(k, chained=True)
    torch.cuda.synchronize()
    ng = f.lib.fs_tile_sync_len(n)
    assert torch.all(f.tile_sync[:ng] == k)


# --- fs_step_many: K steps in one persistent streaming launch -----------------

@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("n", [1 << 17, 300001])
def test_step_many_bitwise_equals_unchained(fs, case, n):
    kw = dict(CASES[case])
    if kw.get("airframes") == "frames":
        kw["airframes"] = _frames()
        kw["airframe_split"] = n // 2
    a, b = _pair(n, seed=13, **kw)
    if kw["mode"] == "mixed":
        m = (torch.arange(n, device=a.device) % 3 == 0).to(torch.uint8)
        a.mode_plane[:n].copy_(m)
        b.mode_plane[:n].copy_(m)
    k = 9
    for _ in range(k):
        a.step()
    b.rollout(k, persistent=True)
    torch.cuda.synchronize()
    assert a.step_index == b.step_index == k
    _same(a, b, n)


@pytest.mark.parametrize("n", [(1 << 15) + 5, 142080, 148 * 640 * 2 + 77])
def test_step_many_small_and_ragged_tile_counts(fs, n):
    """Fewer tiles than CTAs, between one and two rounds, and just over two
    rounds per step: the publication lag shrinks so that no CTA waits on a
    tile it has not yet published itself."""
    a, b = _pair(n, "position", seed=3, reset_prob=0.05, want_stats=True)
    k = 23
    for _ in range(k):
        a.step()
    b.rollout(k, persistent=True)
    torch.cuda.synchronize()
    _same(a, b, n)


def test_step_many_in_graph_replayed_twice(fs):
    n, k = 1 << 18, 16
    a, b = _pair(n, "velocity", seed=6)
    g = b.capture(k, persistent=True)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for _ in range(2 * k):
        a.step()
    # (velocity mode: no step-indexed draws, so replaying the baked indices is exact)
    _same(a, b, n)


def test_step_many_bench_size(fs):
    n, k = 1 << 22, 40
    a, b = _pair(n, "velocity", seed=2024)
    for _ in range(k):
        a.step()
    b.step_many(k)
    torch.cuda.synchronize()
    _same(a, b, n)


def test_step_many_validation(fs):
    from paper_2305_16510_b200 import _native as N
    from paper_2305_16510_b200.fleet import Fleet
    f = Fleet(1 << 16, mode="velocity")
    d = f._desc(True)
    h = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    assert f.lib.fs_step_many(C.byref(d), f._robot, f._gains, f._limits, f._frames, 4, h) \
        == N.FS_EINVAL            # steps > 1 without tile_sync
    assert "tile_sync" in f.lib.fs_last_error().decode()
    d.tile_sync = C.c_void_p(f.tile_sync.data_ptr())
    d.sync_wait, d.sync_post = 0, 2
    assert f.lib.fs_step_many(C.byref(d), f._robot, f._gains, f._limits, f._frames, 4, h) \
        == N.FS_EINVAL
    assert "sync_post" in f.lib.fs_last_error().decode()
    small = Fleet(1000, mode="velocity")
    with pytest.raises(ValueError, match="step_many"):
        small.step_many(3)


def test_step_many_shard_invariance(fs):
    """One persistent launch over the whole fleet == four shards with their
    global-id offsets (re-spawn keys per step and global id), bitwise, with
    integer statistics summing to the same totals."""
    from paper_2305_16510_b200.fleet import Fleet
    from paper_2305_16510_b200.parallel import shard_bounds
    n, k = 300000, 11
    whole = Fleet(n, mode="position", seed=21, reset_prob=0.03, want_stats=True)
    whole.rollout(k, persistent=True)
    parts, tot = [], torch.zeros(3, dtype=torch.int64)
    for r in range(4):
        lo, hi = shard_bounds(n, 4, r)
        f = Fleet(hi - lo, mode="position", seed=21, first_id=lo, reset_prob=0.03,
                  want_stats=True)
        f.rollout(k, persistent=True)
        parts.append(f.state[:, :hi - lo])
        tot += f.stats_local().cpu()
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(parts, dim=1), whole.state[:, :n])
    assert torch.equal(tot, whole.stats_local().cpu())


def test_step_many_continues_a_chain(fs):
    """Two fs_step_many launches back to back, the second continuing the
    first's counters (sync_wait = 4: a programmatic dependent AND a
    cooperative launch), equal 7 plain steps; K = 1 equals fs_step."""
    from paper_2305_16510_b200 import _native as N
    n = 200000
    a, b = _pair(n, "position", seed=8, reset_prob=0.02, want_stats=True)
    for _ in range(7):
        a.step()
    h = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    b.tile_sync.zero_()
    for k0, k, wait in ((0, 4, 0), (4, 3, 4)):
        d = b._desc(True)
        d.step_index = k0
        d.tile_sync = C.c_void_p(b.tile_sync.data_ptr())
        d.sync_wait, d.sync_post = wait, wait + 1
        N.check(b.lib.fs_step_many(C.byref(d), b._robot, b._gains, b._limits, b._frames, k, h),
                "fs_step_many")
    torch.cuda.synchronize()
    ng = b.lib.fs_tile_sync_len(n)
    assert torch.all(b.tile_sync[:ng] == 7)
    _same(a, b, n)
    c, e = _pair(n, "velocity", seed=4)
    c.step()
    e.step_many(1)
    torch.cuda.synchronize()
    _same(c, e, n)


@pytest.mark.parametrize("case", ["velocity", "position_respawn_stats", "flags_outputs"])
def test_step_many_out_of_place_equals_in_place(fs, case):
    """fs_step_many with state_in != state_out: step 0 reads
    state_in, every later step the previous step's state_out, so K steps
    out of place equal K in-place steps bitwise and leave state_in intact."""
    from paper_2305_16510_b200 import _native as N
    from paper_2305_16510_b200._tensors import alloc_planes, stride0
    n, k = 150001, 6
    a, b = _pair(n, seed=17, **CASES[case])
    for _ in range(k):
        a.step()
    src = b.state.clone()
    out = alloc_planes(13, n, b.device)
    out.fill_(float("nan"))
    h = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    b.tile_sync.zero_()
    d = b._desc(True)
    d.state_out = C.c_void_p(out.data_ptr())
    d.state_out_stride = stride0(out)
    d.tile_sync = C.c_void_p(b.tile_sync.data_ptr())
    d.sync_wait, d.sync_post = 0, 1
    N.check(b.lib.fs_step_many(C.byref(d), b._robot, b._gains, b._limits, b._frames, k, h),
            "fs_step_many")
    torch.cuda.synchronize()
    assert torch.equal(b.state[:, :n], src[:, :n])          # input untouched
    assert torch.equal(out[:, :n], a.state[:, :n])
    assert torch.equal(b.cmd[:, :n], a.cmd[:, :n])
    if a.stats_slots is not None:
        assert torch.equal(a.stats_local(), b.stats_local())
    if a.flags is not None:
        assert torch.equal(a.flags[:n], b.flags[:n])


def test_sync_timeout_tuning_validation(fs):
    from paper_2305_16510_b200 import _native as N
    lib = N.load()
    assert lib.fs_set_tuning(N.FS_TUNE_SYNC_TIMEOUT_MS, -1) == N.FS_EINVAL
    assert lib.fs_set_tuning(N.FS_TUNE_SYNC_TIMEOUT_MS, 0) == N.FS_OK
    assert lib.fs_set_tuning(N.FS_TUNE_SYNC_TIMEOUT_MS, 10000) == N.FS_OK


@pytest.mark.parametrize("acq", [0, 1, 3, 4, 7])
def test_step_many_acquire_variants_bitwise(fs, acq):
    """Every load-side handoff variant (FS_TUNE_CHAIN_ACQUIRE bits: acquire
    loads, proxy fence, fence.acq_rel) changes only ordering strength, never
    results; the default (2) is covered by every other chained test."""
    from paper_2305_16510_b200 import _native as N
    n, k = 200003, 7
    a, b = _pair(n, "position", seed=31, reset_prob=0.02, want_stats=True)
    for _ in range(k):
        a.step()
    N.set_tuning(N.FS_TUNE_CHAIN_ACQUIRE, acq)
    try:
        b.step_many(k)
        torch.cuda.synchronize()
    finally:
        N.set_tuning(N.FS_TUNE_CHAIN_ACQUIRE, 2)
    _same(a, b, n)
    assert N.load().fs_set_tuning(N.FS_TUNE_CHAIN_ACQUIRE, 8) == N.FS_EINVAL
