"""CPU tests of the counter-based RNG twin (oracle/rng_twin.py).

Philox4x32-10 known-answer vectors are the published Random123 test vectors
for the algorithm (Salmon et al., SC'11); the twin must reproduce them
bit-exactly, and the device kernels (fs_rng.cuh) are checked against the
twin in tests/test_fleet_gpu.py.
"""

import numpy as np

from oracle import rng_twin as R


def _hex(t):
    return [int(x) for x in t]


def test_philox_known_answers():
    assert _hex(R.philox4x32_10(0, 0, 0, 0, 0, 0)) == [
        0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    f = 0xFFFFFFFF
    assert _hex(R.philox4x32_10(f, f, f, f, f, f)) == [
        0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert _hex(R.philox4x32_10(0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344,
                                0xA4093822, 0x299F31D0)) == [
        0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


def test_uniform_is_exact_and_in_range():
    w = np.array([0, 255, 256, 0xFFFFFFFF], dtype=np.uint32)
    u = R.u01(w)
    assert u.dtype == np.float32
    assert u[0] == 0.0 and u[1] == 0.0 and u[2] == np.float32(2.0 ** -24)
    assert u[3] < 1.0


def test_reset_mask_rate_and_determinism():
    gid = np.arange(1 << 18, dtype=np.uint64)
    m1 = R.reset_mask(42, gid, 7, 0.01)
    m2 = R.reset_mask(42, gid, 7, 0.01)
    assert np.array_equal(m1, m2)
    rate = m1.mean()
    assert abs(rate - 0.01) < 5 * np.sqrt(0.01 * 0.99 / gid.size)
    # different step -> different (independent) mask
    m3 = R.reset_mask(42, gid, 8, 0.01)
    assert (m1 & m3).mean() < 0.001


def test_shard_invariance_of_spawn():
    """Vehicle g's spawn depends on (seed, g, step) only: any sharding of the
    global ids reproduces the same vehicles bit for bit."""
    gid = np.arange(1000, dtype=np.uint64)
    full, cmd = R.spawn(5, gid, R.INIT_STEP, "position")
    a, ca = R.spawn(5, gid[:333], R.INIT_STEP, "position")
    b, cb = R.spawn(5, gid[333:], R.INIT_STEP, "position")
    assert np.array_equal(np.concatenate([a, b], axis=1), full)
    assert np.array_equal(np.concatenate([ca, cb], axis=1), cmd)


def test_spawn_distributions():
    gid = np.arange(1 << 16, dtype=np.uint64)
    st, cmd = R.spawn(1, gid, R.INIT_STEP, "velocity")
    assert np.all(np.abs(st[0:3]) <= 5.0)
    np.testing.assert_allclose(np.linalg.norm(st[3:7], axis=0), 1.0, atol=1e-12)
    assert abs(np.mean(st[3] < 0) - 0.5) < 0.02            # no canonical sign
    assert abs(st[7:10].std() - 1.0) < 0.02
    assert abs(st[10:13].std() - 0.5) < 0.01
    assert abs(cmd[0:3].std() - 1.0) < 0.02
    assert np.all(np.abs(cmd[3]) <= 1.0)
    st, cmd = R.spawn(1, gid, R.INIT_STEP, "attitude")
    assert np.all(np.abs(cmd[0:2]) <= 0.5)
    assert np.all((cmd[3] >= 0.5 * 9.81 - 1e-5) & (cmd[3] <= 1.5 * 9.81 + 1e-5))
