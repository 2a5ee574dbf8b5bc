"""CPU twin of the device RNG (paper_2305_16510_b200/csrc/fs_rng.cuh).

TEST INFRASTRUCTURE.  EXTENSION: the reference has no device RNG; its
counter-based streams are NumPy Philox-4x64 per (seed, env, reset)
(assets.py:310-315).  The build uses Philox4x32-10 (Salmon et al., SC'11,
"Parallel random numbers: as easy as 1, 2, 3"; the Random123 published
algorithm, restated here) keyed by the 64-bit seed with counter
(gid_lo, gid_hi, step, block).  Integer outputs and the uniform affine maps
are bit-exact with the device; Box-Muller normals and the Shoemake
quaternion agree to ~1 ulp (libm vs CUDA math).
"""

from __future__ import annotations

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
INIT_STEP = 0xFFFFFFFF
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorized Philox4x32-10 over uint32 arrays."""
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32) for x in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint32)
    k1 = np.asarray(k1, dtype=np.uint32)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = M0 * c0.astype(np.uint64)
            p1 = M1 * c2.astype(np.uint64)
            hi0, lo0 = (p0 >> np.uint64(32)).astype(np.uint32), (p0 & MASK32).astype(np.uint32)
            hi1, lo1 = (p1 >> np.uint64(32)).astype(np.uint32), (p1 & MASK32).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = (k0 + W0).astype(np.uint32)
            k1 = (k1 + W1).astype(np.uint32)
    return c0, c1, c2, c3


def draw_block(seed, gid, step, block):
    gid = np.asarray(gid, dtype=np.uint64)
    n = gid.shape
    return philox4x32_10((gid & MASK32).astype(np.uint32), (gid >> np.uint64(32)).astype(np.uint32),
                         np.full(n, step & 0xFFFFFFFF, np.uint32), np.full(n, block, np.uint32),
                         np.uint32(seed & 0xFFFFFFFF), np.uint32((seed >> 32) & 0xFFFFFFFF))


def u01(w):
    return (np.asarray(w, dtype=np.uint32) >> np.uint32(8)).astype(np.float32) * np.float32(2.0 ** -24)


def uaff(w, lo, span):
    return np.float32(lo) + np.float32(span) * u01(w)


def box_muller(w1, w2):
    u1 = ((np.asarray(w1, np.uint32) >> np.uint32(8)).astype(np.float64) + 1.0) * 2.0 ** -24
    u2 = u01(w2).astype(np.float64)
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2 * np.pi * u2), r * np.sin(2 * np.pi * u2)


def reset_threshold(p: float) -> int:
    t = np.floor(np.float64(np.float32(p)) * 4294967296.0)
    return 0xFFFFFFFF if t >= 4294967295.0 else int(t)


def step_key(seed, step):
    """Per-step 32-bit key (fs_rng.cuh step_key): splitmix64 finalizer over
    seed ^ step * C, upper 32 bits."""
    with np.errstate(over="ignore"):
        x = np.uint64(seed) ^ (np.uint64(step & 0xFFFFFFFF) * np.uint64(0xD1B54A32D192ED03))
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        x = x ^ (x >> np.uint64(31))
    return np.uint32(x >> np.uint64(32))


def lowbias32(x):
    x = np.asarray(x, dtype=np.uint32)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint32(16))
        x = x * np.uint32(0x7FEB352D)
        x = x ^ (x >> np.uint32(15))
        x = x * np.uint32(0x846CA68B)
        x = x ^ (x >> np.uint32(16))
    return x


def reset_word(seed, gid, step):
    """Re-spawn word (fs_rng.cuh reset_word): lowbias32 of the global id's
    low word ^ the step key ^ (high word * 0x85EBCA6B)."""
    gid = np.asarray(gid, dtype=np.uint64)
    lo = (gid & MASK32).astype(np.uint32)
    with np.errstate(over="ignore"):
        hi = (gid >> np.uint64(32)).astype(np.uint32) * np.uint32(0x85EBCA6B)
    return lowbias32(lo ^ step_key(seed, step) ^ hi)


def reset_mask(seed, gid, step, p):
    """Bit-exact per-vehicle Bernoulli(p) re-spawn decision at `step`."""
    return reset_word(seed, gid, step) < np.uint32(reset_threshold(p))


def spawn(seed, gid, step, mode, mass=1.0, gravity=9.81):
    """(state (13, n) float64, cmd (4 or 8, n) float64) -- device `spawn`."""
    b0 = draw_block(seed, gid, step, 0)
    b1 = draw_block(seed, gid, step, 1)
    b2 = draw_block(seed, gid, step, 2)
    b3 = draw_block(seed, gid, step, 3)
    b4 = draw_block(seed, gid, step, 4)
    p = [uaff(b0[k], -5.0, 10.0) for k in (1, 2, 3)]
    u1 = u01(b1[0]).astype(np.float64)
    a, b = np.sqrt(1.0 - u1), np.sqrt(u1)
    t1 = 2 * np.pi * u01(b1[1]).astype(np.float64)
    t2 = 2 * np.pi * u01(b1[2]).astype(np.float64)
    q = np.stack([b * np.cos(t2), a * np.sin(t1), a * np.cos(t1), b * np.sin(t2)])
    q = q / np.linalg.norm(q, axis=0, keepdims=True)
    n0, n1 = box_muller(b3[0], b3[1])
    n2, n3 = box_muller(b3[2], b3[3])
    n4, n5 = box_muller(b4[0], b4[1])
    n6, n7 = box_muller(b4[2], b4[3])
    st = np.stack([*[x.astype(np.float64) for x in p], *q, n0, n1, n2, 0.5 * n3, 0.5 * n4,
                   0.5 * n5])
    mg = np.float32(np.float32(mass) * np.float32(gravity))
    cmds = []
    if mode in ("attitude", "mixed"):
        cmds += [uaff(b1[3], -0.5, 1.0), uaff(b2[0], -0.5, 1.0), uaff(b2[1], -1.0, 2.0),
                 uaff(b2[2], 0.5, 1.0) * mg]
    if mode in ("velocity", "mixed"):
        b6 = draw_block(seed, gid, step, 6)
        n8, _ = box_muller(b6[0], b6[1])
        cmds += [n6, n7, n8, uaff(b2[1], -1.0, 2.0)]
    if mode == "position":
        cmds += [uaff(b1[3], -5.0, 10.0), uaff(b2[0], -5.0, 10.0), uaff(b2[2], -5.0, 10.0),
                 uaff(b2[1], -3.14159274, 6.28318548)]
    return st, np.stack([np.asarray(c, dtype=np.float64) for c in cmds])


def spawn_vparams(seed, gid, mass=1.0, jdiag=(0.01, 0.01, 0.02)):
    b = draw_block(seed, gid, INIT_STEP, 5)
    base = [mass, *jdiag]
    return np.stack([(np.float32(base[k]) * uaff(b[k], 0.8, 0.4)).astype(np.float64)
                     for k in range(4)])


PLACE_BLOCK = 0x100


def world_place(seed, gid, counter, goal, lo, hi, bounds, r, attempts=100):
    """Device placement (fs_world.cu `place`): p = (lo + u*(hi-lo)) * bounds in
    float32 with explicit rounding, accepted when r <= p <= bounds - r; attempt
    a uses Philox block PLACE_BLOCK + 2a (+1 for goals).  Returns (3, n)
    float64 (bit-exact) and the success mask."""
    gid = np.atleast_1d(np.asarray(gid, dtype=np.uint64))
    lo32 = np.asarray(lo, dtype=np.float64).astype(np.float32)
    span32 = (np.asarray(hi, dtype=np.float64) - np.asarray(lo, dtype=np.float64)).astype(np.float32)
    b32 = np.asarray(bounds, dtype=np.float64).astype(np.float32)
    r32 = np.float32(r)
    out = np.zeros((3, gid.size), dtype=np.float32)
    done = np.zeros(gid.size, dtype=bool)
    for a in range(attempts):
        blk = draw_block(seed, gid, counter, PLACE_BLOCK + 2 * a + (1 if goal else 0))
        p = np.stack([(lo32[k] + u01(blk[k]) * span32[k]) * b32[k] for k in range(3)])
        ok = ((p >= r32) & (p <= b32[:, None] - r32)).all(axis=0)
        take = ok & ~done
        out[:, take] = p[:, take]
        done |= ok
        if done.all():
            break
    return out.astype(np.float64), done
