"""Seeded host-side samples of the BASELINE.json config distributions.

TEST INFRASTRUCTURE (CPU baseline and parity inputs only).  Values are
rounded to float32 so the same numbers can be fed to the fp32 kernels.
Distributions: SURVEY.md 8(d) -- p ~ U[-5,5]^3, q uniform on S^3
(Shoemake), v ~ N(0,1)^3, w ~ N(0,0.5^2)^3; commands per mode.
"""

from __future__ import annotations

import numpy as np


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def shoemake(u1, u2, u3):
    a, b = np.sqrt(1.0 - u1), np.sqrt(u1)
    t1, t2 = 2 * np.pi * u2, 2 * np.pi * u3
    return np.stack([b * np.cos(t2), a * np.sin(t1), a * np.cos(t1), b * np.sin(t2)])


def config_states(rng, n):
    p = rng.uniform(-5.0, 5.0, (3, n))
    q = f32(shoemake(rng.random(n), rng.random(n), rng.random(n)))
    q = f32(q / np.linalg.norm(q, axis=0, keepdims=True))
    v = rng.normal(0.0, 1.0, (3, n))
    w = rng.normal(0.0, 0.5, (3, n))
    return np.concatenate([f32(p), q, f32(v), f32(w)])


def config_batch(mode, n, seed=0, mass=1.0, gravity=9.81):
    """(state (13,n), mode (n,), att (4,n), vel (4,n), pos (4,n))."""
    rng = np.random.default_rng(seed)
    s = config_states(rng, n)
    att = f32(np.stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n),
                        rng.uniform(-1.0, 1.0, n), rng.uniform(0.5, 1.5, n) * mass * gravity]))
    vel = f32(np.concatenate([rng.normal(0.0, 1.0, (3, n)), rng.uniform(-1.0, 1.0, (1, n))]))
    pos = f32(np.concatenate([rng.uniform(-5.0, 5.0, (3, n)),
                              rng.uniform(-np.pi, np.pi, (1, n))]))
    m = np.full(n, 1 if mode == "velocity" else 0, dtype=np.uint8)
    return s, m, att, vel, pos
