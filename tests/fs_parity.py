"""Parity criteria shared by the GPU tests (fp32 CUDA vs float64 reference).

North-star bar (BASELINE.json): every output within 1e-5 relative / 1e-6
absolute per step, i.e. |got - ref| <= 1e-6 + 1e-5 |ref|, for EVERY vehicle
outside the gimbal conditioning band |R20| >= 0.99.

Inside the band the yaw extraction atan2(r10, r00) is ill-conditioned and the
float64 reference itself moves by more than the bar under half-ulp input
noise.  There the criterion is conditioning-aware:
|got - ref| <= bar + 4 * spread, where spread is the reference's own maximum
output change over 8 random half-ulp perturbations of the fp32 inputs.
"""

from __future__ import annotations

import numpy as np

RTOL = 1e-5
ATOL = 1e-6
BAND = 0.99
SPREAD_FACTOR = 4.0


def r20(state):
    """|R20| = |2 (qx qz - qw qy)| per vehicle of a planar (13, N) state."""
    qw, qx, qy, qz = state[3], state[4], state[5], state[6]
    return np.abs(2.0 * (qx * qz - qw * qy))


def _excess(got, ref, rtol, atol):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    with np.errstate(invalid="ignore"):
        d = np.abs(got - ref) - (atol + rtol * np.abs(ref))
    both_nan = np.isnan(got) & np.isnan(ref)
    same_inf = np.isinf(got) & np.isinf(ref) & (np.sign(got) == np.sign(ref))
    d = np.where(both_nan | same_inf, -1.0, d)
    return np.where(np.isnan(d), np.inf, d)


def violations(got, ref, rtol=RTOL, atol=ATOL):
    """Per-vehicle violation mask (components along axis 0)."""
    bad = _excess(got, ref, rtol, atol) > 0
    return bad.any(axis=0) if bad.ndim > 1 else bad


def oracle_spread(fn, state, k=8, seed=0):
    """Max |fn(perturbed) - fn(state)| over k half-ulp perturbations of the
    fp32 state (relative 2^-24 per component).  fn: (13, m) -> (c, m)."""
    rng = np.random.default_rng(seed)
    base = np.asarray(fn(state), dtype=np.float64)
    spread = np.zeros_like(base)
    with np.errstate(invalid="ignore", over="ignore"):
        for _ in range(k):
            u = rng.uniform(-1.0, 1.0, state.shape) * 2.0 ** -24
            out = np.asarray(fn(state * (1.0 + u)), dtype=np.float64)
            spread = np.fmax(spread, np.abs(out - base))
    return spread


def assert_parity(got, ref, state_in, what, spread_fn=None, rtol=RTOL, atol=ATOL, band=BAND):
    """Assert the bar outside the band; inside it, the conditioning-aware
    bound when `spread_fn(state_columns, column_indices)` (the oracle as a
    function of the state) is given.
    Returns (violations outside band, in-band rows beyond the bar)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if got.ndim == 1:
        got, ref = got[None], ref[None]
    bad = violations(got, ref, rtol, atol)
    in_band = r20(state_in) >= band
    outside = bad & ~in_band
    if outside.any():
        idx = np.nonzero(outside)[0][:5]
        raise AssertionError(
            f"{what}: {int(outside.sum())}/{int((~in_band).sum())} vehicles outside the gimbal "
            f"band violate {rtol:g} rel / {atol:g} abs; first {idx.tolist()}:\n"
            f" got={got[:, idx]}\n ref={ref[:, idx]}\n"
            f" max|d|={np.nanmax(np.abs(got[:, idx] - ref[:, idx]))}")
    band_bad = bad & in_band
    if band_bad.any() and spread_fn is not None:
        cols = np.nonzero(band_bad)[0]
        spread = oracle_spread(lambda st: spread_fn(st, cols), np.asarray(state_in)[:, cols])
        ex = _excess(got[:, cols], ref[:, cols], rtol, atol) - SPREAD_FACTOR * spread
        worst = np.nonzero((ex > 0).any(axis=0))[0]
        if worst.size:
            c = cols[worst[:5]]
            raise AssertionError(
                f"{what}: {worst.size} in-band vehicles exceed bar + {SPREAD_FACTOR:g} x "
                f"reference spread; first {c.tolist()}:\n got={got[:, c]}\n ref={ref[:, c]}")
    return int(outside.sum()), int(band_bad.sum())


# K-step drift bound: per component group (p, q, v, w), the
# max |GPU - float64 reference| over the sample stays within DRIFT_FACTOR x
# the group's "fp32-storage floor" (float64 math, state rounded to fp32 after
# every step) + DRIFT_ATOL.
DRIFT_FACTOR = 16.0
DRIFT_ATOL = 1e-5
GROUPS = {"p": slice(0, 3), "q": slice(3, 7), "v": slice(7, 10), "w": slice(10, 13)}


def assert_drift(got, ref, floor, what):
    d_gpu = np.abs(np.asarray(got) - np.asarray(ref))
    d_floor = np.abs(np.asarray(floor) - np.asarray(ref))
    for name, sl in GROUPS.items():
        g, f = float(d_gpu[sl].max()), float(d_floor[sl].max())
        assert g <= DRIFT_FACTOR * f + DRIFT_ATOL, \
            f"{what}: {name} drift {g:.3e} > {DRIFT_FACTOR:g} x floor {f:.3e} + {DRIFT_ATOL:g}"
