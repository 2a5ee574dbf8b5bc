"""Rotation-group primitives -- drop-in for ``flocksim.se3`` (se3.py:1-266).

Same conventions: scalar-first unit quaternions ``[w, x, y, z]`` in
``(..., 4)`` arrays encoding body-to-world rotations, intrinsic ZYX Euler
angles (``R = R_z(yaw) R_y(pitch) R_x(roll)``), broadcasting over leading
batch dimensions.  Every function evaluates in the CUDA library
(``fs_se3``, csrc/fs_se3.cu) in float64 and returns float64 CUDA tensors;
inputs may be NumPy arrays, scalars or tensors.  Results agree with the
reference to an ulp or two of float64 (tests/test_se3_gpu.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from ._tensors import default_device, ptr, stream_handle

_EXP_TAYLOR_ANGLE = 1e-8      # se3.py:19
SKEW_TOL = 1e-9               # se3.py:22
GIMBAL_TOL = 1e-6             # se3.py:25


class NotSkewSymmetricError(ValueError):
    """vee() received a matrix that is not skew-symmetric (se3.py:28-29)."""


def _t(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float64)
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=device)


def _device(*xs):
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device
    return default_device()


def _run(op: str, inputs, widths, out_width, out2: bool = False):
    """Broadcast the inputs' leading dims, flatten to contiguous rows, launch."""
    dev = _device(*inputs)
    ts = [_t(x, dev) for x in inputs]
    lead = [t.shape[:t.dim() - (1 if w > 1 else 0)] if w > 1 else t.shape
            for t, w in zip(ts, widths)]
    for t, w in zip(ts, widths):
        if w > 1 and (t.dim() == 0 or t.shape[-1] != w):
            raise ValueError(f"{op.lower()}: expected trailing dimension {w}, got {tuple(t.shape)}")
    shape = torch.broadcast_shapes(*lead)
    rows = [t.expand(*shape, w).reshape(-1, w).contiguous() if w > 1
            else t.expand(shape).reshape(-1).contiguous() for t, w in zip(ts, widths)]
    n = int(np.prod(shape)) if len(shape) else 1
    out = torch.empty((max(n, 1), out_width), dtype=torch.float64, device=dev)
    o2 = torch.empty(max(n, 1), dtype=torch.float64, device=dev) if out2 else None
    args = [ptr(r) for r in rows] + [C.c_void_p(0)] * (3 - len(rows))
    with torch.cuda.device(dev):
        N.check(N.load().fs_se3(N.FS_SE3[op], n, *args, ptr(out), ptr(o2), stream_handle()),
                f"se3.{op.lower()}")
    out = out[:n].reshape(*shape, out_width) if out_width > 1 else out[:n].reshape(shape)
    return (out, o2[:n].reshape(shape)) if out2 else out


def hat(w):
    """Skew-symmetric matrix of a 3-vector: hat(w) @ u == cross(w, u) (se3.py:32-48)."""
    m = _run("HAT", [w], [3], 9)
    return m.reshape(*m.shape[:-1], 3, 3)


def vee(s):
    """Inverse of hat(); raises NotSkewSymmetricError when max |S + S^T| > SKEW_TOL
    (se3.py:51-67)."""
    st = _t(s, _device(s))
    if st.dim() < 2 or tuple(st.shape[-2:]) != (3, 3):
        raise ValueError(f"vee: expected (..., 3, 3), got {tuple(st.shape)}")
    v, res = _run("VEE", [st.reshape(*st.shape[:-2], 9)], [9], 3, out2=True)
    residual = float(res.max()) if res.numel() else 0.0
    if residual > SKEW_TOL:
        raise NotSkewSymmetricError(
            f"matrix is not skew-symmetric: max |S + S^T| = {residual:.3e}")
    return v


def quat_normalize(q):
    return _run("QUAT_NORMALIZE", [q], [4], 4)


def quat_multiply(q1, q2):
    """Hamilton product q1 (x) q2, renormalized (se3.py:78-97)."""
    return _run("QUAT_MULTIPLY", [q1, q2], [4, 4], 4)


def quat_conjugate(q):
    return _run("QUAT_CONJUGATE", [q], [4], 4)


def quat_rotate(q, v):
    """R(q) @ v (se3.py:106-130)."""
    return _run("QUAT_ROTATE", [q, v], [4, 3], 3)


def quat_rotate_inverse(q, v):
    """R(q)^T @ v (se3.py:133-135)."""
    return _run("QUAT_ROTATE_INVERSE", [q, v], [4, 3], 3)


def quat_to_matrix(q):
    """(..., 3, 3) rotation matrix of unit quaternions (se3.py:138-153)."""
    m = _run("QUAT_TO_MATRIX", [q], [4], 9)
    return m.reshape(*m.shape[:-1], 3, 3)


def quat_from_matrix(r):
    """Unit quaternion (w >= 0) from rotation matrices, Shepperd's method
    (se3.py:156-197)."""
    rt = _t(r, _device(r))
    if rt.dim() < 2 or tuple(rt.shape[-2:]) != (3, 3):
        raise ValueError(f"quat_from_matrix: expected (..., 3, 3), got {tuple(rt.shape)}")
    return _run("QUAT_FROM_MATRIX", [rt.reshape(*rt.shape[:-2], 9)], [9], 4)


def rot_zyx(roll, pitch, yaw):
    """R_z(yaw) R_y(pitch) R_x(roll) as a unit quaternion (se3.py:200-215)."""
    return _run("ROT_ZYX", [roll, pitch, yaw], [1, 1, 1], 4)


def rot_z(yaw):
    """Pure yaw rotation (se3.py:218-223)."""
    return _run("ROT_Z", [yaw], [1], 4)


def yaw_of(q):
    """(psi, degenerate): ZYX yaw atan2(R10, R00) and the flag for pitch within
    GIMBAL_TOL of +-pi/2 (se3.py:226-243)."""
    psi, flag = _run("YAW_OF", [q], [4], 1, out2=True)
    return psi, flag != 0


def exp_so3(w):
    """Exponential map so(3) -> SO(3) as a unit quaternion (se3.py:246-266)."""
    return _run("EXP_SO3", [w], [3], 4)


__all__ = ["GIMBAL_TOL", "SKEW_TOL", "NotSkewSymmetricError", "exp_so3", "hat", "quat_conjugate",
           "quat_from_matrix", "quat_multiply", "quat_normalize", "quat_rotate",
           "quat_rotate_inverse", "quat_to_matrix", "rot_z", "rot_zyx", "vee", "yaw_of"]
