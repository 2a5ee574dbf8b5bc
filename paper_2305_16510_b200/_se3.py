"""Host-side float64 rotation helpers for scene construction (NumPy).

Used only while building data on the host -- parsing asset files
(assets.parse_urdf_subset), the nominal camera mount
(camera.CameraConfig.mount_rotation) and flattening explicit instance lists
(scene.compile_instances).  The stepping, collision, reset and render paths
run on the GPU (csrc/fs_scene.cuh holds their device twins).

Conventions follow flocksim.se3 (se3.py:70-215): scalar-first unit
quaternions, products renormalized, R(q) acting on column vectors,
rot_zyx = R_z(yaw) R_y(pitch) R_x(roll).
"""

from __future__ import annotations

import numpy as np


def quat_normalize(q):
    q = np.asarray(q, dtype=np.float64)
    n = np.sqrt(q[..., 0] ** 2 + q[..., 1] ** 2 + q[..., 2] ** 2 + q[..., 3] ** 2)
    return q / n[..., None]


def quat_multiply(a, b):
    """Hamilton product a (x) b (rotate by b, then a), renormalized."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    aw, ax, ay, az = (a[..., i] for i in range(4))
    bw, bx, by, bz = (b[..., i] for i in range(4))
    out = np.stack([aw * bw - ax * bx - ay * by - az * bz,
                    aw * bx + ax * bw + ay * bz - az * by,
                    aw * by - ax * bz + ay * bw + az * bx,
                    aw * bz + ax * by - ay * bx + az * bw], axis=-1)
    return quat_normalize(out)


def quat_rotate(q, v):
    """R(q) v as v + w t + u x t with t = 2 u x v."""
    q = np.asarray(q, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    w, x, y, z = (q[..., i] for i in range(4))
    vx, vy, vz = v[..., 0], v[..., 1], v[..., 2]
    tx = 2.0 * (y * vz - z * vy)
    ty = 2.0 * (z * vx - x * vz)
    tz = 2.0 * (x * vy - y * vx)
    return np.stack([vx + w * tx + (y * tz - z * ty),
                     vy + w * ty + (z * tx - x * tz),
                     vz + w * tz + (x * ty - y * tx)], axis=-1)


def quat_to_matrix(q):
    q = np.asarray(q, dtype=np.float64)
    w, x, y, z = (q[..., i] for i in range(4))
    return np.stack([
        np.stack([1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)], -1),
        np.stack([2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)], -1),
        np.stack([2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)], -1),
    ], axis=-2)


def rot_zyx(roll, pitch, yaw):
    """Unit quaternion of R_z(yaw) R_y(pitch) R_x(roll) from half-angle axis quaternions."""
    hr, hp, hy = (np.asarray(a, dtype=np.float64) / 2.0 for a in (roll, pitch, yaw))
    zr, zp, zy = np.zeros_like(hr), np.zeros_like(hp), np.zeros_like(hy)
    qx = np.stack([np.cos(hr), np.sin(hr), zr, zr], axis=-1)
    qy = np.stack([np.cos(hp), zp, np.sin(hp), zp], axis=-1)
    qz = np.stack([np.cos(hy), zy, zy, np.sin(hy)], axis=-1)
    return quat_multiply(qz, quat_multiply(qy, qx))
