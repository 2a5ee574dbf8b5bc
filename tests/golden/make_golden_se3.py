"""Golden vectors for flocksim.se3 from the UNMODIFIED reference.

    python tests/golden/make_golden_se3.py   (in the build container)

Seeded random inputs plus the branch cases: rotation vectors below the
series threshold (1e-8) and zero, rotation matrices whose largest Shepperd
pivot is each of w, x, y, z, quaternions with negative scalar parts and at
gimbal lock, skew matrices within and beyond SKEW_TOL.
"""

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF_SRC)
    from flocksim import se3
    rng = np.random.default_rng(3)
    n = 512
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    q2 = rng.normal(size=(n, 4))
    q2 /= np.linalg.norm(q2, axis=1, keepdims=True)
    v = rng.normal(size=(n, 3)) * 3.0
    w = rng.normal(size=(n, 3))
    w[:8] *= 1e-9                      # series branch
    w[8] = 0.0
    ang = rng.uniform(-3.5, 3.5, size=(n, 3))
    # pivots: rotations by ~pi about x, y, z and small ones (w pivot)
    piv = np.concatenate([se3.exp_so3(np.array([[3.1, 0.1, 0.0], [0.1, 3.1, 0.0],
                                                [0.0, 0.1, 3.1], [0.1, 0.2, 0.3]])), q])
    gimbal = se3.rot_zyx(0.3, np.pi / 2, -0.7)[None, :]
    qy = np.concatenate([q, gimbal])
    skew = se3.hat(v)
    out = dict(q=q, q2=q2, v=v, w=w, ang=ang, piv=piv, qy=qy, skew=skew,
               normalize=se3.quat_normalize(q * 2.5), multiply=se3.quat_multiply(q, q2),
               conjugate=se3.quat_conjugate(q), rotate=se3.quat_rotate(q, v),
               rotate_inv=se3.quat_rotate_inverse(q, v), to_matrix=se3.quat_to_matrix(q),
               from_matrix=se3.quat_from_matrix(se3.quat_to_matrix(piv)),
               rot_zyx=se3.rot_zyx(ang[:, 0], ang[:, 1], ang[:, 2]), rot_z=se3.rot_z(ang[:, 2]),
               exp=se3.exp_so3(w), hat=skew, vee=se3.vee(skew))
    psi, deg = se3.yaw_of(qy)
    out["yaw"], out["yaw_deg"] = psi, deg
    np.savez_compressed(os.path.join(HERE, "se3.npz"), **out)
    print("wrote se3.npz; gimbal flags:", int(deg.sum()))


if __name__ == "__main__":
    main()
