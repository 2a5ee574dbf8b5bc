"""CPU oracle of the obstacle scene and depth camera -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use this module;
the product path is the CUDA library.  float64 NumPy restatements of:

  _primitive_aabb        scene.py:62-73
  compile_instances      scene.py:76-124    (instance pose o primitive pose)
  signed_distances       scene.py:127-165   (box / z-cylinder / sphere SDF)
  min_distance           scene.py:168-181
  check_collisions       world.py:95-106    (primitives + env bounds)
  _pixel_rays            camera.py:122-130
  _cast_one_primitive    camera.py:170-227  (slab box, quadratic sphere,
                                             lateral quadratic + cap slab cylinder)
  cast_rays              camera.py:230-282  (nearest collision-enabled hit,
                                             lowest slot wins ties)
  render                 camera.py:306-335  (camera pose = robot pose o mount)

Pinned against the reference itself (tests/golden/scene.npz, made by
tests/golden/make_golden_scene.py from the unmodified flocksim) in
tests/test_scene_oracle.py.  Arrays follow the reference's (E, K, ...)
PrimitiveSet layout (a dict with kind, dims, position, rot, seg_id,
collision, aabb_min, aabb_max).

``rebuild_twin`` restates the library's device-side obstacle reset
(csrc/fs_scene.cuh rebuild_env / pick_env / randomize_mount: the Philox
draw layout and the float64 pose arithmetic) so the device resets can be
checked independently.
"""

from __future__ import annotations

import numpy as np

from . import flocksim_oracle as O
from . import rng_twin as R

BOX, CYL, SPH, PAD = 0, 1, 2, -1


# ---- rotations (se3.py) ------------------------------------------------------------

def qmul(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    w = a[..., 0] * b[..., 0] - a[..., 1] * b[..., 1] - a[..., 2] * b[..., 2] - a[..., 3] * b[..., 3]
    x = a[..., 0] * b[..., 1] + a[..., 1] * b[..., 0] + a[..., 2] * b[..., 3] - a[..., 3] * b[..., 2]
    y = a[..., 0] * b[..., 2] - a[..., 1] * b[..., 3] + a[..., 2] * b[..., 0] + a[..., 3] * b[..., 1]
    z = a[..., 0] * b[..., 3] + a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1] + a[..., 3] * b[..., 0]
    q = np.stack([w, x, y, z], axis=-1)
    return q / np.sqrt((q * q).sum(axis=-1))[..., None]


def qrot(q, v):
    q = np.asarray(q, np.float64)
    v = np.asarray(v, np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    vx, vy, vz = v[..., 0], v[..., 1], v[..., 2]
    tx, ty, tz = 2.0 * (y * vz - z * vy), 2.0 * (z * vx - x * vz), 2.0 * (x * vy - y * vx)
    return np.stack([vx + w * tx + (y * tz - z * ty), vy + w * ty + (z * tx - x * tz),
                     vz + w * tz + (x * ty - y * tx)], axis=-1)


def qmat(q):
    q = np.asarray(q, np.float64)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    r = np.empty(q.shape[:-1] + (3, 3))
    r[..., 0, 0] = 1.0 - 2.0 * (y * y + z * z)
    r[..., 0, 1] = 2.0 * (x * y - w * z)
    r[..., 0, 2] = 2.0 * (x * z + w * y)
    r[..., 1, 0] = 2.0 * (x * y + w * z)
    r[..., 1, 1] = 1.0 - 2.0 * (x * x + z * z)
    r[..., 1, 2] = 2.0 * (y * z - w * x)
    r[..., 2, 0] = 2.0 * (x * z - w * y)
    r[..., 2, 1] = 2.0 * (y * z + w * x)
    r[..., 2, 2] = 1.0 - 2.0 * (x * x + y * y)
    return r


def rot_zyx(roll, pitch, yaw):
    hr, hp, hy = (np.asarray(a, np.float64) / 2.0 for a in (roll, pitch, yaw))
    z = np.zeros(np.broadcast(hr, hp, hy).shape)
    qx = np.stack([np.cos(hr) + z, np.sin(hr) + z, z, z], axis=-1)
    qy = np.stack([np.cos(hp) + z, z, np.sin(hp) + z, z], axis=-1)
    qz = np.stack([np.cos(hy) + z, z, z, np.sin(hy) + z], axis=-1)
    return qmul(qz, qmul(qy, qx))


# ---- primitive sets --------------------------------------------------------------------

def aabb(kind, dims, position, rot):
    """Conservative AABBs (scene.py:62-73) for (..., 3) arrays."""
    kind = np.asarray(kind)[..., None]
    half_box = (np.abs(rot) * (dims / 2.0)[..., None, :]).sum(axis=-1)
    axis = rot[..., :, 2]
    half_cyl = np.abs(axis) * (dims[..., 1:2] / 2.0) + dims[..., 0:1] * np.sqrt(
        np.maximum(0.0, 1.0 - axis * axis))
    half_sph = np.repeat(dims[..., 0:1], 3, axis=-1)
    half = np.where(kind == BOX, half_box, np.where(kind == CYL, half_cyl, half_sph))
    lo, hi = position - half, position + half
    pad = kind[..., 0] == PAD
    lo[pad] = 0.0
    hi[pad] = 0.0
    return lo, hi


def compile_rows(rows, width=None):
    """rows: per env a list of (kind, dims(3), prim pos(3), prim quat(4), inst
    pos(3), inst quat(4), seg, collision); the instance pose composes onto the
    primitive pose (scene.py:100-105).  Returns the PrimitiveSet dict."""
    k = max((len(r) for r in rows), default=0) if width is None else width
    e = len(rows)
    out = dict(kind=np.full((e, k), PAD, np.int8), dims=np.zeros((e, k, 3)),
               position=np.zeros((e, k, 3)), rot=np.broadcast_to(np.eye(3), (e, k, 3, 3)).copy(),
               seg_id=np.zeros((e, k), np.int32), collision=np.zeros((e, k), bool))
    for ei, row in enumerate(rows):
        for ki, (kd, dm, pp, pq, ip, iq, sg, cl) in enumerate(row):
            out["kind"][ei, ki] = kd
            out["dims"][ei, ki] = dm
            out["position"][ei, ki] = np.asarray(ip) + qrot(iq, pp)
            out["rot"][ei, ki] = qmat(qmul(iq, pq))
            out["seg_id"][ei, ki] = sg
            out["collision"][ei, ki] = cl
    out["aabb_min"], out["aabb_max"] = aabb(out["kind"], out["dims"], out["position"], out["rot"])
    return out


def signed_distances(ps, points):
    """(E, K) signed distances of one point per env, +inf on pads (scene.py:127-165)."""
    p = np.asarray(points, np.float64)
    d = p[:, None, :] - ps["position"]                      # (E, K, 3)
    r = ps["rot"]
    l = np.einsum("ekij,eki->ekj", r, d)                    # R^T d
    lx, ly, lz = l[..., 0], l[..., 1], l[..., 2]
    d0, d1, d2 = ps["dims"][..., 0], ps["dims"][..., 1], ps["dims"][..., 2]
    q = np.stack([np.abs(lx) - d0 / 2.0, np.abs(ly) - d1 / 2.0, np.abs(lz) - d2 / 2.0], -1)
    box = np.sqrt((np.maximum(q, 0.0) ** 2).sum(-1)) + np.minimum(q.max(-1), 0.0)
    rho = np.sqrt(lx * lx + ly * ly) - d0
    ax = np.abs(lz) - d1 / 2.0
    cyl = (np.sqrt(np.maximum(rho, 0.0) ** 2 + np.maximum(ax, 0.0) ** 2)
           + np.minimum(np.maximum(rho, ax), 0.0))
    sph = np.sqrt(lx * lx + ly * ly + lz * lz) - d0
    kind = ps["kind"]
    dist = np.where(kind == BOX, box, np.where(kind == CYL, cyl, sph))
    return np.where(kind == PAD, np.inf, dist)


def min_distance(ps, points, collision_only=True):
    d = signed_distances(ps, points)
    if collision_only:
        d = np.where(ps["collision"], d, np.inf)
    if d.shape[1] == 0:
        return np.full(d.shape[0], np.inf)
    return d.min(axis=1)


def check_collisions(p, r, ps, bounds):
    """world.py:95-106 on (E, 3) positions: (collided, out_of_bounds)."""
    p = np.asarray(p, np.float64)
    b = np.asarray(bounds, np.float64)
    hit = min_distance(ps, p) < r
    oob = ((p < r) | (p > b - r)).any(axis=1)
    return hit | oob, oob


# ---- ray casting -----------------------------------------------------------------------

def pixel_rays(width, height, hfov):
    """(H*W, 3) unit camera-frame rays (camera.py:122-130)."""
    s = 2.0 * np.tan(hfov / 2.0) / width
    u = (np.arange(width) + 0.5 - width / 2.0) * s
    v = (np.arange(height) + 0.5 - height / 2.0) * s
    xs, ys = np.meshgrid(u, v)
    d = np.stack([xs.ravel(), ys.ravel(), np.ones(width * height)], axis=-1)
    return d / np.sqrt((d * d).sum(axis=1))[:, None]


def _slab(o, d, h, lo, hi):
    with np.errstate(divide="ignore", invalid="ignore"):
        t1 = (-h - o) / d
        t2 = (h - o) / d
    par = d == 0.0
    inside = np.abs(o) <= h
    a = np.where(par, np.where(inside, -np.inf, np.inf), np.minimum(t1, t2))
    b = np.where(par, np.where(inside, np.inf, -np.inf), np.maximum(t1, t2))
    return np.maximum(lo, a), np.minimum(hi, b)


def _interval(lo, hi):
    t = np.where(lo > 0.0, lo, hi)
    return np.where((hi >= lo) & (t > 0.0), t, np.inf)


def ray_prim(o, d, kind, dims, center, rot):
    """(M,) hit parameters of rays (o (M,3) or (3,), d (M,3)) on one primitive."""
    rel = np.asarray(o, np.float64) - center
    ol = rel @ rot          # columns of rot = primitive axes: R^T rel
    dl = np.asarray(d, np.float64) @ rot
    if ol.ndim == 1:
        ol = np.broadcast_to(ol, dl.shape)
    m = dl.shape[0]
    if kind == BOX:
        lo, hi = np.full(m, -np.inf), np.full(m, np.inf)
        for i in range(3):
            lo, hi = _slab(ol[:, i], dl[:, i], dims[i] / 2.0, lo, hi)
        return _interval(lo, hi)
    if kind == SPH:
        b = (ol * dl).sum(axis=1)
        c = (ol * ol).sum(axis=1) - dims[0] * dims[0]
        disc = b * b - c
        root = np.sqrt(np.maximum(disc, 0.0))
        t1, t2 = -b - root, -b + root
        t = np.where(t1 > 0.0, t1, t2)
        return np.where((disc >= 0.0) & (t > 0.0), t, np.inf)
    rad, length = dims[0], dims[1]
    a = dl[:, 0] ** 2 + dl[:, 1] ** 2
    b = ol[:, 0] * dl[:, 0] + ol[:, 1] * dl[:, 1]
    c = ol[:, 0] ** 2 + ol[:, 1] ** 2 - rad * rad
    par = a == 0.0
    with np.errstate(divide="ignore", invalid="ignore"):
        disc = b * b - a * c
        root = np.sqrt(np.maximum(disc, 0.0))
        qlo = (-b - root) / a
        qhi = (-b + root) / a
    inr = c <= 0.0
    qlo = np.where(par, np.where(inr, -np.inf, np.inf), qlo)
    qhi = np.where(par, np.where(inr, np.inf, -np.inf), qhi)
    nolat = ~par & (disc < 0.0)
    qlo = np.where(nolat, np.inf, qlo)
    qhi = np.where(nolat, -np.inf, qhi)
    lo, hi = _slab(ol[:, 2], dl[:, 2], length / 2.0, qlo, qhi)
    return _interval(lo, hi)


def cast_rays(origin, dirs, ps, e, max_range):
    """Nearest collision-enabled hit per ray in env e (camera.py:230-282)."""
    dirs = np.asarray(dirs, np.float64)
    best = np.full(dirs.shape[0], np.inf)
    seg = np.zeros(dirs.shape[0], np.int32)
    for k in range(ps["kind"].shape[1]):
        kd = int(ps["kind"][e, k])
        if kd == PAD or not ps["collision"][e, k]:
            continue
        t = ray_prim(origin, dirs, kd, ps["dims"][e, k], ps["position"][e, k], ps["rot"][e, k])
        closer = t < best
        best[closer] = t[closer]
        seg[closer] = ps["seg_id"][e, k]
    miss = best > max_range
    return np.where(miss, max_range, best), np.where(miss, 0, seg).astype(np.int32)


def camera_pose(p, q, mount_p, mount_q):
    """camera.py:322-324: origin p + R(q) mount_p, orientation q (x) mount_q."""
    return np.asarray(p, np.float64) + qrot(q, mount_p), qmul(q, mount_q)


def render(p, q, mount_p, mount_q, ps, width, height, hfov, max_range, envs=None):
    """(n, H, W) float32 depth and int32 segmentation (camera.py:306-335).
    p (E, 3), q (E, 4), mounts (E, 3) / (E, 4)."""
    rays = pixel_rays(width, height, hfov)
    envs = range(len(p)) if envs is None else envs
    depth, seg = [], []
    for i in envs:
        o, qc = camera_pose(p[i], q[i], mount_p[i], mount_q[i])
        d, s = cast_rays(o, qrot(qc[None, :], rays), ps, i, max_range)
        depth.append(d.reshape(height, width).astype(np.float32))
        seg.append(s.reshape(height, width))
    return np.stack(depth), np.stack(seg)


def ill_conditioned_pixels(p, q, mount_p, mount_q, ps, width, height, hfov, max_range,
                           envs=None, eps=1e-6):
    """Pixels whose segmentation changes when the ray direction is jittered by
    ~eps rad (silhouette / grazing pixels): a hit-set flip there is a
    conditioning effect, not an arithmetic error.  Returns (n, H, W) bool."""
    rays = pixel_rays(width, height, hfov)
    rng = np.random.default_rng(0)
    envs = range(len(p)) if envs is None else envs
    out = []
    for i in envs:
        o, qc = camera_pose(p[i], q[i], mount_p[i], mount_q[i])
        dw = qrot(qc[None, :], rays)
        _, s0 = cast_rays(o, dw, ps, i, max_range)
        bad = np.zeros(len(rays), bool)
        for _ in range(4):
            j = dw + eps * rng.normal(size=dw.shape)
            j /= np.linalg.norm(j, axis=1, keepdims=True)
            _, s1 = cast_rays(o, j, ps, i, max_range)
            bad |= s1 != s0
        out.append(bad.reshape(height, width))
    return np.stack(out)


# ---- twin of the device obstacle reset (csrc/fs_scene.cuh) -------------------------------

POSE_BLOCK, POSE_EULER, PICK_BLOCK, MOUNT_BLOCK = 0x10000, 0x8000, 0x20000, 0x30000


def _u01d(w):
    return (np.asarray(w, np.uint32) >> np.uint32(8)).astype(np.float64) * 2.0 ** -24


def twin_picks(seed, gid, classes):
    """Prototype id per instance: classes = [(count, pool_first, pool_size)]."""
    picks = []
    j = 0
    for count, first, size in classes:
        for _ in range(count):
            w = R.draw_block(seed, gid, 0, PICK_BLOCK + (j >> 2))[j & 3]
            picks.append(first + int((int(w) * size) >> 32))
            j += 1
    return picks


def twin_poses(seed, gid, counter, class_cfgs, bounds):
    """Instance poses (position (J, 3), quaternion (J, 4)) of one reset.
    class_cfgs: per instance (pos_min, pos_max, euler_min, euler_max, frozen)."""
    b = np.asarray(bounds, np.float64)
    pos, quat = [], []
    for j, (pmin, pmax, emin, emax, frozen) in enumerate(class_cfgs):
        wp = R.draw_block(seed, gid, counter, POSE_BLOCK + j)
        we = R.draw_block(seed, gid, counter, POSE_BLOCK + POSE_EULER + j)
        up, ue = _u01d(wp[:3]), _u01d(we[:3])
        p = (np.asarray(pmin) + up * (np.asarray(pmax) - np.asarray(pmin))) * b
        for i, v in enumerate(frozen):
            if v is not None:
                p[i] = v
        eul = np.asarray(emin) + ue * (np.asarray(emax) - np.asarray(emin))
        pos.append(p)
        quat.append(rot_zyx(eul[0], eul[1], eul[2]))
    return np.array(pos).reshape(-1, 3), np.array(quat).reshape(-1, 4)


def twin_mount(seed, gid, counter, mount_position, mount_euler, rand_position, rand_euler):
    wp = R.draw_block(seed, gid, counter, MOUNT_BLOCK)
    we = R.draw_block(seed, gid, counter, MOUNT_BLOCK + 1)
    dp = (-1.0 + 2.0 * _u01d(wp[:3])) * np.asarray(rand_position)
    de = (-1.0 + 2.0 * _u01d(we[:3])) * np.asarray(rand_euler)
    e = np.asarray(mount_euler) + de
    return np.asarray(mount_position) + dp, rot_zyx(e[0], e[1], e[2])


__all__ = ["aabb", "compile_rows", "signed_distances", "min_distance", "check_collisions",
           "pixel_rays", "ray_prim", "cast_rays", "camera_pose", "render",
           "ill_conditioned_pixels", "twin_picks", "twin_poses", "twin_mount"]
