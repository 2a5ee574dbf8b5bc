"""Primitive soup on the GPU -- drop-in for ``flocksim.scene``.

``PrimitiveSet`` keeps the reference's per-environment arrays padded to a
common width K (scene.py:24-59) as fp32 device memory in the layout of
include/flocksim_b200.h ``fs_scene``: one 96-byte record per (env, slot),
``[lo xyz, kind] [hi xyz, collision] [dims xyz, seg_id] [pos xyz, R22]
[R00 R01 R02 R10] [R11 R12 R20 R21]`` (ints as bit patterns).  The
reference's (E, K, ...) arrays are exposed with the reference shapes (views
where the record layout allows; rot, kind and collision are converted
copies).  Distance queries run in the CUDA library
(``fs_scene_distances``): float64 arithmetic on the stored fp32 values,
restating scene.py:127-181.  AABBs are stored rounded outward, so they stay
conservative after the fp32 store.

``compile_instances`` flattens explicit instance lists on the host
(float64, scene.py:76-124) and uploads them; the GPU World compiles its own
rows on the device at every reset (csrc/fs_scene.cuh ``rebuild_env``).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from . import _se3
from ._tensors import default_device, padded, ptr, stream_handle
from .assets import BOX, CYLINDER, SPHERE

KIND_CODES = {BOX: 0, CYLINDER: 1, SPHERE: 2}      # scene.py:20
PAD = -1                                          # scene.py:21
FIELDS = N.FS_PRIM_FIELDS                          # 24 floats per record
F_LO, F_KIND, F_HI, F_COLL, F_DIM, F_SEG, F_POS = 0, 3, 4, 7, 8, 11, 12
# record index of R[i][j] (row-major)
F_ROT = (16, 17, 18, 19, 20, 21, 22, 23, 15)


class PrimitiveSet:
    """Per-environment primitive soup padded to width K, on the device.

    Attributes (views, reference shapes): kind (E, K) int8, dims (E, K, 3),
    position (E, K, 3), rot (E, K, 3, 3), seg_id (E, K) int32, collision
    (E, K) bool, aabb_min / aabb_max (E, K, 3).  Geometry is float32.
    """

    def __init__(self, num_envs: int, width: int, device=None):
        self.device = device if device is not None else default_device()
        self._e = int(num_envs)
        self._k = int(width)
        self._rec = torch.zeros((max(self._e, 1), max(self._k, 0), FIELDS), dtype=torch.float32,
                                device=self.device)
        if self._k:
            self._rec[:, :, F_ROT[0]] = 1.0
            self._rec[:, :, F_ROT[4]] = 1.0
            self._rec[:, :, F_ROT[8]] = 1.0
            self._ints[:, :, F_KIND] = PAD

    @property
    def _ints(self) -> torch.Tensor:
        return self._rec.view(torch.int32)

    # -- native descriptor ---------------------------------------------------------
    def native(self) -> N.fs_scene:
        d = N.fs_scene()
        d.num_envs = self._e
        d.width = self._k
        d.rec = ptr(self._rec) if self._k else None
        return d

    # -- reference surface (scene.py:24-59) -------------------------------------------
    @property
    def num_envs(self) -> int:
        return self._e

    @property
    def width(self) -> int:
        return self._k

    @property
    def kind(self) -> torch.Tensor:
        return self._ints[:self._e, :, F_KIND].to(torch.int8)

    @property
    def dims(self) -> torch.Tensor:
        return self._rec[:self._e, :, F_DIM:F_DIM + 3]

    @property
    def position(self) -> torch.Tensor:
        return self._rec[:self._e, :, F_POS:F_POS + 3]

    @property
    def rot(self) -> torch.Tensor:
        return self._rec[:self._e][:, :, list(F_ROT)].reshape(self._e, self._k, 3, 3)

    @property
    def seg_id(self) -> torch.Tensor:
        return self._ints[:self._e, :, F_SEG]

    @property
    def collision(self) -> torch.Tensor:
        return self._ints[:self._e, :, F_COLL] != 0

    @property
    def aabb_min(self) -> torch.Tensor:
        return self._rec[:self._e, :, F_LO:F_LO + 3]

    @property
    def aabb_max(self) -> torch.Tensor:
        return self._rec[:self._e, :, F_HI:F_HI + 3]

    def env_view(self, e: int) -> "PrimitiveSet":
        """Environment e as a 1-env set (a copy on the device)."""
        if not 0 <= e < self._e:
            raise IndexError(f"env index {e} out of range")
        out = PrimitiveSet(1, self._k, self.device)
        out._copy_env(0, self, e)
        return out

    def write_env(self, e: int, other: "PrimitiveSet") -> None:
        """Overwrite env e's rows from a 1-env set of equal width (scene.py:50-59)."""
        if other.width != self.width or other.num_envs != 1:
            raise ValueError("environment row shape mismatch")
        self._copy_env(e, other, 0)

    def _copy_env(self, e: int, other: "PrimitiveSet", src: int) -> None:
        if self._k:
            self._rec[e].copy_(other._rec[src])

    def load_arrays(self, kind, dims, position, rot, seg_id, collision, aabb_min=None,
                    aabb_max=None) -> "PrimitiveSet":
        """Upload host (E, K, ...) float64 arrays (e.g. a reference PrimitiveSet).
        Geometry rounds to nearest fp32; a given AABB rounds outward, a missing
        one is recomputed (scene.py:62-73)."""
        e, k = self._e, self._k
        kind = np.asarray(kind).reshape(e, k)
        dims = np.asarray(dims, np.float64).reshape(e, k, 3)
        position = np.asarray(position, np.float64).reshape(e, k, 3)
        rot = np.asarray(rot, np.float64).reshape(e, k, 3, 3)
        if aabb_min is None or aabb_max is None:
            aabb_min, aabb_max = _aabb(kind, dims, position, rot)
        host = np.zeros((e, k, FIELDS), dtype=np.float32)
        ints = host.view(np.int32)
        host[:, :, F_LO:F_LO + 3] = _round_down(np.asarray(aabb_min, np.float64).reshape(e, k, 3))
        host[:, :, F_HI:F_HI + 3] = _round_up(np.asarray(aabb_max, np.float64).reshape(e, k, 3))
        host[:, :, F_DIM:F_DIM + 3] = dims
        host[:, :, F_POS:F_POS + 3] = position
        host[:, :, list(F_ROT)] = rot.reshape(e, k, 9)
        ints[:, :, F_KIND] = kind.astype(np.int32)
        ints[:, :, F_SEG] = np.asarray(seg_id, np.int32).reshape(e, k)
        ints[:, :, F_COLL] = np.asarray(collision, bool).reshape(e, k).astype(np.int32)
        if k:
            self._rec[:e].copy_(torch.from_numpy(host))
        return self

    def to_numpy(self) -> dict:
        """Host copies of every array (float64 geometry), reference shapes."""
        return {"kind": self.kind.cpu().numpy(), "dims": self.dims.double().cpu().numpy(),
                "position": self.position.double().cpu().numpy(),
                "rot": self.rot.double().cpu().numpy(), "seg_id": self.seg_id.cpu().numpy(),
                "collision": self.collision.cpu().numpy(),
                "aabb_min": self.aabb_min.double().cpu().numpy(),
                "aabb_max": self.aabb_max.double().cpu().numpy()}


def _round_down(x: np.ndarray) -> np.ndarray:
    f = x.astype(np.float32)
    return np.where(f.astype(np.float64) > x, np.nextafter(f, np.float32(-np.inf)), f)


def _round_up(x: np.ndarray) -> np.ndarray:
    f = x.astype(np.float32)
    return np.where(f.astype(np.float64) < x, np.nextafter(f, np.float32(np.inf)), f)


def _aabb(kind, dims, position, rot):
    """Conservative env-frame AABBs (scene.py:62-73), vectorized, float64."""
    half_box = np.abs(rot) @ (dims / 2.0)[..., None]
    half_box = half_box[..., 0]
    axis = rot[..., :, 2]
    half_cyl = np.abs(axis) * (dims[..., 1:2] / 2.0) + dims[..., 0:1] * np.sqrt(
        np.maximum(0.0, 1.0 - axis * axis))
    half_sph = np.repeat(dims[..., 0:1], 3, axis=-1)
    k = np.asarray(kind)[..., None]
    half = np.where(k == 0, half_box, np.where(k == 1, half_cyl, half_sph))
    return position - half, position + half


def compile_instances(instances_per_env: list, width: int | None = None,
                      device=None) -> PrimitiveSet:
    """Flatten per-env asset instances into a padded device PrimitiveSet
    (scene.py:76-124): every primitive posed by its instance, in instance
    order; width defaults to the widest environment."""
    rows = []
    for env in instances_per_env:
        row = []
        for inst in env:
            for prim in inst.prototype.primitives:
                pos = inst.position + _se3.quat_rotate(inst.rotation, prim.position)
                q = _se3.quat_multiply(inst.rotation, prim.rotation)
                row.append((KIND_CODES[prim.kind], prim.dims, pos, _se3.quat_to_matrix(q),
                            inst.segmentation_id, inst.collision_enabled))
        rows.append(row)
    widest = max((len(r) for r in rows), default=0)
    k = widest if width is None else int(width)
    if widest > k:
        raise ValueError("width smaller than an environment's primitive count")
    e = len(rows)
    kind = np.full((e, k), PAD, dtype=np.int8)
    dims = np.zeros((e, k, 3))
    position = np.zeros((e, k, 3))
    rot = np.broadcast_to(np.eye(3), (e, k, 3, 3)).copy()
    seg = np.zeros((e, k), dtype=np.int32)
    coll = np.zeros((e, k), dtype=bool)
    for ei, row in enumerate(rows):
        for ki, (code, d, p, r, sg, cl) in enumerate(row):
            kind[ei, ki], dims[ei, ki], position[ei, ki], rot[ei, ki] = code, d, p, r
            seg[ei, ki], coll[ei, ki] = sg, cl
    lo, hi = _aabb(kind, dims, position, rot)
    pad = kind == PAD
    lo[pad] = 0.0
    hi[pad] = 0.0
    return PrimitiveSet(e, k, device).load_arrays(kind, dims, position, rot, seg, coll, lo, hi)


def _points(pset: PrimitiveSet, points) -> torch.Tensor:
    """(E, 3) points -> (3, stride) fp32 planes on the set's device."""
    t = points if isinstance(points, torch.Tensor) else torch.as_tensor(np.asarray(points))
    t = t.to(device=pset.device, dtype=torch.float32).reshape(-1, 3)
    if t.shape[0] != pset.num_envs:
        raise ValueError(f"expected {pset.num_envs} points, got {t.shape[0]}")
    buf = torch.zeros((3, padded(pset.num_envs)), dtype=torch.float32, device=pset.device)
    buf[:, :pset.num_envs].copy_(t.T)
    return buf


def _distances(pset: PrimitiveSet, points, collision_only: bool, want_all: bool):
    lib = N.load()
    e, k = pset.num_envs, pset.width
    pts = _points(pset, points)
    dist = (torch.empty((max(k, 1), padded(e)), dtype=torch.float64, device=pset.device)
            if want_all else None)
    mins = torch.empty(max(e, 1), dtype=torch.float64, device=pset.device)
    desc = pset.native()
    with torch.cuda.device(pset.device):
        N.check(lib.fs_scene_distances(C.byref(desc), ptr(pts), pts.stride(0),
                                       1 if collision_only else 0, ptr(dist),
                                       padded(e) if want_all else 0, ptr(mins),
                                       stream_handle()), "fs_scene_distances")
    return dist, mins


def signed_distances(pset: PrimitiveSet, points) -> torch.Tensor:
    """(E, K) float64 signed distance of each env's point to each of its
    primitives, +inf on pads, negative inside (scene.py:127-165)."""
    if pset.width == 0:
        return torch.full((pset.num_envs, 0), float("inf"), dtype=torch.float64,
                          device=pset.device)
    dist, _ = _distances(pset, points, False, True)
    return dist[:pset.width, :pset.num_envs].T


def min_distance(pset: PrimitiveSet, points, collision_only: bool = True) -> torch.Tensor:
    """Smallest signed distance per env; +inf with no (collision) primitives
    (scene.py:168-181)."""
    _, mins = _distances(pset, points, collision_only, False)
    return mins[:pset.num_envs]


__all__ = ["KIND_CODES", "PAD", "PrimitiveSet", "compile_instances", "signed_distances",
           "min_distance"]
