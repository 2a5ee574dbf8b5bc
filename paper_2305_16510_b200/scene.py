"""Primitive soup on the GPU -- drop-in for ``flocksim.scene``.

``PrimitiveSet`` keeps the reference's per-environment arrays padded to a
common width K (scene.py:24-59) as planar fp32 device memory (the layout of
include/flocksim_b200.h ``fs_scene``): slot k of env e is column e of plane
(f * K + k).  The reference's (E, K, ...) arrays are exposed as views with
the reference shapes.  Distance queries run in the CUDA library
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
FIELDS = N.FS_PRIM_FIELDS                          # dims 3 | pos 3 | rot 9 | lo 3 | hi 3
F_DIM, F_POS, F_ROT, F_LO, F_HI = 0, 3, 6, 15, 18


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
        s = padded(self._e)
        k = max(self._k, 0)
        self._prim = torch.zeros((FIELDS * k, s), dtype=torch.float32, device=self.device)
        rot = self._prim.view(FIELDS, k, s)[F_ROT:F_ROT + 9]
        rot[0].fill_(1.0)
        rot[4].fill_(1.0)
        rot[8].fill_(1.0)
        self._kind = torch.full((k, s), PAD, dtype=torch.int8, device=self.device)
        self._seg = torch.zeros((k, s), dtype=torch.int32, device=self.device)
        self._coll = torch.zeros((k, s), dtype=torch.uint8, device=self.device)

    # -- native descriptor ---------------------------------------------------------
    def native(self) -> N.fs_scene:
        d = N.fs_scene()
        d.num_envs = self._e
        d.width = self._k
        d.prim = ptr(self._prim) if self._k else None
        d.stride = int(self._prim.shape[1])
        d.kind = ptr(self._kind) if self._k else None
        d.seg_id = ptr(self._seg) if self._k else None
        d.collision = ptr(self._coll) if self._k else None
        return d

    @property
    def stride(self) -> int:
        return int(self._prim.shape[1])

    # -- reference surface (scene.py:24-59) -------------------------------------------
    @property
    def num_envs(self) -> int:
        return self._e

    @property
    def width(self) -> int:
        return self._k

    def _fields(self, f0: int, nf: int) -> torch.Tensor:
        return self._prim.view(FIELDS, self._k, self.stride)[f0:f0 + nf, :, :self._e]

    @property
    def kind(self) -> torch.Tensor:
        return self._kind[:, :self._e].T

    @property
    def dims(self) -> torch.Tensor:
        return self._fields(F_DIM, 3).permute(2, 1, 0)

    @property
    def position(self) -> torch.Tensor:
        return self._fields(F_POS, 3).permute(2, 1, 0)

    @property
    def rot(self) -> torch.Tensor:
        return self._fields(F_ROT, 9).reshape(3, 3, self._k, self._e).permute(3, 2, 0, 1)

    @property
    def seg_id(self) -> torch.Tensor:
        return self._seg[:, :self._e].T

    @property
    def collision(self) -> torch.Tensor:
        return self._coll[:, :self._e].T.bool()

    @property
    def aabb_min(self) -> torch.Tensor:
        return self._fields(F_LO, 3).permute(2, 1, 0)

    @property
    def aabb_max(self) -> torch.Tensor:
        return self._fields(F_HI, 3).permute(2, 1, 0)

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
        if self._k == 0:
            return
        self._prim[:, e].copy_(other._prim[:, src])
        self._kind[:, e].copy_(other._kind[:, src])
        self._seg[:, e].copy_(other._seg[:, src])
        self._coll[:, e].copy_(other._coll[:, src])

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
        host = np.zeros((FIELDS, k, e), dtype=np.float32)
        host[F_DIM:F_DIM + 3] = dims.transpose(2, 1, 0)
        host[F_POS:F_POS + 3] = position.transpose(2, 1, 0)
        host[F_ROT:F_ROT + 9] = rot.reshape(e, k, 9).transpose(2, 1, 0)
        host[F_LO:F_LO + 3] = _round_down(np.asarray(aabb_min, np.float64)).transpose(2, 1, 0)
        host[F_HI:F_HI + 3] = _round_up(np.asarray(aabb_max, np.float64)).transpose(2, 1, 0)
        if k == 0:
            return self
        self._prim.view(FIELDS, k, self.stride)[:, :, :e].copy_(torch.from_numpy(host))
        self._kind[:, :e].copy_(torch.from_numpy(kind.astype(np.int8).T.copy()))
        self._seg[:, :e].copy_(torch.from_numpy(np.asarray(seg_id, np.int32).reshape(e, k).T.copy()))
        self._coll[:, :e].copy_(torch.from_numpy(
            np.asarray(collision, bool).reshape(e, k).T.astype(np.uint8).copy()))
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
    buf = torch.zeros((3, pset.stride), dtype=torch.float32, device=pset.device)
    buf[:, :pset.num_envs].copy_(t.T)
    return buf


def _distances(pset: PrimitiveSet, points, collision_only: bool, want_all: bool):
    lib = N.load()
    e, k = pset.num_envs, pset.width
    pts = _points(pset, points)
    dist = (torch.empty((max(k, 1), pset.stride), dtype=torch.float64, device=pset.device)
            if want_all else None)
    mins = torch.empty(max(e, 1), dtype=torch.float64, device=pset.device)
    desc = pset.native()
    with torch.cuda.device(pset.device):
        N.check(lib.fs_scene_distances(C.byref(desc), ptr(pts), pts.stride(0),
                                       1 if collision_only else 0, ptr(dist),
                                       pset.stride if want_all else 0, ptr(mins),
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
