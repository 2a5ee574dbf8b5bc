"""Per-robot depth + segmentation cameras -- drop-in for ``flocksim.camera``.

SURVEY.md 8(f) rank 4.  Pinhole cameras with square pixels, +z optical axis,
+x right, +y down (camera.py:1-11); depth is the Euclidean range along the
ray, max_range (and segmentation 0) where nothing is hit within range.

``render`` runs the sm_100a ray caster (``fs_render``, csrc/fs_scene.cu):
one CTA per (env, run of 32x16-pixel tiles), the env's primitives staged in
shared memory, culled per tile against the tile's view cone, and every ray
intersected in float64 with the reference's arithmetic
(camera.py:132-227).  Images are (N, H, W) device tensors: float32 depth,
int32 segmentation.  ``workers`` is accepted and ignored (results never
depend on partitioning, camera.py:9-11).
"""

from __future__ import annotations

import ctypes as C
import math
import struct
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np
import torch

from . import _native as N
from . import _se3
from ._tensors import padded, ptr, stream_handle
from .scene import KIND_CODES, PrimitiveSet

FORWARD_MOUNT_EULER = (-math.pi / 2, 0.0, -math.pi / 2)     # camera.py:29
MAGIC = b"FSDEPTH1"
DTYPE_F32_I32 = 1


class CameraDisabledError(RuntimeError):
    """Rendering was requested but no camera is configured (camera.py:35-36)."""


def _vec(x, n):
    return np.asarray(x, dtype=np.float64).reshape(n)


@dataclass
class CameraConfig:
    """Pinhole intrinsics and body-frame mount (camera.py:39-69)."""

    width: int = 480
    height: int = 270
    hfov: float = 1.57
    max_range: float = 10.0
    mount_position: np.ndarray = field(default_factory=lambda: np.zeros(3))
    mount_euler: np.ndarray = field(default_factory=lambda: np.array(FORWARD_MOUNT_EULER))
    randomize_position: np.ndarray = field(default_factory=lambda: np.zeros(3))
    randomize_euler: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        self.mount_position = _vec(self.mount_position, 3)
        self.mount_euler = _vec(self.mount_euler, 3)
        self.randomize_position = _vec(self.randomize_position, 3)
        self.randomize_euler = _vec(self.randomize_euler, 3)
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be at least 1x1")
        if not 0.0 < self.hfov < math.pi:
            raise ValueError("hfov must lie in (0, pi)")
        if self.max_range <= 0.0:
            raise ValueError("max_range must be positive")

    @property
    def mount_rotation(self) -> np.ndarray:
        return _se3.rot_zyx(*self.mount_euler)

    def native(self) -> N.fs_camera:
        c = N.fs_camera()
        c.width, c.height = int(self.width), int(self.height)
        c.pixel_scale = 2.0 * math.tan(self.hfov / 2.0) / self.width
        c.max_range = float(self.max_range)
        c.mount_position[:] = [float(x) for x in self.mount_position]
        c.mount_rotation[:] = [float(x) for x in self.mount_rotation]
        return c


@dataclass
class DepthImageBatch:
    """Rendered depth (m, float32) and segmentation ids (int32), (N, H, W)."""

    depth: torch.Tensor
    segmentation: torch.Tensor
    max_range: float

    @property
    def n(self) -> int:
        return int(self.depth.shape[0])

    def write_binary(self, path) -> None:
        """magic, u32 N/height/width/dtype, float32 depth, int32 segmentation,
        little-endian, row-major (camera.py:85-97)."""
        n, h, w = self.depth.shape
        depth = np.ascontiguousarray(_host(self.depth), dtype="<f4")
        seg = np.ascontiguousarray(_host(self.segmentation), dtype="<i4")
        with open(path, "wb") as f:
            f.write(MAGIC)
            f.write(struct.pack("<4I", n, h, w, DTYPE_F32_I32))
            f.write(depth.tobytes())
            f.write(seg.tobytes())

    @classmethod
    def read_binary(cls, path, max_range: float = 0.0) -> "DepthImageBatch":
        with open(path, "rb") as f:
            if f.read(8) != MAGIC:
                raise ValueError(f"{path}: not a depth dump")
            n, h, w, code = struct.unpack("<4I", f.read(16))
            if code != DTYPE_F32_I32:
                raise ValueError(f"{path}: unknown dtype code {code}")
            depth = np.frombuffer(f.read(n * h * w * 4), dtype="<f4").reshape(n, h, w)
            seg = np.frombuffer(f.read(n * h * w * 4), dtype="<i4").reshape(n, h, w)
        return cls(depth=torch.from_numpy(depth.copy()), segmentation=torch.from_numpy(seg.copy()),
                   max_range=max_range)

    def write_png(self, index: int, path) -> None:
        """16-bit grayscale export of one frame (camera.py:112-119)."""
        from PIL import Image

        scale = 65535.0 / self.max_range if self.max_range > 0 else 1.0
        img = np.clip(_host(self.depth[index]) * scale, 0, 65535).astype(np.uint16)
        Image.fromarray(img).save(path)


def _host(t) -> np.ndarray:
    return t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@lru_cache(maxsize=8)
def _pixel_rays(width: int, height: int, hfov: float) -> np.ndarray:
    """Unit camera-frame ray per pixel, (H*W, 3) row-major (camera.py:122-130);
    the kernel evaluates the same expression per pixel."""
    scale = 2.0 * math.tan(hfov / 2.0) / width
    u = (np.arange(width) + 0.5 - width / 2.0) * scale
    v = (np.arange(height) + 0.5 - height / 2.0) * scale
    xs, ys = np.meshgrid(u, v)
    d = np.stack([xs.ravel(), ys.ravel(), np.ones(width * height)], axis=-1)
    out = d / np.sqrt((d * d).sum(axis=1))[:, None]
    out.setflags(write=False)
    return out


def randomize_mount(cfg: CameraConfig, rng: np.random.Generator):
    """A mount pose uniform within the configured +- bounds (camera.py:238-244).
    Host-side helper; the GPU World draws its mounts on the device."""
    dp = rng.uniform(-1.0, 1.0, size=3) * cfg.randomize_position
    de = rng.uniform(-1.0, 1.0, size=3) * cfg.randomize_euler
    e = cfg.mount_euler + de
    return cfg.mount_position + dp, _se3.rot_zyx(e[0], e[1], e[2])


def cast_rays(origin, dirs, pset: PrimitiveSet, env_index: int, max_range: float):
    """Nearest collision-enabled hit per ray within one env (camera.py:230-282).
    Returns (depth (M,) float64, seg (M,) int32) device tensors."""
    lib = N.load()
    o = [float(x) for x in np.asarray(_host(origin), dtype=np.float64).reshape(3)]
    d = dirs if isinstance(dirs, torch.Tensor) else torch.as_tensor(np.asarray(dirs))
    d = d.to(device=pset.device, dtype=torch.float64).reshape(-1, 3).contiguous()
    m = int(d.shape[0])
    depth = torch.empty(max(m, 1), dtype=torch.float64, device=pset.device)
    seg = torch.empty(max(m, 1), dtype=torch.int32, device=pset.device)
    desc = pset.native()
    with torch.cuda.device(pset.device):
        N.check(lib.fs_cast_rays(C.byref(desc), int(env_index), o[0], o[1], o[2], ptr(d), m,
                                 float(max_range), ptr(depth), ptr(seg), stream_handle()),
                "fs_cast_rays")
    return depth[:m], seg[:m]


def ray_primitive(origin, direction, prim, seg_id: int = 0, max_range: float = np.inf):
    """Smallest positive hit of one ray on one primitive, tangential grazes
    counting as hits (camera.py:285-303).  Returns (t, seg_id) or None."""
    origin = np.asarray(origin, dtype=np.float64)
    direction = np.asarray(direction, dtype=np.float64)
    if abs(float(np.linalg.norm(direction)) - 1.0) > 1e-9:
        raise ValueError("ray direction must be a unit vector")
    pset = PrimitiveSet(1, 1)
    pset.load_arrays([[KIND_CODES[prim.kind]]], [[prim.dims]], [[prim.position]],
                     [[_se3.quat_to_matrix(prim.rotation)]], [[seg_id]], [[True]])
    depth, seg = cast_rays(origin, direction[None, :], pset, 0, np.inf)
    t = float(depth[0])
    if not math.isfinite(t) or t > max_range:
        return None
    return t, seg_id


def _mount_planes(world, cfg: CameraConfig, device):
    """(7, stride) float64 mount planes for `world`, or None for the nominal
    mount of cfg (World.camera_mounts, world.py:355-361)."""
    planes = getattr(world, "mount_planes", None)
    if callable(planes):
        got = planes(cfg)
        if got is not None:
            return got
    mp, mq = world.camera_mounts(cfg)
    mp = np.asarray(_host(mp), dtype=np.float64)
    mq = np.asarray(_host(mq), dtype=np.float64)
    if np.array_equal(mp, np.broadcast_to(cfg.mount_position, mp.shape)) and np.array_equal(
            mq, np.broadcast_to(cfg.mount_rotation, mq.shape)):
        return None
    n = mp.shape[0]
    buf = torch.zeros((7, padded(n)), dtype=torch.float64, device=device)
    buf[0:3, :n].copy_(torch.from_numpy(mp.T.copy()))
    buf[3:7, :n].copy_(torch.from_numpy(mq.T.copy()))
    return buf


def render(world, cam_cfg: CameraConfig | None = None, workers: int = 1,
           out: DepthImageBatch | None = None, envs: tuple | None = None) -> DepthImageBatch:
    """Render every robot's depth and segmentation image (camera.py:306-335).

    The camera sits at p + R(q) mount_p with orientation q (x) mount_q;
    mounts are the world's randomized ones when cam_cfg is world.camera.
    ``out`` (optional) is a preallocated batch of the right shape to render
    into (no allocation, CUDA-graph friendly); ``envs`` (optional) = (first,
    count) renders only that range of envs into out's images of the same
    indices (on the current stream; lets a caller pipeline read-back).
    """
    cfg = cam_cfg if cam_cfg is not None else world.camera
    if cfg is None:
        raise CameraDisabledError("world has no camera configured")
    lib = N.load()
    pset: PrimitiveSet = world.pset
    states = world.states
    n = int(states.n)
    device = pset.device
    if out is None:
        out = DepthImageBatch(
            depth=torch.empty((n, cfg.height, cfg.width), dtype=torch.float32, device=device),
            segmentation=torch.empty((n, cfg.height, cfg.width), dtype=torch.int32,
                                     device=device),
            max_range=float(cfg.max_range))
    if n == 0:
        return out
    mount = _mount_planes(world, cfg, device)
    buf = states.buf
    desc = pset.native()
    cam = cfg.native()
    lo, hi = (0, n) if envs is None else (int(envs[0]), int(envs[0]) + int(envs[1]))
    if not 0 <= lo <= hi <= n:
        raise ValueError(f"env range {envs} outside [0, {n})")
    with torch.cuda.device(device):
        for first in range(lo, hi, 65535):
            cnt = min(65535, hi - first)
            N.check(lib.fs_render(C.byref(desc), C.byref(cam), ptr(buf), buf.stride(0),
                                  ptr(mount), 0 if mount is None else mount.stride(0), first,
                                  cnt, ptr(out.depth[first]), ptr(out.segmentation[first]),
                                  stream_handle()), "fs_render")
    return out


__all__ = ["CameraConfig", "CameraDisabledError", "DepthImageBatch", "FORWARD_MOUNT_EULER",
           "cast_rays", "randomize_mount", "ray_primitive", "render"]
