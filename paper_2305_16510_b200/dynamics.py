"""Batched rigid-body dynamics on B200 -- drop-in for ``flocksim.dynamics``.

Mirrors /root/reference/pkg/src/flocksim/dynamics.py: the same names,
argument meaning, validation and exception types.  Differences by design:

* arrays are float32 CUDA tensors in a planar layout (see ``_tensors``);
  every per-vehicle computation runs in the CUDA kernels of
  ``lib/libflocksim_b200.so`` -- there is no CPU fallback;
* ``workers`` is accepted for signature compatibility; results never depend
  on partitioning (dynamics.py:18-19), so it is ignored.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._tensors import (alloc_planes, as_device, default_device, pack_rows, ptr, stride0,
                       stream_handle)

DEFAULT_GRAVITY = 9.81          # dynamics.py:31
GIMBAL_TOL = 1e-6               # se3.py:25


class NonFiniteStateError(RuntimeError):
    """Raised by the scalar step when the integrated state is non-finite
    (dynamics.py:34-35)."""


@dataclass
class RobotParams:
    """Physical parameters shared by every robot in a batch (dynamics.py:38-90)."""

    mass: float = 1.0
    inertia: np.ndarray = field(default_factory=lambda: np.diag([0.01, 0.01, 0.02]))
    collision_radius: float = 0.2
    thrust_max: float = 25.0
    moment_max: np.ndarray = field(default_factory=lambda: np.array([2.0, 2.0, 1.0]))
    gravity: float = DEFAULT_GRAVITY
    v_limit: float = 50.0
    omega_limit: float = 100.0

    def __post_init__(self):
        self.inertia = np.asarray(self.inertia, dtype=np.float64)
        self.moment_max = np.asarray(self.moment_max, dtype=np.float64)
        if self.mass <= 0.0:
            raise ValueError(f"mass must be positive, got {self.mass}")
        if self.inertia.shape != (3, 3):
            raise ValueError("inertia must be a 3x3 matrix")
        if np.abs(self.inertia - self.inertia.T).max() > 1e-12:
            raise ValueError("inertia matrix must be symmetric")
        if np.linalg.eigvalsh(self.inertia).min() <= 0.0:
            raise ValueError("inertia matrix must be positive definite")
        if self.thrust_max <= self.mass * self.gravity:
            raise ValueError(f"thrust_max {self.thrust_max} does not exceed hover thrust "
                             f"{self.mass * self.gravity}")
        if (self.moment_max <= 0.0).any():
            raise ValueError("moment_max components must be positive")
        self._inertia_inv = np.linalg.inv(self.inertia)

    @property
    def inertia_inv(self) -> np.ndarray:
        return self._inertia_inv

    @property
    def hover_thrust(self) -> float:
        return self.mass * self.gravity

    def native(self) -> N.fs_robot:
        r = N.fs_robot()
        r.mass = self.mass
        r.gravity = self.gravity
        r.inertia[:] = [float(x) for x in self.inertia.reshape(-1)]
        r.inertia_inv[:] = [float(x) for x in self._inertia_inv.reshape(-1)]
        r.thrust_max = self.thrust_max
        r.moment_max[:] = [float(x) for x in self.moment_max]
        r.v_limit = self.v_limit
        r.omega_limit = self.omega_limit
        r.gimbal_cos = math.cos(GIMBAL_TOL)
        return r


# =============================================================================
# state containers
# =============================================================================

class _Planar:
    """Common plumbing of planar (k, stride) device records."""

    K = 0

    def _init_buf(self, n, device):
        self.buf = alloc_planes(self.K, n, device)
        self._n = int(n)

    @property
    def n(self) -> int:
        return self._n

    @property
    def stride(self) -> int:
        return stride0(self.buf)

    @property
    def device(self) -> torch.device:
        return self.buf.device


@dataclass
class RigidState:
    """One robot: p (3,), q (4,) scalar-first body->world, v (3,), omega (3,)
    (dynamics.py:93-117).  Host-side float64 values."""

    p: np.ndarray
    q: np.ndarray
    v: np.ndarray
    omega: np.ndarray

    def __post_init__(self):
        self.p = np.asarray(_host(self.p), dtype=np.float64).reshape(3)
        self.q = np.asarray(_host(self.q), dtype=np.float64).reshape(4)
        self.v = np.asarray(_host(self.v), dtype=np.float64).reshape(3)
        self.omega = np.asarray(_host(self.omega), dtype=np.float64).reshape(3)

    @classmethod
    def rest(cls, p=(0.0, 0.0, 0.0)) -> "RigidState":
        return cls(p=np.array(p), q=np.array([1.0, 0.0, 0.0, 0.0]), v=np.zeros(3),
                   omega=np.zeros(3))


def _host(x):
    if isinstance(x, torch.Tensor):
        return x.detach().cpu().numpy()
    return x


class RigidStateBatch(_Planar):
    """Structure-of-arrays state for N robots (dynamics.py:119-165), stored as
    13 fp32 planes ``px py pz qw qx qy qz vx vy vz wx wy wz`` on the GPU."""

    K = 13

    def __init__(self, p, q, v, omega, device=None):
        device = device if device is not None else (
            p.device if isinstance(p, torch.Tensor) and p.is_cuda else default_device())
        n = int(np.shape(p)[0]) if not isinstance(p, torch.Tensor) else int(p.shape[0])
        self._init_buf(n, device)
        pack_rows(self.buf, 0, p, n, 3)
        pack_rows(self.buf, 3, q, n, 4)
        pack_rows(self.buf, 7, v, n, 3)
        pack_rows(self.buf, 10, omega, n, 3)

    @classmethod
    def from_planes(cls, buf: torch.Tensor, n: int) -> "RigidStateBatch":
        """Wrap an existing (13, stride) fp32 CUDA buffer (no copy)."""
        if buf.dim() != 2 or buf.shape[0] != 13 or buf.dtype != torch.float32 or not buf.is_cuda:
            raise ValueError("expected a (13, stride) float32 CUDA tensor")
        if buf.stride(1) != 1 or buf.shape[1] < n:
            raise ValueError("planes must be contiguous along vehicles and hold n entries")
        obj = cls.__new__(cls)
        obj.buf = buf
        obj._n = int(n)
        return obj

    @classmethod
    def empty(cls, n: int, device=None) -> "RigidStateBatch":
        obj = cls.__new__(cls)
        obj._init_buf(n, device)
        return obj

    @classmethod
    def rest(cls, n: int, p=None, device=None) -> "RigidStateBatch":
        """Level, motionless batch, optionally at given positions (dynamics.py:134-142)."""
        obj = cls.empty(n, device)
        obj.buf.zero_()
        obj.buf[3, :n] = 1.0
        if p is not None:
            pack_rows(obj.buf, 0, p, n, 3)
        return obj

    @classmethod
    def from_states(cls, states) -> "RigidStateBatch":
        return cls(p=np.stack([s.p for s in states]), q=np.stack([s.q for s in states]),
                   v=np.stack([s.v for s in states]), omega=np.stack([s.omega for s in states]))

    @property
    def p(self) -> torch.Tensor:
        return self.buf[0:3, :self._n].T

    @property
    def q(self) -> torch.Tensor:
        return self.buf[3:7, :self._n].T

    @property
    def v(self) -> torch.Tensor:
        return self.buf[7:10, :self._n].T

    @property
    def omega(self) -> torch.Tensor:
        return self.buf[10:13, :self._n].T

    def planes(self) -> torch.Tensor:
        return self.buf[:, :self._n]

    def at(self, i: int) -> RigidState:
        col = self.buf[:, i].double().cpu().numpy()
        return RigidState(p=col[0:3], q=col[3:7], v=col[7:10], omega=col[10:13])

    def copy(self) -> "RigidStateBatch":
        return RigidStateBatch.from_planes(self.buf.clone(), self._n)

    def slice(self, sl: slice) -> "RigidStateBatch":
        """A view of rows `sl` (dynamics.py:163-165); step=1 slices only."""
        start, stop, step = sl.indices(self._n)
        if step != 1:
            raise ValueError("only contiguous slices are supported")
        obj = RigidStateBatch.__new__(RigidStateBatch)
        obj.buf = self.buf[:, start:stop] if stop > start else self.buf[:, 0:0]
        obj._n = max(0, stop - start)
        return obj

    def numpy(self) -> np.ndarray:
        """(13, n) float64 host copy in the planar layout."""
        return self.buf[:, :self._n].double().cpu().numpy()


@dataclass
class Wrench:
    """Collective thrust (N, along +b3) and body moment (N m) for one robot."""

    thrust: float
    moment: np.ndarray

    def __post_init__(self):
        self.thrust = float(self.thrust)
        self.moment = np.asarray(_host(self.moment), dtype=np.float64).reshape(3)


class WrenchBatch(_Planar):
    """thrust (N,) and moment (N, 3) as 4 fp32 planes (dynamics.py:179-200)."""

    K = 4

    def __init__(self, thrust, moment, device=None):
        device = device if device is not None else (
            thrust.device if isinstance(thrust, torch.Tensor) and thrust.is_cuda
            else default_device())
        t = as_device(thrust, device).reshape(-1)
        self._init_buf(t.shape[0], device)
        self.buf[0, :self._n].copy_(t)
        pack_rows(self.buf, 1, moment, self._n, 3)

    @classmethod
    def empty(cls, n: int, device=None) -> "WrenchBatch":
        obj = cls.__new__(cls)
        obj._init_buf(n, device)
        return obj

    @classmethod
    def zeros(cls, n: int, device=None) -> "WrenchBatch":
        obj = cls.empty(n, device)
        obj.buf.zero_()
        return obj

    @property
    def thrust(self) -> torch.Tensor:
        return self.buf[0, :self._n]

    @property
    def moment(self) -> torch.Tensor:
        return self.buf[1:4, :self._n].T

    def at(self, i: int) -> Wrench:
        col = self.buf[:, i].double().cpu().numpy()
        return Wrench(thrust=col[0], moment=col[1:4])

    def slice(self, sl: slice) -> "WrenchBatch":
        start, stop, step = sl.indices(self._n)
        if step != 1:
            raise ValueError("only contiguous slices are supported")
        obj = WrenchBatch.__new__(WrenchBatch)
        obj.buf = self.buf[:, start:stop]
        obj._n = max(0, stop - start)
        return obj


@dataclass
class StepFlags:
    """Per-robot diagnostics from one integration step (dynamics.py:203-211)."""

    clamped: torch.Tensor      # (N,) bool: velocity or rate hit its hard limit
    nonfinite: torch.Tensor    # (N,) bool: state went non-finite, caller resets

    def slice(self, sl: slice) -> "StepFlags":
        return StepFlags(clamped=self.clamped[sl], nonfinite=self.nonfinite[sl])

    @classmethod
    def from_bits(cls, bits: torch.Tensor) -> "StepFlags":
        return cls(clamped=(bits & N.FS_FLAG_CLAMPED) != 0,
                   nonfinite=(bits & N.FS_FLAG_NONFINITE) != 0)


# =============================================================================
# operations
# =============================================================================

def saturate_batch(wrench: WrenchBatch, params: RobotParams) -> WrenchBatch:
    """Clamp thrust to [0, thrust_max] and moments to +-moment_max (dynamics.py:214-218)."""
    lib = N.load()
    out = WrenchBatch.empty(wrench.n, wrench.device)
    r = params.native()
    with torch.cuda.device(wrench.device):
        N.check(lib.fs_saturate(wrench.n, ptr(wrench.buf), wrench.stride, r, ptr(out.buf),
                                out.stride, stream_handle()), "saturate_batch")
    return out


def saturate(wrench: Wrench, params: RobotParams) -> Wrench:
    """Scalar form of saturate_batch (dynamics.py:221-226)."""
    return saturate_batch(WrenchBatch(thrust=[wrench.thrust], moment=wrench.moment[None, :]),
                          params).at(0)


def step_batch(states: RigidStateBatch, params: RobotParams, wrenches: WrenchBatch,
               dt: float, workers: int = 1, out: RigidStateBatch | None = None
               ) -> tuple[RigidStateBatch, StepFlags]:
    """Advance every robot by one semi-implicit Euler step (dynamics.py:238-264).

    Pure: returns a new batch (or writes `out`, which may be `states` for an
    in-place update).  flags.nonfinite marks robots the caller must reset.
    """
    if not 0.0 < dt <= 0.1:
        raise ValueError(f"dt must be in (0, 0.1], got {dt}")
    if states.n != wrenches.n:
        raise ValueError("states and wrenches must have the same length")
    lib = N.load()
    out = out if out is not None else RigidStateBatch.empty(states.n, states.device)
    bits = torch.empty(max(states.n, 1), dtype=torch.uint8, device=states.device)
    with torch.cuda.device(states.device):
        N.check(lib.fs_integrate(states.n, ptr(states.buf), states.stride, ptr(wrenches.buf),
                                 wrenches.stride, params.native(), float(dt), ptr(out.buf),
                                 out.stride, ptr(bits), stream_handle()), "step_batch")
    return out, StepFlags.from_bits(bits[:states.n])


def step(state: RigidState, params: RobotParams, wrench: Wrench, dt: float) -> RigidState:
    """Single-robot step; raises NonFiniteStateError instead of flagging
    (dynamics.py:344-358)."""
    batch = RigidStateBatch(p=state.p[None, :], q=state.q[None, :], v=state.v[None, :],
                            omega=state.omega[None, :])
    wb = WrenchBatch(thrust=[wrench.thrust], moment=wrench.moment[None, :])
    out, flags = step_batch(batch, params, wb, dt)
    if bool(flags.nonfinite[0]):
        raise NonFiniteStateError("integrated state is non-finite")
    return out.at(0)
