"""Batched geometric SE(3) controllers on B200 -- drop-in for ``flocksim.control``.

Mirrors /root/reference/pkg/src/flocksim/control.py (names, argument
meaning, validation, exception types).  Every per-vehicle evaluation is a
CUDA kernel behind include/flocksim_b200.h; command validation is the only
host synchronisation and happens once, at command construction, exactly
where the reference performs it (control.py:86-95, 122-126).

Extensions (not in the reference): ``PositionCommands``
and ``position_control`` (Lee position controller with yaw setpoint) and the
``fused_step`` entry point (control + integration in one kernel).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._tensors import alloc_planes, as_device, default_device, pack_rows, ptr, stride0, stream_handle
from .dynamics import (GIMBAL_TOL, RigidStateBatch, RobotParams, StepFlags, WrenchBatch,
                       saturate_batch)

MODE_ATTITUDE = 0           # control.py:29
MODE_VELOCITY = 1           # control.py:30
MODE_POSITION = 3           # EXTENSION (FS_MODE_POSITION)
DEGENERATE_ACCEL = 1e-6     # control.py:33


class InvalidCommandError(ValueError):
    """Raised for non-finite or out-of-range command values (control.py:36-38)."""


@dataclass
class ControlGains:
    """Diagonal gains, strictly positive 3-vectors (control.py:40-59).

    ``position`` is the EXTENSION position-loop gain k_p.
    """

    attitude: np.ndarray = field(default_factory=lambda: np.array([8.0, 8.0, 2.0]))
    rate: np.ndarray = field(default_factory=lambda: np.array([1.2, 1.2, 0.6]))
    velocity: np.ndarray = field(default_factory=lambda: np.array([3.0, 3.0, 3.0]))
    position: np.ndarray = field(default_factory=lambda: np.array([2.0, 2.0, 2.0]))

    def __post_init__(self):
        for name in ("attitude", "rate", "velocity", "position"):
            v = np.asarray(getattr(self, name), dtype=np.float64)
            setattr(self, name, v)
            if v.shape != (3,) or (v <= 0.0).any():
                raise ValueError(f"{name} gains must be strictly positive 3-vectors")

    def native(self) -> N.fs_gains:
        g = N.fs_gains()
        g.attitude[:] = [float(x) for x in self.attitude]
        g.rate[:] = [float(x) for x in self.rate]
        g.velocity[:] = [float(x) for x in self.velocity]
        g.position[:] = [float(x) for x in self.position]
        return g


@dataclass
class ControlLimits:
    """Command envelope keeping the tilt parameterization away from pi/2
    (control.py:62-74)."""

    max_tilt: float = 0.6
    max_speed_cmd: float = 5.0
    max_yaw_rate: float = 3.0

    def __post_init__(self):
        if not 0.0 < self.max_tilt < np.pi / 2:
            raise ValueError("max_tilt must be in (0, pi/2)")
        if self.max_speed_cmd <= 0.0 or self.max_yaw_rate <= 0.0:
            raise ValueError("command limits must be positive")

    def native(self) -> N.fs_limits:
        l = N.fs_limits()
        l.max_tilt = self.max_tilt
        l.max_speed_cmd = self.max_speed_cmd
        l.max_yaw_rate = self.max_yaw_rate
        return l


def _device_of(*xs):
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device
    return default_device()


def _n_of(x) -> int:
    if isinstance(x, torch.Tensor):
        return int(x.reshape(-1).shape[0]) if x.dim() <= 1 else int(x.shape[0])
    a = np.atleast_1d(np.asarray(x))
    return int(a.shape[0])


class _Commands:
    """4-plane command record; `buf` is a (4, stride) fp32 CUDA tensor view."""

    K = 4

    @property
    def n(self) -> int:
        return self._n

    @property
    def stride(self) -> int:
        return stride0(self.buf)

    @property
    def device(self):
        return self.buf.device

    def _wrap(self, buf, n):
        self.buf = buf
        self._n = int(n)


class AttitudeCommands(_Commands):
    """Batched attitude-mode commands: roll, pitch, yaw_rate, thrust
    (control.py:77-112).  Planes: roll, pitch, yaw_rate, thrust."""

    def __init__(self, roll, pitch, yaw_rate, thrust, device=None, validate=True):
        device = device if device is not None else _device_of(roll, pitch, yaw_rate, thrust)
        n = _n_of(roll)
        if validate:
            # the reference validates its float64 arrays (control.py:86-95):
            # check the inputs before they are rounded to the fp32 planes, so
            # a tilt just below pi/2 that rounds up to fp32(pi/2) is accepted
            # exactly when the reference accepts it
            src = [as_device(x, device, dtype=torch.float64).reshape(-1)
                   for x in (roll, pitch, yaw_rate, thrust)]
            if not all(bool(torch.isfinite(t).all()) for t in src):
                raise InvalidCommandError("attitude command contains non-finite values")
            if bool((src[0].abs() >= np.pi / 2).any()) or bool((src[1].abs() >= np.pi / 2).any()):
                raise InvalidCommandError("commanded tilt angles must satisfy |angle| < pi/2")
        buf = alloc_planes(4, n, device)
        for k, x in enumerate((roll, pitch, yaw_rate, thrust)):
            pack_rows(buf, k, x, n, 1)
        self._wrap(buf, n)

    def validate(self):
        """Validation of fp32 planes (from_planes); the constructor checks
        the float64 inputs instead."""
        v = self.buf[:, :self._n]
        if not bool(torch.isfinite(v).all()):
            raise InvalidCommandError("attitude command contains non-finite values")
        if bool((v[0:2].abs() >= np.pi / 2).any()):
            raise InvalidCommandError("commanded tilt angles must satisfy |angle| < pi/2")

    @classmethod
    def from_planes(cls, buf, n, validate=False):
        obj = cls.__new__(cls)
        obj._wrap(buf, n)
        if validate:
            obj.validate()
        return obj

    @classmethod
    def single(cls, roll, pitch, yaw_rate, thrust) -> "AttitudeCommands":
        return cls(roll=[roll], pitch=[pitch], yaw_rate=[yaw_rate], thrust=[thrust])

    @classmethod
    def hover(cls, n: int, params: RobotParams, device=None) -> "AttitudeCommands":
        buf = alloc_planes(4, n, device, zero=True)
        buf[3, :n] = params.hover_thrust
        return cls.from_planes(buf, n)

    roll = property(lambda self: self.buf[0, :self._n])
    pitch = property(lambda self: self.buf[1, :self._n])
    yaw_rate = property(lambda self: self.buf[2, :self._n])
    thrust = property(lambda self: self.buf[3, :self._n])

    def slice(self, sl: slice) -> "AttitudeCommands":
        a, b, _ = sl.indices(self._n)
        return AttitudeCommands.from_planes(self.buf[:, a:b], max(0, b - a))


class VelocityCommands(_Commands):
    """Batched velocity-mode commands: vehicle-frame velocity (N, 3) and yaw
    rate (N,) (control.py:115-137).  Planes: vx, vy, vz, yaw_rate."""

    def __init__(self, v, yaw_rate, device=None, validate=True):
        device = device if device is not None else _device_of(v, yaw_rate)
        vt = as_device(v, device)
        if vt.dim() == 1:
            vt = vt.reshape(1, 3)
        n = int(vt.shape[0])
        if validate:
            # float64 inputs, as the reference checks them (control.py:122-126)
            v64 = as_device(v, device, dtype=torch.float64)
            y64 = as_device(yaw_rate, device, dtype=torch.float64)
            if not (bool(torch.isfinite(v64).all()) and bool(torch.isfinite(y64).all())):
                raise InvalidCommandError("velocity command contains non-finite values")
        buf = alloc_planes(4, n, device)
        pack_rows(buf, 0, vt, n, 3)
        pack_rows(buf, 3, yaw_rate, n, 1)
        self._wrap(buf, n)

    def validate(self):
        if not bool(torch.isfinite(self.buf[:, :self._n]).all()):
            raise InvalidCommandError("velocity command contains non-finite values")

    @classmethod
    def from_planes(cls, buf, n, validate=False):
        obj = cls.__new__(cls)
        obj._wrap(buf, n)
        if validate:
            obj.validate()
        return obj

    @classmethod
    def single(cls, v, yaw_rate) -> "VelocityCommands":
        return cls(v=np.asarray(v, dtype=np.float64)[None, :], yaw_rate=[yaw_rate])

    v = property(lambda self: self.buf[0:3, :self._n].T)
    yaw_rate = property(lambda self: self.buf[3, :self._n])

    def slice(self, sl: slice) -> "VelocityCommands":
        a, b, _ = sl.indices(self._n)
        return VelocityCommands.from_planes(self.buf[:, a:b], max(0, b - a))


class PositionCommands(_Commands):
    """EXTENSION: position setpoint (N, 3) and yaw setpoint (N,).
    Planes: px_d, py_d, pz_d, yaw_d."""

    def __init__(self, p, yaw, device=None, validate=True):
        device = device if device is not None else _device_of(p, yaw)
        pt = as_device(p, device)
        if pt.dim() == 1:
            pt = pt.reshape(1, 3)
        n = int(pt.shape[0])
        buf = alloc_planes(4, n, device)
        pack_rows(buf, 0, pt, n, 3)
        pack_rows(buf, 3, yaw, n, 1)
        self._wrap(buf, n)
        if validate and not bool(torch.isfinite(buf[:, :n]).all()):
            raise InvalidCommandError("position command contains non-finite values")

    @classmethod
    def from_planes(cls, buf, n):
        obj = cls.__new__(cls)
        obj._wrap(buf, n)
        return obj

    p = property(lambda self: self.buf[0:3, :self._n].T)
    yaw = property(lambda self: self.buf[3, :self._n])

    def slice(self, sl: slice) -> "PositionCommands":
        a, b, _ = sl.indices(self._n)
        return PositionCommands.from_planes(self.buf[:, a:b], max(0, b - a))


class CommandBatch:
    """Per-robot tagged union of attitude- and velocity-mode commands
    (control.py:140-171).  Stored as one (8, stride) buffer (attitude planes
    then velocity planes) plus a uint8 mode plane; ``uniform_mode`` records a
    batch built by all_attitude/all_velocity so no device scan is needed."""

    def __init__(self, mode, attitude: AttitudeCommands, velocity: VelocityCommands,
                 uniform_mode: int | None = None):
        n = attitude.n
        device = attitude.device
        if velocity.n != n:
            raise ValueError("attitude and velocity commands differ in length")
        self.mode = as_device(mode, device, dtype=torch.uint8).reshape(-1)
        if self.mode.numel() == 1 and n != 1:
            self.mode = self.mode.expand(n).contiguous()
        self.buf = alloc_planes(8, n, device)
        self.buf[0:4, :n].copy_(attitude.buf[:, :n])
        self.buf[4:8, :n].copy_(velocity.buf[:, :n])
        self._n = n
        self.uniform_mode = uniform_mode

    @classmethod
    def _from_buf(cls, buf, mode, n, uniform_mode):
        obj = cls.__new__(cls)
        obj.buf, obj.mode, obj._n, obj.uniform_mode = buf, mode, n, uniform_mode
        return obj

    @classmethod
    def all_attitude(cls, att: AttitudeCommands) -> "CommandBatch":
        n = att.n
        buf = alloc_planes(8, n, att.device, zero=True)
        buf[0:4, :n].copy_(att.buf[:, :n])
        mode = torch.zeros(n, dtype=torch.uint8, device=att.device)
        return cls._from_buf(buf, mode, n, MODE_ATTITUDE)

    @classmethod
    def all_velocity(cls, vel: VelocityCommands) -> "CommandBatch":
        n = vel.n
        buf = alloc_planes(8, n, vel.device, zero=True)
        buf[4:8, :n].copy_(vel.buf[:, :n])
        mode = torch.full((n,), MODE_VELOCITY, dtype=torch.uint8, device=vel.device)
        return cls._from_buf(buf, mode, n, MODE_VELOCITY)

    @property
    def n(self) -> int:
        return self._n

    @property
    def device(self):
        return self.buf.device

    @property
    def attitude(self) -> AttitudeCommands:
        return AttitudeCommands.from_planes(self.buf[0:4], self._n)

    @property
    def velocity(self) -> VelocityCommands:
        return VelocityCommands.from_planes(self.buf[4:8], self._n)

    def slice(self, sl: slice) -> "CommandBatch":
        a, b, _ = sl.indices(self._n)
        return CommandBatch._from_buf(self.buf[:, a:b], self.mode[a:b], max(0, b - a),
                                      self.uniform_mode)

    def kernel_mode(self):
        """(FS mode, cmd pointer view, stride) for the fused kernel."""
        if self.uniform_mode == MODE_ATTITUDE:
            return N.FS_MODE_ATTITUDE, self.buf[0:4]
        if self.uniform_mode == MODE_VELOCITY:
            return N.FS_MODE_VELOCITY, self.buf[4:8]
        return N.FS_MODE_MIXED, self.buf


@dataclass
class ControlErrors:
    """Rotation and angular-velocity tracking errors (control.py:174-179)."""

    rotation: torch.Tensor  # (N, 3), e_R = 0.5 * vee(Rd^T R - R^T Rd)
    rate: torch.Tensor      # (N, 3), e_w = w - R^T Rd wd


@dataclass
class ControlFlags:
    """Per-robot diagnostic flags (control.py:182-187)."""

    gimbal_degenerate: torch.Tensor
    degenerate_acceleration: torch.Tensor


# =============================================================================
# operations
# =============================================================================

def yaw_of(q) -> tuple[torch.Tensor, torch.Tensor]:
    """ZYX yaw psi = atan2(R10, R00) and the gimbal flag (se3.py:226-243).
    `q` is an (N, 4) tensor view (e.g. RigidStateBatch.q) or array."""
    lib = N.load()
    if isinstance(q, torch.Tensor) and q.is_cuda and q.dim() == 2 and q.stride(0) == 1:
        qt, qs, n = q, int(q.stride(1)), int(q.shape[0])
    else:
        qa = as_device(q, _device_of(q)).reshape(-1, 4)
        n = int(qa.shape[0])
        buf = alloc_planes(4, n, qa.device)
        buf[:, :n].copy_(qa.T)
        qt, qs = buf, stride0(buf)
    yaw = torch.empty(max(n, 1), dtype=torch.float32, device=qt.device)
    gim = torch.empty(max(n, 1), dtype=torch.uint8, device=qt.device)
    with torch.cuda.device(qt.device):
        N.check(lib.fs_yaw_of(n, ptr(qt), qs, math.cos(GIMBAL_TOL), ptr(yaw), ptr(gim),
                              stream_handle()), "yaw_of")
    return yaw[:n], gim[:n].bool()


def desired_attitude(yaw, cmd: AttitudeCommands) -> tuple[torch.Tensor, torch.Tensor]:
    """Desired orientation and body rate for attitude-mode commands
    (control.py:190-218).  Returns (q_d (N, 4), omega_d (N, 3)) views."""
    lib = N.load()
    n = cmd.n
    y = as_device(yaw, cmd.device).reshape(-1).contiguous()
    qd = alloc_planes(4, n, cmd.device)
    wd = alloc_planes(3, n, cmd.device)
    with torch.cuda.device(cmd.device):
        N.check(lib.fs_desired_attitude(n, ptr(y), ptr(cmd.buf), cmd.stride, ptr(qd), stride0(qd),
                                        ptr(wd), stride0(wd), stream_handle()),
                "desired_attitude")
    return qd[:, :n].T, wd[:, :n].T


def _as_planes(x, k, device):
    """(N, k) view/array -> ((k, stride) tensor, stride, n)."""
    if isinstance(x, torch.Tensor) and x.is_cuda and x.dim() == 2 and x.stride(0) == 1 \
            and x.dtype == torch.float32:
        return x, int(x.stride(1)), int(x.shape[0])
    t = as_device(x, device).reshape(-1, k)
    n = int(t.shape[0])
    buf = alloc_planes(k, n, device)
    buf[:, :n].copy_(t.T)
    return buf, stride0(buf), n


def attitude_errors(q, omega, q_d, omega_d) -> ControlErrors:
    """Geometric attitude and rate errors (control.py:221-258)."""
    lib = N.load()
    dev = _device_of(q, omega, q_d, omega_d)
    qt, qs, n = _as_planes(q, 4, dev)
    wt, ws, _ = _as_planes(omega, 3, dev)
    qdt, qds, _ = _as_planes(q_d, 4, dev)
    wdt, wds, _ = _as_planes(omega_d, 3, dev)
    er = alloc_planes(3, n, dev)
    ew = alloc_planes(3, n, dev)
    with torch.cuda.device(dev):
        N.check(lib.fs_attitude_errors(n, ptr(qt), qs, ptr(wt), ws, ptr(qdt), qds, ptr(wdt), wds,
                                       ptr(er), ptr(ew), stride0(er), stream_handle()),
                "attitude_errors")
    return ControlErrors(rotation=er[:, :n].T, rate=ew[:, :n].T)


def attitude_control(states: RigidStateBatch, cmd: AttitudeCommands, gains: ControlGains,
                     params: RobotParams) -> WrenchBatch:
    """Attitude-mode law M = -k_R e_R - k_W e_W + w x J w, saturated
    (control.py:261-280)."""
    if cmd.n != states.n:
        raise ValueError("command batch length does not match state batch")
    lib = N.load()
    out = WrenchBatch.empty(states.n, states.device)
    with torch.cuda.device(states.device):
        N.check(lib.fs_attitude_control(states.n, ptr(states.buf), states.stride, ptr(cmd.buf),
                                        cmd.stride, params.native(), gains.native(),
                                        ptr(out.buf), out.stride, stream_handle()),
                "attitude_control")
    return out


def velocity_control(states: RigidStateBatch, cmd: VelocityCommands, gains: ControlGains,
                     params: RobotParams, limits: ControlLimits | None = None
                     ) -> tuple[AttitudeCommands, torch.Tensor]:
    """Velocity-mode outer loop -> (attitude commands, degenerate mask)
    (control.py:283-349)."""
    if cmd.n != states.n:
        raise ValueError("command batch length does not match state batch")
    limits = limits if limits is not None else ControlLimits()
    lib = N.load()
    n = states.n
    att = alloc_planes(4, n, states.device)
    deg = torch.empty(max(n, 1), dtype=torch.uint8, device=states.device)
    with torch.cuda.device(states.device):
        N.check(lib.fs_velocity_control(n, ptr(states.buf), states.stride, ptr(cmd.buf), cmd.stride,
                                        params.native(), gains.native(), limits.native(),
                                        ptr(att), stride0(att), ptr(deg), stream_handle()),
                "velocity_control")
    return AttitudeCommands.from_planes(att, n), deg[:n].bool()


def position_control(states: RigidStateBatch, cmd: PositionCommands, gains: ControlGains,
                     params: RobotParams, limits: ControlLimits | None = None
                     ) -> tuple[WrenchBatch, torch.Tensor]:
    """EXTENSION: Lee geometric position controller with a yaw setpoint
     -> (saturated wrench, degenerate
    mask).  Shaped like the reference's controllers (velocity_control,
    control.py:283-349, returns its output and the degenerate mask): the
    commanded acceleration a = -k_p (p - p_d) - k_v v + g e3 is tilt-limited
    to max_tilt, f = m a . b3, R_d = [b2d x b3d, b3d x b1c / |.|, a / |a|],
    omega_d = 0, and the moment law and saturation are attitude_control's.
    No reference code exists, so the oracle is the builder's float64
    restatement (oracle/flocksim_oracle.py position_control; parity
    unpinned by the reference)."""
    if cmd.n != states.n:
        raise ValueError("command batch length does not match state batch")
    limits = limits if limits is not None else ControlLimits()
    lib = N.load()
    n = states.n
    wrench = WrenchBatch.empty(n, states.device)
    bits = torch.empty(max(n, 1), dtype=torch.uint8, device=states.device)
    d = _step_desc(states, cmd.buf, N.FS_MODE_POSITION, 0.01, False, wrench=wrench, flags=bits)
    with torch.cuda.device(states.device):
        N.check(lib.fs_step(d, params.native(), gains.native(), limits.native(), None,
                            stream_handle()), "position_control")
    return wrench, (bits[:n] & N.FS_FLAG_DEGENERATE) != 0


def _step_desc(states, cmd_view, mode, dt, integrate, out=None, wrench=None, flags=None,
               mode_plane=None, rotor=None, vparams=None, airframe_split=0,
               rotor_dynamics=False, reset_prob=0.0, seed=0, step_index=0, stats=None,
               first_id=0):
    d = N.fs_step_desc()
    d.n = states.n
    d.first_id = first_id
    d.state_in = ptr(states.buf)
    d.state_in_stride = states.stride
    d.state_out = ptr(out.buf) if out is not None else None
    d.state_out_stride = out.stride if out is not None else 0
    d.mode = mode
    d.integrate = 1 if integrate else 0
    d.mode_per_vehicle = ptr(mode_plane) if mode_plane is not None else None
    d.cmd = ptr(cmd_view)
    d.cmd_stride = stride0(cmd_view)
    d.vparams = ptr(vparams) if vparams is not None else None
    d.vparams_stride = stride0(vparams) if vparams is not None else 0
    d.airframe_split = airframe_split
    d.wrench_out = ptr(wrench.buf) if wrench is not None else None
    d.wrench_stride = wrench.stride if wrench is not None else 0
    d.rotor_out = ptr(rotor) if rotor is not None else None
    d.rotor_stride = stride0(rotor) if rotor is not None else 0
    d.flags_out = ptr(flags) if flags is not None else None
    d.rotor_dynamics = 1 if rotor_dynamics else 0
    d.dt = dt
    d.reset_prob = reset_prob
    d.seed = seed
    d.step_index = step_index
    d.stats_slots = ptr(stats) if stats is not None else None
    d.stats_nslots = int(stats.shape[0]) if stats is not None else 0
    return d


def control_batch(states: RigidStateBatch, cmds: CommandBatch, gains: ControlGains,
                  params: RobotParams, limits: ControlLimits | None = None
                  ) -> tuple[WrenchBatch, ControlFlags]:
    """Route a mixed-mode command batch through the controllers
    (control.py:352-386): one kernel, velocity rows run the outer loop
    first, every row is tracked by the attitude law and saturated."""
    if cmds.n != states.n:
        raise ValueError("command batch length does not match state batch")
    limits = limits if limits is not None else ControlLimits()
    lib = N.load()
    n = states.n
    wrench = WrenchBatch.empty(n, states.device)
    bits = torch.empty(max(n, 1), dtype=torch.uint8, device=states.device)
    mode, view = cmds.kernel_mode()
    d = _step_desc(states, view, mode, 0.01, False, wrench=wrench, flags=bits,
                   mode_plane=cmds.mode if mode == N.FS_MODE_MIXED else None)
    with torch.cuda.device(states.device):
        N.check(lib.fs_step(d, params.native(), gains.native(), limits.native(), None,
                            stream_handle()), "control_batch")
    bits = bits[:n]
    return wrench, ControlFlags(gimbal_degenerate=(bits & N.FS_FLAG_GIMBAL) != 0,
                                degenerate_acceleration=(bits & N.FS_FLAG_DEGENERATE) != 0)


def fused_step(states: RigidStateBatch, cmds, gains: ControlGains, params: RobotParams,
               dt: float, limits: ControlLimits | None = None,
               out: RigidStateBatch | None = None, want_flags: bool = True,
               wrench: WrenchBatch | None = None):
    """control_batch followed by step_batch in ONE kernel (the hot path;
    bench.py:146-149 / world.py:254-257).  `cmds` is a CommandBatch,
    AttitudeCommands, VelocityCommands or PositionCommands.  `out` may be
    `states` (in place).  Returns (new states, StepFlags | None)."""
    if not 0.0 < dt <= 0.1:
        raise ValueError(f"dt must be in (0, 0.1], got {dt}")
    if cmds.n != states.n:
        raise ValueError("command batch length does not match state batch")
    limits = limits if limits is not None else ControlLimits()
    lib = N.load()
    n = states.n
    out = out if out is not None else RigidStateBatch.empty(n, states.device)
    mode_plane = None
    if isinstance(cmds, CommandBatch):
        mode, view = cmds.kernel_mode()
        mode_plane = cmds.mode if mode == N.FS_MODE_MIXED else None
    elif isinstance(cmds, AttitudeCommands):
        mode, view = N.FS_MODE_ATTITUDE, cmds.buf
    elif isinstance(cmds, VelocityCommands):
        mode, view = N.FS_MODE_VELOCITY, cmds.buf
    elif isinstance(cmds, PositionCommands):
        mode, view = N.FS_MODE_POSITION, cmds.buf
    else:
        raise TypeError(f"unsupported command type {type(cmds).__name__}")
    bits = torch.empty(max(n, 1), dtype=torch.uint8, device=states.device) if want_flags else None
    d = _step_desc(states, view, mode, float(dt), True, out=out, wrench=wrench, flags=bits,
                   mode_plane=mode_plane)
    with torch.cuda.device(states.device):
        N.check(lib.fs_step(d, params.native(), gains.native(), limits.native(), None,
                            stream_handle()), "fused_step")
    return out, (StepFlags.from_bits(bits[:n]) if want_flags else None)


__all__ = [
    "MODE_ATTITUDE", "MODE_VELOCITY", "MODE_POSITION", "DEGENERATE_ACCEL",
    "InvalidCommandError", "ControlGains", "ControlLimits", "AttitudeCommands",
    "VelocityCommands", "PositionCommands", "CommandBatch", "ControlErrors", "ControlFlags",
    "yaw_of", "desired_attitude", "attitude_errors", "attitude_control", "velocity_control",
    "position_control", "control_batch", "fused_step", "saturate_batch",
]
