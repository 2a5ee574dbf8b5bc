"""Reference-side drop-in: flocksim's NumPy dataclasses in, the same classes out.

The reference's callers hand float64 NumPy dataclasses to its pure functions
(``World._pipeline``, world.py:254-257; ``bench._pipeline_step``,
bench.py:146-149).  This module accepts those very objects -- duck-typed, it
never imports the reference -- packs them into pinned fp32 planes, runs the
step through the C ABI's host entry point ``fs_step_host_ex`` (chunked
H2D copy -> fused control + integration kernel -> D2H copy, over 8 streams)
and returns instances of the CALLER'S classes (the module of
``type(states)`` supplies ``WrenchBatch`` / ``StepFlags``, the module of
``type(cmds)`` ``ControlFlags``).  A maintainer swaps it in with one
assignment:

    flocksim.bench._pipeline_step = compat.pipeline_step
    world._pipeline = compat.world_pipeline(world)

Functions (same names, arguments and errors as the reference):

* ``control_batch(states, cmds, gains, params, limits=None)``
  (control.py:352-386) -> (WrenchBatch, ControlFlags)
* ``step_batch(states, params, wrenches, dt, workers=1)``
  (dynamics.py:238-264) -> (RigidStateBatch, StepFlags)
* ``pipeline(states, cmds, gains, params, limits, dt)`` -- control_batch
  then step_batch fused in one kernel -> (RigidStateBatch, StepFlags)
* ``pipeline_step(...)`` -- ``bench._pipeline_step``'s signature and result

Numerics: the state and commands are rounded to fp32 on the way in (the
B200 layout); the controller runs in float64 from those
values and the integrator in fp32, to the 1e-5 rel / 1e-6 abs bar per step
(DESIGN.md 4.2).  Non-finite commands are the reference's constructors'
business (InvalidCommandError); a non-finite STATE in velocity mode is
flagged nonfinite instead of raising.
"""

from __future__ import annotations

import ctypes as C
import importlib
import threading
from types import SimpleNamespace

import numpy as np
import torch

from . import _native as N
from ._tensors import default_device, padded
from .control import ControlGains, ControlLimits
from .dynamics import RobotParams

MODE_ATTITUDE, MODE_VELOCITY = 0, 1      # control.py:29-30


# -- parameter conversion (the reference's dataclasses -> ours) ---------------

def _robot(params) -> RobotParams:
    return RobotParams(mass=float(params.mass), inertia=np.asarray(params.inertia, np.float64),
                       collision_radius=float(getattr(params, "collision_radius", 0.2)),
                       thrust_max=float(params.thrust_max),
                       moment_max=np.asarray(params.moment_max, np.float64),
                       gravity=float(params.gravity), v_limit=float(params.v_limit),
                       omega_limit=float(params.omega_limit))


def _gains(gains) -> ControlGains:
    return ControlGains(attitude=np.asarray(gains.attitude, np.float64),
                        rate=np.asarray(gains.rate, np.float64),
                        velocity=np.asarray(gains.velocity, np.float64))


def _limits(limits) -> ControlLimits:
    if limits is None:
        return ControlLimits()
    return ControlLimits(max_tilt=float(limits.max_tilt),
                         max_speed_cmd=float(limits.max_speed_cmd),
                         max_yaw_rate=float(limits.max_yaw_rate))


def _sibling(obj, name):
    """Class `name` from the module that defines type(obj) (the caller's
    flocksim module), or a plain namespace factory for duck-typed inputs."""
    mod = importlib.import_module(type(obj).__module__)
    cls = getattr(mod, name, None)
    return cls if cls is not None else SimpleNamespace


def _check_dt(dt):
    if not 0.0 < dt <= 0.1:                       # dynamics.py:257-258
        raise ValueError(f"dt must be in (0, 0.1], got {dt}")


# -- host session: pinned planes, device workspaces, streams --------------------

class HostSession:
    """Pinned host planes + device workspaces of one capacity on one device,
    reused across calls (grown on demand); one call at a time (a lock, since
    World._step_dynamics calls _pipeline from worker threads)."""

    def __init__(self, device=None, chunks: int = 8, nstreams: int = 8):
        self.device = torch.device(device) if device is not None else default_device()
        self.chunks, self.nstreams = int(chunks), int(nstreams)
        self.lib = N.load()
        self.cap = 0
        self.lock = threading.Lock()
        with torch.cuda.device(self.device):
            self.streams = [torch.cuda.Stream(self.device) for _ in range(self.nstreams)]
        self.handles = (C.c_void_p * self.nstreams)(*[s.cuda_stream for s in self.streams])

    def _ensure(self, n: int) -> None:
        if n <= self.cap:
            return
        cap = padded(max(n, 2 * self.cap))
        pin = dict(dtype=torch.float32, pin_memory=True)
        self.h_state = torch.empty((13, cap), **pin)
        self.h_cmd = torch.empty((8, cap), **pin)
        self.h_mode = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
        self.h_wrench = torch.empty((4, cap), **pin)
        self.h_flags = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
        dev = dict(dtype=torch.float32, device=self.device)
        self.d_state = torch.empty((13, cap), **dev)
        self.d_cmd = torch.empty((8, cap), **dev)
        self.d_mode = torch.empty(cap, dtype=torch.uint8, device=self.device)
        self.d_wrench = torch.empty((4, cap), **dev)
        self.d_flags = torch.empty(cap, dtype=torch.uint8, device=self.device)
        self.cap = cap

    def _pack(self, h, row, arr, n, w):
        """float64 (n, w) rows -> fp32 planes h[row:row + w] (fs_host_pack_f64,
        all host threads)."""
        a = np.ascontiguousarray(np.asarray(arr, np.float64).reshape(n, w))
        N.check(self.lib.fs_host_pack_f64(a.ctypes.data, n, w, w,
                                          h.data_ptr() + row * self.cap * 4, self.cap, 0),
                "fs_host_pack_f64")

    def _unpack(self, h, row, n, w):
        """fp32 planes h[row:row + w] -> a new float64 (n, w) array."""
        out = np.empty((n, w), np.float64)
        N.check(self.lib.fs_host_unpack_f64(h.data_ptr() + row * self.cap * 4, self.cap, n, w,
                                            out.ctypes.data, w, 0), "fs_host_unpack_f64")
        return out

    def _pack_states(self, states, n):
        for row, arr, w in ((0, states.p, 3), (3, states.q, 4), (7, states.v, 3),
                            (10, states.omega, 3)):
            self._pack(self.h_state, row, arr, n, w)

    def _pack_cmds(self, cmds, n):
        """-> (FS mode, number of command planes)"""
        mode = np.asarray(cmds.mode).reshape(-1)
        att, vel = cmds.attitude, cmds.velocity
        h = self.h_cmd
        if mode.size and (mode == MODE_ATTITUDE).all():
            fs_mode, off = N.FS_MODE_ATTITUDE, None
        elif mode.size and (mode == MODE_VELOCITY).all():
            fs_mode, off = N.FS_MODE_VELOCITY, None
        else:
            fs_mode, off = N.FS_MODE_MIXED, 4
            self.h_mode[:n].copy_(torch.from_numpy(mode.astype(np.uint8)))
        if fs_mode != N.FS_MODE_VELOCITY:
            for k, a in enumerate((att.roll, att.pitch, att.yaw_rate, att.thrust)):
                self._pack(h, k, a, n, 1)
        if fs_mode != N.FS_MODE_ATTITUDE:
            b = off or 0
            self._pack(h, b, vel.v, n, 3)
            self._pack(h, b + 3, vel.yaw_rate, n, 1)
        return fs_mode

    def run(self, states, cmds, gains, params, limits, dt, integrate, want_wrench):
        """One fs_step_host_ex call; returns new host float64 arrays
        (state (p, q, v, omega) rows | None, wrench (thrust (n,), moment (n, 3)) | None,
        flags (n,))."""
        n = int(np.asarray(states.p).shape[0])
        with self.lock:
            self._ensure(max(n, 1))
            if n == 0:
                return ((np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros((0, 3)))
                        if integrate else None,
                        (np.zeros(0), np.zeros((0, 3))) if want_wrench else None,
                        np.zeros(0, np.uint8))
            self._pack_states(states, n)
            fs_mode = self._pack_cmds(cmds, n)
            d = N.fs_step_desc()
            d.n = n
            d.state_in = d.state_out = C.c_void_p(self.h_state.data_ptr())
            d.state_in_stride = d.state_out_stride = self.cap
            d.mode = fs_mode
            d.integrate = 1 if integrate else 0
            d.mode_per_vehicle = C.c_void_p(self.h_mode.data_ptr()) \
                if fs_mode == N.FS_MODE_MIXED else None
            d.cmd = C.c_void_p(self.h_cmd.data_ptr())
            d.cmd_stride = self.cap
            d.wrench_out = C.c_void_p(self.h_wrench.data_ptr()) if want_wrench else None
            d.wrench_stride = self.cap
            d.flags_out = C.c_void_p(self.h_flags.data_ptr())
            d.dt = float(dt)
            ws = N.fs_host_ws()
            ws.dev_state = C.c_void_p(self.d_state.data_ptr())
            ws.dev_cmd = C.c_void_p(self.d_cmd.data_ptr())
            ws.dev_mode = C.c_void_p(self.d_mode.data_ptr())
            ws.dev_wrench = C.c_void_p(self.d_wrench.data_ptr())
            ws.dev_flags = C.c_void_p(self.d_flags.data_ptr())
            ws.dev_stride = self.cap
            ws.chunks, ws.nstreams = self.chunks, self.nstreams
            ws.streams = self.handles
            with torch.cuda.device(self.device):
                N.check(self.lib.fs_step_host_ex(C.byref(d), params.native(), gains.native(),
                                                 limits.native(), None, C.byref(ws)),
                        "fs_step_host_ex")
                for s in self.streams:
                    s.synchronize()
            st = tuple(self._unpack(self.h_state, row, n, w)
                       for row, w in ((0, 3), (3, 4), (7, 3), (10, 3))) if integrate else None
            wr = ((self._unpack(self.h_wrench, 0, n, 1).reshape(n),
                   self._unpack(self.h_wrench, 1, n, 3)) if want_wrench else None)
            return st, wr, self.h_flags[:n].numpy().copy()


_SESSIONS: dict = {}
_SESSIONS_LOCK = threading.Lock()


def session(device=None) -> HostSession:
    """The process-wide HostSession of `device` (default: the current one)."""
    dev = torch.device(device) if device is not None else default_device()
    with _SESSIONS_LOCK:
        s = _SESSIONS.get(dev)
        if s is None:
            s = _SESSIONS[dev] = HostSession(dev)
        return s


def _states_like(states, st):
    """The caller's RigidStateBatch class from (p, q, v, omega) rows, or from
    a (13, n) plane array."""
    cls = type(states)
    if isinstance(st, tuple):
        return cls(p=st[0], q=st[1], v=st[2], omega=st[3])
    return cls(p=np.ascontiguousarray(st[0:3].T), q=np.ascontiguousarray(st[3:7].T),
               v=np.ascontiguousarray(st[7:10].T), omega=np.ascontiguousarray(st[10:13].T))


def _step_flags(states, bits):
    return _sibling(states, "StepFlags")(clamped=(bits & N.FS_FLAG_CLAMPED) != 0,
                                         nonfinite=(bits & N.FS_FLAG_NONFINITE) != 0)


# -- the reference's functions ---------------------------------------------------

def control_batch(states, cmds, gains, params, limits=None, device=None):
    """control.py:352-386 on the GPU -> (WrenchBatch, ControlFlags) of the
    caller's classes."""
    n = int(np.asarray(states.p).shape[0])
    if int(np.asarray(cmds.mode).reshape(-1).shape[0]) != n:
        raise ValueError("command batch length does not match state batch")   # control.py:363
    _, wr, bits = session(device).run(states, cmds, _gains(gains), _robot(params),
                                      _limits(limits), 0.01, False, True)
    wrench = _sibling(states, "WrenchBatch")(thrust=wr[0], moment=wr[1])
    flags = _sibling(cmds, "ControlFlags")(
        gimbal_degenerate=(bits & N.FS_FLAG_GIMBAL) != 0,
        degenerate_acceleration=(bits & N.FS_FLAG_DEGENERATE) != 0)
    return wrench, flags


def pipeline(states, cmds, gains, params, limits, dt, device=None):
    """control_batch -> step_batch fused in one kernel (world.py:254-257):
    -> (RigidStateBatch, StepFlags) of the caller's classes."""
    _check_dt(dt)
    n = int(np.asarray(states.p).shape[0])
    if int(np.asarray(cmds.mode).reshape(-1).shape[0]) != n:
        raise ValueError("command batch length does not match state batch")
    st, _, bits = session(device).run(states, cmds, _gains(gains), _robot(params),
                                      _limits(limits), dt, True, False)
    return _states_like(states, st), _step_flags(states, bits)


def pipeline_step(states, cmds, gains, params, limits, dt, workers=1):
    """bench._pipeline_step (bench.py:146-149): `workers` is accepted and
    ignored (results never depend on partitioning, dynamics.py:18-19)."""
    out, _ = pipeline(states, cmds, gains, params, limits, dt)
    return out


def step_batch(states, params, wrenches, dt, workers=1, device=None):
    """dynamics.py:238-264 on the GPU: the integrator alone on given
    (already saturated) wrenches -> (RigidStateBatch, StepFlags)."""
    from .dynamics import RigidStateBatch, WrenchBatch
    from .dynamics import step_batch as _step_batch
    _check_dt(dt)
    n = int(np.asarray(states.p).shape[0])
    if int(np.asarray(wrenches.thrust).reshape(-1).shape[0]) != n:
        raise ValueError("states and wrenches must have the same length")     # dynamics.py:260
    dev = torch.device(device) if device is not None else default_device()
    with torch.cuda.device(dev):
        st = RigidStateBatch(p=np.asarray(states.p), q=np.asarray(states.q),
                             v=np.asarray(states.v), omega=np.asarray(states.omega), device=dev)
        w = WrenchBatch(thrust=np.asarray(wrenches.thrust, np.float64).reshape(n),
                        moment=np.asarray(wrenches.moment, np.float64).reshape(n, 3), device=dev)
        out, flags = _step_batch(st, _robot(params), w, dt)
        bits = (flags.clamped.to(torch.uint8) * N.FS_FLAG_CLAMPED
                | flags.nonfinite.to(torch.uint8) * N.FS_FLAG_NONFINITE).cpu().numpy()
        arr = out.numpy()
    return _states_like(states, arr), _step_flags(states, bits)


def world_pipeline(world):
    """A drop-in for World._pipeline (world.py:254-257) bound to `world`'s
    gains, robot, limits and dt: assign it to ``world._pipeline``."""
    def _pipeline(states, commands, sl):
        return pipeline(states.slice(sl), commands.slice(sl), world.gains, world.robot,
                        world.limits, world.dt)
    return _pipeline


__all__ = ["HostSession", "session", "control_batch", "pipeline", "pipeline_step", "step_batch",
           "world_pipeline"]
