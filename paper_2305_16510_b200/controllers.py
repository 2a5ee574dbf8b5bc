"""Controller objects: batched robot-state and command tensors in, wrenches
or rotor thrusts out (BASELINE.json north_star).

The reference evaluates its controllers as module-level functions over NumPy
dataclasses (``attitude_control`` control.py:261-280, ``velocity_control``
283-349, ``control_batch`` 352-386); these objects bind the parameters of
those calls (``RobotParams``, ``ControlGains``, ``ControlLimits``) once and
evaluate the same law with one fused kernel launch per call
(``fs_step`` with ``integrate = 0``, include/flocksim_b200.h):

* ``AttitudeController()(states, AttitudeCommands)`` is
  ``attitude_control`` (control.py:261-280);
* ``VelocityController()(states, VelocityCommands)`` is ``velocity_control``
  followed by ``attitude_control`` -- ``control_batch`` on an all-velocity
  ``CommandBatch`` (control.py:352-386);
* ``PositionController()(states, PositionCommands)`` is the EXTENSION
  position law (``control.position_control``).

Each returns the saturated ``WrenchBatch`` (thrust (N,), moment (N, 3),
dynamics.py:179-200).  With an ``airframe`` (``allocation.QUAD_X`` /
``HEXAROTOR``, EXTENSION) the same launch also
allocates the wrench to rotors and the call returns ``(WrenchBatch, rotors)``
with ``rotors`` an (N, n_rotors) view of T = clip(A^+ w, 0, rotor_max).
``flags`` holds the last call's ``ControlFlags`` (control.py:182-187).
``step(states, commands, dt)`` runs the same controller fused with the
integrator (``step_batch``, dynamics.py:238-264) in the same launch.

``states`` is a ``RigidStateBatch`` or an (N, 13) tensor ``[p q v omega]``;
``commands`` is the controller's command class or an (N, 4) tensor in that
class's plane order (validated like the class constructor).  Every output is
a CUDA tensor; nothing returns to the host.
"""

from __future__ import annotations

import torch

from . import _native as N
from ._tensors import alloc_planes, as_device, default_device, stream_handle
from .allocation import Airframe, native_pair
from .control import (AttitudeCommands, ControlFlags, ControlGains, ControlLimits,
                      PositionCommands, VelocityCommands, _step_desc)
from .dynamics import RigidStateBatch, RobotParams, StepFlags, WrenchBatch


def as_states(states, device=None) -> RigidStateBatch:
    """RigidStateBatch, or an (N, 13) tensor/array [p(3) q(4) v(3) omega(3)]
    packed into planes (one copy)."""
    if isinstance(states, RigidStateBatch):
        return states
    t = as_device(states, device if device is not None else default_device())
    if t.dim() != 2 or t.shape[1] != 13:
        raise ValueError(f"expected a RigidStateBatch or an (N, 13) tensor, got shape "
                         f"{tuple(t.shape)}")
    n = int(t.shape[0])
    buf = alloc_planes(13, n, t.device)
    buf[:, :n].copy_(t.T)
    return RigidStateBatch.from_planes(buf, n)


class _Controller:
    """Binds (params, gains, limits, airframe) to one control law."""

    MODE = None           # FS_MODE_*
    COMMANDS = None       # command class

    def __init__(self, params: RobotParams | None = None, gains: ControlGains | None = None,
                 limits: ControlLimits | None = None, airframe: Airframe | None = None,
                 rotor_dynamics: bool = False):
        self.params = params or RobotParams()
        self.gains = gains or ControlGains()
        self.limits = limits or ControlLimits()
        self.airframe = airframe
        self.rotor_dynamics = bool(rotor_dynamics)
        if self.rotor_dynamics and airframe is None:
            raise ValueError("rotor_dynamics needs an airframe")
        self.lib = N.load()
        self._robot = self.params.native()
        self._gains = self.gains.native()
        self._limits = self.limits.native()
        self._frames = native_pair(airframe) if airframe is not None else None
        self.flags: ControlFlags | None = None

    @property
    def n_rotors(self) -> int:
        return self.airframe.n_rotors if self.airframe is not None else 0

    def _commands(self, commands, n, device):
        if isinstance(commands, self.COMMANDS):
            return commands
        # float64 keeps float64 inputs exact for the constructor's validation
        t = as_device(commands, device, dtype=torch.float64)
        if t.dim() != 2 or t.shape[1] != 4:
            raise ValueError(f"expected {self.COMMANDS.__name__} or an (N, 4) tensor, got shape "
                             f"{tuple(t.shape)}")
        return self._from_rows(t)

    def _from_rows(self, t):
        raise NotImplementedError

    def _launch(self, st: RigidStateBatch, cmd, integrate: bool, dt: float, out):
        n = st.n
        if cmd.n != n:
            raise ValueError("command batch length does not match state batch")
        wrench = WrenchBatch.empty(n, st.device)
        bits = torch.empty(max(n, 1), dtype=torch.uint8, device=st.device)
        rotors = (alloc_planes(N.FS_MAX_ROTORS, n, st.device) if self._frames is not None
                  else None)
        d = _step_desc(st, cmd.buf, self.MODE, float(dt), integrate, out=out, wrench=wrench,
                       flags=bits, rotor=rotors, rotor_dynamics=self.rotor_dynamics)
        with torch.cuda.device(st.device):
            N.check(self.lib.fs_step(d, self._robot, self._gains, self._limits, self._frames,
                                     stream_handle()), type(self).__name__)
        bits = bits[:n]
        self.flags = ControlFlags(gimbal_degenerate=(bits & N.FS_FLAG_GIMBAL) != 0,
                                  degenerate_acceleration=(bits & N.FS_FLAG_DEGENERATE) != 0)
        rot = rotors[:self.n_rotors, :n].T if rotors is not None else None
        return wrench, rot, bits

    def __call__(self, states, commands):
        """Wrench (or (wrench, rotor thrusts)) for every vehicle."""
        st = as_states(states)
        cmd = self._commands(commands, st.n, st.device)
        wrench, rot, _ = self._launch(st, cmd, False, 0.01, None)
        return (wrench, rot) if rot is not None else wrench

    def step(self, states, commands, dt: float, out: RigidStateBatch | None = None):
        """This controller fused with step_batch (dynamics.py:238-264) in one
        launch: returns (new states, StepFlags).  `out` may be `states` (in
        place).  With rotor_dynamics the integrator applies the realized
        rotor wrench A clip(A^+ w)."""
        if not 0.0 < dt <= 0.1:
            raise ValueError(f"dt must be in (0, 0.1], got {dt}")
        st = as_states(states)
        cmd = self._commands(commands, st.n, st.device)
        out = out if out is not None else RigidStateBatch.empty(st.n, st.device)
        _, _, bits = self._launch(st, cmd, True, dt, out)
        return out, StepFlags.from_bits(bits)


class AttitudeController(_Controller):
    """Roll / pitch / yaw-rate / collective-thrust tracking (attitude_control,
    control.py:261-280): M = -k_R e_R - k_W e_W + w x J w, saturated."""

    MODE = N.FS_MODE_ATTITUDE
    COMMANDS = AttitudeCommands

    def _from_rows(self, t):
        return AttitudeCommands(t[:, 0], t[:, 1], t[:, 2], t[:, 3])


class VelocityController(_Controller):
    """Vehicle-frame velocity + yaw-rate tracking: velocity_control's outer
    loop (control.py:283-349) into attitude_control (261-280), as
    control_batch routes velocity rows (352-386)."""

    MODE = N.FS_MODE_VELOCITY
    COMMANDS = VelocityCommands

    def _from_rows(self, t):
        return VelocityCommands(v=t[:, 0:3], yaw_rate=t[:, 3])


class PositionController(_Controller):
    """EXTENSION: position + yaw setpoint tracking (control.position_control;
    SURVEY.md Appendix A.5).  `airframe` adds the rotor allocation (BASELINE
    config 0: QUAD_X, 1024 quads -> 4 rotor thrusts each)."""

    MODE = N.FS_MODE_POSITION
    COMMANDS = PositionCommands

    def _from_rows(self, t):
        return PositionCommands(p=t[:, 0:3], yaw=t[:, 3])


__all__ = ["AttitudeController", "VelocityController", "PositionController", "as_states"]
