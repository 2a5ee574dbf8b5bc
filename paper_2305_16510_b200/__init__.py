"""B200-native batched multirotor control step (Aerial Gym / flocksim hot path).

Drop-in for the reference's controller and dynamics API
(/root/reference/pkg/src/flocksim/control.py, dynamics.py): batched state
and command tensors in, wrenches / rotor thrusts / integrated states out,
every per-vehicle evaluation in hand-written sm_100a CUDA kernels behind the
C ABI in include/flocksim_b200.h.  No CPU fallback.
"""

from . import _native
from .control import (DEGENERATE_ACCEL, MODE_ATTITUDE, MODE_POSITION, MODE_VELOCITY,
                      AttitudeCommands, CommandBatch, ControlErrors, ControlFlags, ControlGains,
                      ControlLimits, InvalidCommandError, PositionCommands, VelocityCommands,
                      attitude_control, attitude_errors, control_batch, desired_attitude,
                      fused_step, velocity_control, yaw_of)
from .dynamics import (DEFAULT_GRAVITY, NonFiniteStateError, RigidState, RigidStateBatch,
                       RobotParams, StepFlags, Wrench, WrenchBatch, saturate, saturate_batch,
                       step, step_batch)

__version__ = "0.1.0"
