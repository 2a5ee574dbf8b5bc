"""B200-native batched multirotor control step (Aerial Gym / flocksim hot path).

Drop-in for the reference's API (/root/reference/pkg/src/flocksim): the
controller and dynamics (control.py, dynamics.py) -- batched state and
command tensors in, wrenches / rotor thrusts / integrated states out -- the
rotation primitives (se3), World.step with obstacle scenes (world, scene,
assets), the depth camera (camera), the benchmark harness (bench), the config
loader and the RL bindings (rl).  Every per-vehicle / per-env / per-ray evaluation runs in hand-written
sm_100a CUDA kernels behind the C ABI in include/flocksim_b200.h.  No CPU
fallback.
"""

from . import _native
from .control import (DEGENERATE_ACCEL, MODE_ATTITUDE, MODE_POSITION, MODE_VELOCITY,
                      AttitudeCommands, CommandBatch, ControlErrors, ControlFlags, ControlGains,
                      ControlLimits, InvalidCommandError, PositionCommands, VelocityCommands,
                      attitude_control, attitude_errors, control_batch, desired_attitude,
                      fused_step, position_control, velocity_control, yaw_of)
from .controllers import AttitudeController, PositionController, VelocityController
from .dynamics import (DEFAULT_GRAVITY, NonFiniteStateError, RigidState, RigidStateBatch,
                       RobotParams, StepFlags, Wrench, WrenchBatch, saturate, saturate_batch,
                       step, step_batch)

from . import allocation, assets, bench, camera, config, scene, se3, world     # noqa: E402
from .allocation import HEXAROTOR, QUAD_X, Airframe                # noqa: E402
from .camera import CameraConfig, DepthImageBatch, render        # noqa: E402
from .config import CONFIG_VERSION, load_config                  # noqa: E402
from .world import OBS_DIM, EnvConfig, RewardConfig, SimConfig, StepResult, World  # noqa: E402

__version__ = "0.1.0"
