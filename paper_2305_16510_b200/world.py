"""Device-resident free-space World -- drop-in for ``flocksim.world.World``.

SURVEY.md 8(f) rank 1: the immediate caller of the hot path.  Mirrors
/root/reference/pkg/src/flocksim/world.py for worlds without obstacles or
camera (asset_classes empty, camera None): the same EnvConfig / RewardConfig
schema and validation (config.py:29-90), ``World.create / step / reset_env /
reset_all / observations`` with ``StepResult`` (observations (E, 16), reward,
terminated, truncated, info{collision, out_of_bounds, nonfinite, autoreset}).
One fused kernel per step (csrc/fs_world.cu): pending auto-resets, the
controller + integrator, box collision, counters, reward, observations.

Deviation (documented): re-spawn points come from the library's Philox
stream keyed by (seed, env, reset counter), not NumPy's Philox-4x64, so the
spawn and goal points differ from the reference's draws; everything given
the points is the reference's semantics (tests/test_world_gpu.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._tensors import alloc_planes, default_device, ptr, stride0, stream_handle
from .control import CommandBatch, ControlGains, ControlLimits
from .dynamics import RigidStateBatch, RobotParams

OBS_DIM = 16                   # world.py:36
PLACEMENT_ATTEMPTS = 100       # world.py:37
CONTROL_MODES = ("attitude", "velocity")   # config.py:23


class ConfigError(ValueError):
    """Malformed or out-of-range configuration content (config.py:26-27)."""


class PlacementFailureError(RuntimeError):
    """No collision-free spawn found within the attempt budget (world.py:41-42)."""


@dataclass
class EnvConfig:
    """World layout (config.py:29-79); the same fields and validation."""

    num_envs: int = 16
    bounds: np.ndarray = field(default_factory=lambda: np.array([10.0, 10.0, 5.0]))
    episode_max_steps: int = 1000
    dt: float = 0.01
    control_mode: str = "velocity"
    seed: int = 0
    wall_enabled: bool = False
    wall_thickness: float = 0.1
    wall_segmentation_id: int = 1
    goal_min: np.ndarray = field(default_factory=lambda: np.array([0.1, 0.1, 0.2]))
    goal_max: np.ndarray = field(default_factory=lambda: np.array([0.9, 0.9, 0.8]))
    spawn_min: np.ndarray = field(default_factory=lambda: np.array([0.1, 0.1, 0.2]))
    spawn_max: np.ndarray = field(default_factory=lambda: np.array([0.9, 0.9, 0.8]))

    def __post_init__(self):
        self.bounds = np.asarray(self.bounds, dtype=np.float64).reshape(3)
        for name in ("goal_min", "goal_max", "spawn_min", "spawn_max"):
            setattr(self, name, np.asarray(getattr(self, name), dtype=np.float64).reshape(3))
        if self.num_envs < 1:
            raise ConfigError("num_envs must be >= 1")
        if (self.bounds <= 0.0).any():
            raise ConfigError("env bounds must be positive")
        if not 0.0 < self.dt <= 0.1:
            raise ConfigError(f"dt must be in (0, 0.1], got {self.dt}")
        if self.episode_max_steps < 1:
            raise ConfigError("episode_max_steps must be >= 1")
        if self.control_mode not in CONTROL_MODES:
            raise ConfigError(f"control_mode must be one of {CONTROL_MODES}")
        for lo, hi in (("goal_min", "goal_max"), ("spawn_min", "spawn_max")):
            a, b = getattr(self, lo), getattr(self, hi)
            if (a > b).any() or (a < 0).any() or (b > 1).any():
                raise ConfigError(f"{lo}/{hi} must satisfy 0 <= min <= max <= 1")
        if self.wall_thickness <= 0.0:
            raise ConfigError("wall_thickness must be positive")
        if self.wall_segmentation_id < 1:
            raise ConfigError("wall_segmentation_id must be >= 1")


@dataclass
class RewardConfig:
    """Goal-reaching reward constants (config.py:82-90)."""

    c_dist: float = 0.1
    c_vel: float = 0.01
    c_step: float = 0.01
    c_success: float = 10.0
    c_crash: float = 10.0
    success_radius: float = 0.2


@dataclass
class SimConfig:
    """config.py:93-103 (asset classes and camera: not supported here)."""

    robot: RobotParams = field(default_factory=RobotParams)
    gains: ControlGains = field(default_factory=ControlGains)
    limits: ControlLimits = field(default_factory=ControlLimits)
    env: EnvConfig = field(default_factory=EnvConfig)
    asset_classes: list = field(default_factory=list)
    camera: object | None = None
    reward: RewardConfig = field(default_factory=RewardConfig)


@dataclass
class StepResult:
    """Vectorized step outputs (world.py:45-53); tensors on the device."""

    observations: torch.Tensor   # (E, OBS_DIM)
    reward: torch.Tensor         # (E,)
    terminated: torch.Tensor     # (E,) bool
    truncated: torch.Tensor      # (E,) bool
    info: dict


class World:
    """N parallel single-robot free-space environments on one GPU."""

    def __init__(self, cfg: SimConfig, device=None, first_env: int = 0):
        if cfg.asset_classes:
            raise ConfigError("obstacles (asset_classes) are out of scope for the GPU World")
        if cfg.camera is not None:
            raise ConfigError("cameras are out of scope for the GPU World")
        self.lib = N.load()
        self.cfg = cfg
        self.robot, self.gains, self.limits = cfg.robot, cfg.gains, cfg.limits
        self.env, self.reward_cfg = cfg.env, cfg.reward
        self.num_envs = int(cfg.env.num_envs)
        self.dt = float(cfg.env.dt)
        self.bounds = cfg.env.bounds
        self.device = device if device is not None else default_device()
        n = self.num_envs
        self._state = alloc_planes(13, n, self.device, zero=True)
        self._goal = alloc_planes(3, n, self.device, zero=True)
        self._obs = alloc_planes(OBS_DIM, n, self.device, zero=True)
        z32 = lambda: torch.zeros(max(n, 1), dtype=torch.int32, device=self.device)
        self._steps = z32()
        self._counter = z32()
        self._pending = torch.zeros(max(n, 1), dtype=torch.uint8, device=self.device)
        self._reward = torch.zeros(max(n, 1), dtype=torch.float32, device=self.device)
        self._info = torch.zeros(max(n, 1), dtype=torch.uint8, device=self.device)
        self._cmd = alloc_planes(8, n, self.device, zero=True)
        self._robot = self.robot.native()
        self._gains_c = self.gains.native()
        self._limits_c = self.limits.native()
        self._wcfg = self._world_cfg()
        self._desc = self._make_desc(first_env)
        # creation-time placement: reset counter 0 (world.py:160-176)
        self._reset(None, increment=0)

    @classmethod
    def create(cls, cfg: SimConfig, asset_root=None, pools: dict | None = None,
               workers: int = 1, device=None) -> "World":
        """world.py:180-188; asset_root / pools are accepted for signature
        compatibility and must be empty (no obstacles)."""
        if asset_root is not None or pools:
            raise ConfigError("obstacle pools are out of scope for the GPU World")
        return cls(cfg, device=device)

    # -- plumbing -------------------------------------------------------------
    def _world_cfg(self) -> N.fs_world_cfg:
        c = N.fs_world_cfg()
        e, r = self.env, self.reward_cfg
        c.bounds[:] = [float(x) for x in e.bounds]
        c.spawn_lo[:] = [float(x) for x in e.spawn_min]
        c.spawn_hi[:] = [float(x) for x in e.spawn_max]
        c.goal_lo[:] = [float(x) for x in e.goal_min]
        c.goal_hi[:] = [float(x) for x in e.goal_max]
        c.collision_radius = float(self.robot.collision_radius)
        c.episode_max_steps = int(e.episode_max_steps)
        c.placement_attempts = PLACEMENT_ATTEMPTS
        c.c_dist, c.c_vel, c.c_step = r.c_dist, r.c_vel, r.c_step
        c.c_success, c.c_crash, c.success_radius = r.c_success, r.c_crash, r.success_radius
        return c

    def _make_desc(self, first_env) -> N.fs_world_desc:
        w = N.fs_world_desc()
        d = w.step
        d.n = self.num_envs
        d.first_id = first_env
        d.state_in = d.state_out = ptr(self._state)
        d.state_in_stride = d.state_out_stride = stride0(self._state)
        d.mode = N.FS_MODE_VELOCITY if self.env.control_mode == "velocity" else N.FS_MODE_ATTITUDE
        d.integrate = 1
        d.cmd = ptr(self._cmd)
        d.cmd_stride = stride0(self._cmd)
        d.dt = self.dt
        d.seed = int(self.env.seed)
        w.goal = ptr(self._goal)
        w.goal_stride = stride0(self._goal)
        w.steps_in_episode = ptr(self._steps)
        w.reset_counter = ptr(self._counter)
        w.pending_reset = ptr(self._pending)
        w.obs = ptr(self._obs)
        w.obs_stride = stride0(self._obs)
        w.reward = ptr(self._reward)
        w.info = ptr(self._info)
        return w

    def _reset(self, mask, increment: int) -> None:
        with torch.cuda.device(self.device):
            N.check(self.lib.fs_world_reset(C.byref(self._desc), self._wcfg, ptr(mask), increment,
                                            stream_handle()), "fs_world_reset")
        if bool((self._info[:self.num_envs] & N.FS_INFO_PLACEMENT_FAILED).any()):
            raise PlacementFailureError(
                f"no collision-free pose after {PLACEMENT_ATTEMPTS} attempts")

    # -- views -----------------------------------------------------------------
    @property
    def states(self) -> RigidStateBatch:
        return RigidStateBatch.from_planes(self._state, self.num_envs)

    @property
    def goals(self) -> torch.Tensor:
        return self._goal[:, :self.num_envs].T

    @property
    def steps_in_episode(self) -> torch.Tensor:
        return self._steps[:self.num_envs]

    @property
    def pending_reset(self) -> torch.Tensor:
        return self._pending[:self.num_envs].bool()

    @property
    def reset_counter(self) -> torch.Tensor:
        return self._counter[:self.num_envs]

    def observations(self) -> torch.Tensor:
        """Flat observations in the documented 16-value layout (world.py:331-342)."""
        return self._obs[:, :self.num_envs].T

    def privileged_info(self):
        """No obstacles: an empty list per environment (world.py:344-353)."""
        return [[] for _ in range(self.num_envs)]

    # -- resets ----------------------------------------------------------------
    def reset_env(self, e: int) -> None:
        """Respawn env e's robot and goal (world.py:229-243)."""
        if not 0 <= e < self.num_envs:
            raise IndexError(f"env index {e} out of range")
        mask = torch.zeros(max(self.num_envs, 1), dtype=torch.uint8, device=self.device)
        mask[e] = 1
        self._reset(mask, increment=1)

    def reset_all(self) -> torch.Tensor:
        """Reset every environment; returns the fresh observations (world.py:245-249)."""
        self._reset(None, increment=1)
        return self.observations()

    # -- stepping ----------------------------------------------------------------
    def step_async(self, commands: CommandBatch, stream=None) -> None:
        """Launch one World.step without building the StepResult views (for
        CUDA-graph capture and benchmarking)."""
        if commands.n != self.num_envs:
            raise ValueError(f"expected {self.num_envs} commands, got {commands.n}")
        mode, view = commands.kernel_mode()
        d = self._desc.step
        d.mode = mode
        d.cmd = ptr(view)
        d.cmd_stride = stride0(view)
        d.mode_per_vehicle = ptr(commands.mode) if mode == N.FS_MODE_MIXED else None
        with torch.cuda.device(self.device):
            N.check(self.lib.fs_world_step(C.byref(self._desc), self._wcfg, self._robot,
                                           self._gains_c, self._limits_c,
                                           stream or stream_handle()), "fs_world_step")

    def step(self, commands: CommandBatch) -> StepResult:
        """Advance all environments by one control + dynamics step (world.py:277-326)."""
        self.step_async(commands)
        return self._result()

    def _result(self) -> StepResult:
        n = self.num_envs
        info = self._info[:n]
        return StepResult(
            observations=self.observations(), reward=self._reward[:n],
            terminated=(info & N.FS_INFO_TERMINATED) != 0,
            truncated=(info & N.FS_INFO_TRUNCATED) != 0,
            info={"collision": (info & N.FS_INFO_COLLISION) != 0,
                  "out_of_bounds": (info & N.FS_INFO_OUT_OF_BOUNDS) != 0,
                  "nonfinite": (info & N.FS_INFO_NONFINITE) != 0,
                  "autoreset": (info & N.FS_INFO_AUTORESET) != 0})

    # -- RL actions (flocksim_rl) ---------------------------
    def step_actions_async(self, actions: torch.Tensor, stream=None) -> None:
        """One World.step driven by normalized actions: (E, 4) float32 or
        float64 rows on this device, clipped to [-1, 1] and denormalized in
        float64 inside the kernel exactly as vec_env.py:85-104 does.  No
        validation beyond the layout (see rl.VecEnvHandle.step)."""
        if actions.dtype == torch.float32:
            code = N.FS_DTYPE_F32
        elif actions.dtype == torch.float64:
            code = N.FS_DTYPE_F64
        else:
            raise TypeError(f"actions must be float32 or float64, got {actions.dtype}")
        if actions.dim() != 2 or actions.shape != (self.num_envs, 4):
            raise ValueError(f"expected actions of shape {(self.num_envs, 4)}, "
                             f"got {tuple(actions.shape)}")
        if actions.device != torch.device(self.device):
            raise ValueError(f"actions on {actions.device}, world on {self.device}")
        if actions.stride(1) != 1 or actions.stride(0) % 4 or actions.data_ptr() % 16:
            # the kernel loads each row as 16-B vectors: repack into a fresh
            # (aligned) allocation
            actions = torch.empty(actions.shape, dtype=actions.dtype,
                                  device=actions.device).copy_(actions)
        d = self._desc.step
        d.mode = N.FS_MODE_VELOCITY if self.env.control_mode == "velocity" else N.FS_MODE_ATTITUDE
        d.mode_per_vehicle = None
        with torch.cuda.device(self.device):
            N.check(self.lib.fs_vecenv_step(C.byref(self._desc), self._wcfg, self._robot,
                                            self._gains_c, self._limits_c, ptr(actions), code,
                                            actions.stride(0), stream or stream_handle()),
                    "fs_vecenv_step")

    def step_actions(self, actions: torch.Tensor) -> StepResult:
        """step_actions_async + the StepResult views."""
        self.step_actions_async(actions)
        return self._result()

    def load(self, state=None, goals=None, pending=None, steps=None) -> None:
        """Overwrite world arrays (testing / checkpoint restore): planar
        (13, E) state, (3, E) goals, (E,) pending flags and step counters."""
        n = self.num_envs
        if state is not None:
            self._state[:, :n].copy_(torch.as_tensor(np.asarray(state), dtype=torch.float32))
        if goals is not None:
            self._goal[:, :n].copy_(torch.as_tensor(np.asarray(goals), dtype=torch.float32))
        if pending is not None:
            self._pending[:n].copy_(torch.as_tensor(np.asarray(pending, dtype=np.uint8)))
        if steps is not None:
            self._steps[:n].copy_(torch.as_tensor(np.asarray(steps, dtype=np.int32)))
