"""Device-resident World -- drop-in for ``flocksim.world.World``.

SURVEY.md 8(f) ranks 1 and 4: the immediate caller of the hot path.  Mirrors
/root/reference/pkg/src/flocksim/world.py: the same EnvConfig / RewardConfig
schema and validation (config.py:29-90), ``World.create / step / reset_env /
reset_all / observations / privileged_info / camera_mounts`` with
``StepResult`` (observations (E, 16), reward, terminated, truncated,
info{collision, out_of_bounds, nonfinite, autoreset}).  One fused kernel per
step (csrc/fs_world.cu): pending auto-resets, the controller + integrator,
collision (env box and, with obstacles, every collision-enabled primitive),
counters, reward, observations.

Obstacle worlds (asset classes, walls, cameras): prototypes come from the
pools on the host; the per-env prototype picks, every obstacle pose, the
SDF-checked spawn / goal placement and the camera mounts are drawn on the
device at creation and at every reset, and the primitive rows are compiled
there too (csrc/fs_scene.cuh).  ``world.pset`` is the device PrimitiveSet;
``camera.render(world)`` ray-casts it.

Deviation (documented): all draws come from the library's Philox stream
keyed by (seed, env, reset counter), not NumPy's Philox-4x64, so picks,
poses, spawn and goal points differ from the reference's draws; everything
given them is the reference's semantics (tests/test_world_gpu.py,
tests/test_scene_gpu.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import assets as assets_mod
from ._tensors import alloc_planes, default_device, padded, ptr, stride0, stream_handle
from .assets import AssetInstance, AssetPrototype, Primitive
from .camera import CameraConfig
from .control import CommandBatch, ControlGains, ControlLimits
from .dynamics import RigidStateBatch, RobotParams
from .scene import KIND_CODES, PrimitiveSet

OBS_DIM = 16                   # world.py:36
PLACEMENT_ATTEMPTS = 100       # world.py:37
WALL_CLASS = "wall"            # world.py:38
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
    """config.py:93-103."""

    robot: RobotParams = field(default_factory=RobotParams)
    gains: ControlGains = field(default_factory=ControlGains)
    limits: ControlLimits = field(default_factory=ControlLimits)
    env: EnvConfig = field(default_factory=EnvConfig)
    asset_classes: list = field(default_factory=list)
    camera: CameraConfig | None = None
    reward: RewardConfig = field(default_factory=RewardConfig)


@dataclass
class AssetState:
    """Privileged ground-truth state of one obstacle (world.py:56-63)."""

    position: np.ndarray
    rotation: np.ndarray
    class_name: str
    segmentation_id: int


@dataclass
class PrivilegedInfo:
    """Ground-truth obstacle states per environment (world.py:66-70)."""

    per_env: list


def make_wall_prototype(bounds, thickness: float) -> AssetPrototype:
    """Six box slabs just outside the bounding planes of one env (world.py:74-91):
    for each axis, a slab of thickness t centred t/2 outside each face,
    spanning the other two axes plus t on both sides."""
    b = np.asarray(bounds, dtype=np.float64)
    t = float(thickness)
    prims = []
    for axis in range(3):
        size = b + 2.0 * t
        size[axis] = t
        for face in (-t / 2.0, b[axis] + t / 2.0):
            centre = b / 2.0
            centre[axis] = face
            prims.append(Primitive(kind=assets_mod.BOX, dims=tuple(size), position=centre,
                                   rotation=np.array([1.0, 0.0, 0.0, 0.0])))
    return AssetPrototype(source="<walls>", class_name=WALL_CLASS, primitives=prims)


@dataclass
class StepResult:
    """Vectorized step outputs (world.py:45-53); tensors on the device."""

    observations: torch.Tensor   # (E, OBS_DIM)
    reward: torch.Tensor         # (E,)
    terminated: torch.Tensor     # (E,) bool
    truncated: torch.Tensor      # (E,) bool
    info: dict


class World:
    """N parallel single-robot environments on one GPU."""

    def __init__(self, cfg: SimConfig, pools: dict | None = None, device=None,
                 first_env: int = 0):
        self.lib = N.load()
        self.cfg = cfg
        self.robot, self.gains, self.limits = cfg.robot, cfg.gains, cfg.limits
        self.env, self.reward_cfg = cfg.env, cfg.reward
        self.camera = cfg.camera
        self.num_envs = int(cfg.env.num_envs)
        self.dt = float(cfg.env.dt)
        self.bounds = cfg.env.bounds
        self.device = device if device is not None else default_device()
        self.class_by_name = {c.name: c for c in cfg.asset_classes}
        self.pools = dict(pools or {})
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
        self._first_env = int(first_env)
        self._ob = None
        self._clear = None
        self._reset_list = None
        self.pset = PrimitiveSet(n, 0, self.device)
        if cfg.asset_classes or cfg.env.wall_enabled or cfg.camera is not None:
            self._build_obstacles()
        # creation-time placement: reset counter 0 (world.py:160-176)
        self._reset(None, increment=0)

    @classmethod
    def create(cls, cfg: SimConfig, asset_root=None, pools: dict | None = None,
               workers: int = 1, device=None) -> "World":
        """world.py:180-188: pools loaded from asset_root, merged with `pools`."""
        merged = {}
        if asset_root is not None:
            merged.update(assets_mod.load_asset_dir(asset_root))
        if pools:
            merged.update(pools)
        return cls(cfg, pools=merged, device=device)

    # -- obstacle scene ----------------------------------------------------------
    def _build_obstacles(self) -> None:
        """Prototype / class tables, the creation-time picks (device), the
        scene width (max primitive count over envs, scene.py:92), and the
        per-env instance and mount planes."""
        n, dev = self.num_envs, self.device
        protos, classes = [], []
        for c in self.cfg.asset_classes:
            if c.name not in self.pools:
                raise assets_mod.UnknownClassError(f"class '{c.name}' not found in asset pools")
            pool = self.pools[c.name]
            if c.count_per_env > 0 and not pool:
                raise ValueError(f"class '{c.name}' has an empty pool")
            rec = N.fs_asset_class()
            rec.position_min[:] = list(c.position_min)
            rec.position_max[:] = list(c.position_max)
            rec.euler_min[:] = list(c.euler_min)
            rec.euler_max[:] = list(c.euler_max)
            rec.frozen_value[:] = [0.0 if v is None else float(v) for v in c.frozen]
            rec.frozen_mask = sum(1 << i for i, v in enumerate(c.frozen) if v is not None)
            rec.segmentation_id = int(c.segmentation_id)
            rec.collision_enabled = int(bool(c.collision_enabled))
            rec.count_per_env = int(c.count_per_env)
            rec.pool_first, rec.pool_size = len(protos), len(pool)
            protos.extend(pool)
            classes.append(rec)
        wall_proto = -1
        if self.env.wall_enabled:
            wall_proto = len(protos)
            protos.append(make_wall_prototype(self.bounds, self.env.wall_thickness))
        self._protos = protos
        offsets = np.zeros(len(protos) + 1, dtype=np.int32)
        flat = []
        for i, pr in enumerate(protos):
            for prim in pr.primitives:
                rec = N.fs_proto_prim()
                rec.kind = KIND_CODES[prim.kind]
                rec.dims[:] = [float(x) for x in prim.dims]
                rec.position[:] = [float(x) for x in prim.position]
                rec.rotation[:] = [float(x) for x in prim.rotation]
                flat.append(rec)
            offsets[i + 1] = offsets[i] + len(pr.primitives)
        self._t_classes = _struct_tensor(N.fs_asset_class, classes, dev)
        self._t_protos = _struct_tensor(N.fs_proto_prim, flat, dev)
        self._t_offsets = torch.from_numpy(offsets).to(dev)
        self.instances_per_env = sum(c.count_per_env for c in self.cfg.asset_classes)
        s = padded(n)
        j = self.instances_per_env
        self._inst_proto = torch.zeros((max(j, 1), s), dtype=torch.int32, device=dev)
        self._inst_pose = torch.zeros((max(7 * j, 1), s), dtype=torch.float64, device=dev)
        self._mount = None
        ob = N.fs_obstacles()
        ob.num_classes = len(classes)
        ob.instances_per_env = j
        ob.classes = ptr(self._t_classes)
        ob.proto_offset = ptr(self._t_offsets)
        ob.proto_prims = ptr(self._t_protos)
        ob.inst_proto = ptr(self._inst_proto)
        # the pose planes are filled on demand (World.instances ->
        # fs_obstacles_poses); the step's resets leave them alone (12 us of
        # scattered float64 stores per step at 2^21 forest envs)
        ob.inst_pose = None
        ob.wall_proto = wall_proto
        ob.wall_seg = int(self.env.wall_segmentation_id)
        if self.camera is not None:
            cam = self.camera
            self._mount = torch.zeros((7, s), dtype=torch.float64, device=dev)
            ob.mount = ptr(self._mount)
            ob.mount_stride = s
            ob.mount_position[:] = list(cam.mount_position)
            ob.mount_euler[:] = list(cam.mount_euler)
            ob.randomize_position[:] = list(cam.randomize_position)
            ob.randomize_euler[:] = list(cam.randomize_euler)
        ob.scene = self.pset.native()
        ob.plane_stride = s
        counts = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        with torch.cuda.device(dev):
            N.check(self.lib.fs_obstacles_pick(C.byref(ob), n, self._first_env,
                                               int(self.env.seed), ptr(counts),
                                               stream_handle()), "fs_obstacles_pick")
        width = int(counts[:n].max().item()) if n else 0
        self.pset = PrimitiveSet(n, width, dev)
        ob.scene = self.pset.native()
        # instance broad phase for the collision test (written by every reset;
        # the device's warp reset handles up to 63 instances + walls per env)
        self._inst_box = None
        self._clear = None
        if 0 < j and j + 1 <= 64 and width < (1 << 15):
            # J records of two float4 per env, instance-major planes of
            # plane_stride envs: record (j, half) of env e at [2 j + half, e]
            self._inst_box = torch.zeros((2 * j, s, 4), dtype=torch.float32, device=dev)
            ob.inst_box = ptr(self._inst_box)
            # collision clearance cache (fs_obstacles.clear): starts invalid;
            # the deferred-collision worklist (count, blocks done, env ids)
            self._clear = torch.full((4, s), -1.0, dtype=torch.float32, device=dev)
            ob.clear = ptr(self._clear)
            self._worklist = torch.zeros(n + 3, dtype=torch.int32, device=dev)
            ob.worklist = ptr(self._worklist)
            # running total of the slot records the deferred test walked
            self._walk_slots = torch.zeros(1, dtype=torch.int64, device=dev)
            ob.walk_slots = ptr(self._walk_slots)
            # the pending envs a step skips (fs_obstacles.reset_list): their
            # auto-resets run after the step, with the deferred collision test
            self._reset_list = torch.zeros(n + 4, dtype=torch.int32, device=dev)
            ob.reset_list = ptr(self._reset_list)
        self._ob = ob
        self._desc.obstacles = C.pointer(ob)

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
        failed = (self._info[:self.num_envs] & N.FS_INFO_PLACEMENT_FAILED) != 0
        if mask is not None:
            failed &= mask[:self.num_envs] != 0
        if bool(failed.any()):
            e = int(torch.nonzero(failed)[0, 0])
            raise PlacementFailureError(
                f"no collision-free robot/goal pose in env {e} after "
                f"{PLACEMENT_ATTEMPTS} attempts")

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

    @property
    def instances(self) -> list:
        """Per-env AssetInstance lists rebuilt from the device (world.py:165-176):
        randomizable instances in class order, then the walls."""
        if self._ob is None:
            return [[] for _ in range(self.num_envs)]
        n, j = self.num_envs, self.instances_per_env
        protos = self._inst_proto[:j, :n].cpu().numpy()
        pose = None
        if j:
            ob = N.fs_obstacles.from_buffer_copy(self._ob)
            ob.inst_pose = ptr(self._inst_pose)
            bounds = (C.c_double * 3)(*[float(x) for x in self.env.bounds])
            with torch.cuda.device(self.device):
                N.check(self.lib.fs_obstacles_poses(C.byref(ob), n, self._first_env,
                                                    int(self.env.seed), ptr(self._counter),
                                                    bounds, stream_handle()),
                        "fs_obstacles_poses")
            pose = self._inst_pose[:7 * j, :n].cpu().numpy().reshape(j, 7, n)
        classes = [c for c in self.cfg.asset_classes for _ in range(c.count_per_env)]
        wall = self._protos[-1] if self.env.wall_enabled else None
        out = []
        for e in range(n):
            env = [AssetInstance(prototype=self._protos[int(protos[i, e])],
                                 position=pose[i, 0:3, e], rotation=pose[i, 3:7, e],
                                 segmentation_id=c.segmentation_id, env_index=e,
                                 class_name=c.name, collision_enabled=c.collision_enabled)
                   for i, c in enumerate(classes)]
            if wall is not None:
                env.append(AssetInstance(prototype=wall, position=np.zeros(3),
                                         rotation=np.array([1.0, 0.0, 0.0, 0.0]),
                                         segmentation_id=self.env.wall_segmentation_id,
                                         env_index=e, class_name=WALL_CLASS))
            out.append(env)
        return out

    def privileged_info(self) -> PrivilegedInfo:
        """Ground-truth obstacle states per env, walls included (world.py:344-353)."""
        return PrivilegedInfo(per_env=[
            [AssetState(position=i.position, rotation=i.rotation, class_name=i.class_name,
                        segmentation_id=i.segmentation_id) for i in env]
            for env in self.instances])

    def mount_planes(self, cfg: CameraConfig):
        """(7, stride) float64 device planes of the randomized camera mounts
        when cfg is this world's camera, else None (nominal mount)."""
        if cfg is self.camera and self._ob is not None and self._mount is not None:
            return self._mount
        return None

    def camera_mounts(self, cfg: CameraConfig):
        """Per-robot camera mounts (world.py:355-361): the randomized ones
        when cfg is the world's camera, else cfg's nominal mount broadcast."""
        planes = self.mount_planes(cfg)
        n = self.num_envs
        if planes is not None:
            return planes[0:3, :n].T, planes[3:7, :n].T
        return (np.broadcast_to(cfg.mount_position, (n, 3)),
                np.broadcast_to(cfg.mount_rotation, (n, 4)))

    # -- resets ----------------------------------------------------------------
    def reset_env(self, e: int) -> None:
        """Re-randomize env e's obstacles and respawn its robot and goal
        (world.py:229-243)."""
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
        """StepResult views; raises PlacementFailureError when an auto-reset of
        this step found no free pose, as the reference's step does through
        reset_env -> _find_free_point (world.py:200-211, 287-289).  That check
        is one device reduction and one host sync; step_async skips it (the
        bit stays readable as info['placement_failed'])."""
        n = self.num_envs
        info = self._info[:n]
        failed = (info & N.FS_INFO_PLACEMENT_FAILED) != 0
        if bool(failed.any()):
            e = int(torch.nonzero(failed)[0, 0])
            raise PlacementFailureError(
                f"no collision-free robot/goal pose in env {e} after "
                f"{PLACEMENT_ATTEMPTS} attempts (auto-reset)")
        return StepResult(
            observations=self.observations(), reward=self._reward[:n],
            terminated=(info & N.FS_INFO_TERMINATED) != 0,
            truncated=(info & N.FS_INFO_TRUNCATED) != 0,
            info={"collision": (info & N.FS_INFO_COLLISION) != 0,
                  "out_of_bounds": (info & N.FS_INFO_OUT_OF_BOUNDS) != 0,
                  "nonfinite": (info & N.FS_INFO_NONFINITE) != 0,
                  "autoreset": (info & N.FS_INFO_AUTORESET) != 0,
                  "placement_failed": failed})

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

    def load(self, state=None, goals=None, pending=None, steps=None, scene=None,
             mounts=None) -> None:
        """Overwrite world arrays (testing / checkpoint restore): planar
        (13, E) state, (3, E) goals, (E,) pending flags and step counters;
        `scene`: a dict of host PrimitiveSet arrays (E, K, ...) -- e.g. a
        reference world's pset -- replacing the obstacle rows (the width may
        change); `mounts`: (mount_p (E, 3), mount_q (E, 4)) camera mounts."""
        n = self.num_envs
        if scene is not None:
            k = int(np.asarray(scene["kind"]).shape[1])
            pset = PrimitiveSet(n, k, self.device)
            pset.load_arrays(scene["kind"], scene["dims"], scene["position"], scene["rot"],
                             scene["seg_id"], scene["collision"], scene.get("aabb_min"),
                             scene.get("aabb_max"))
            self.pset = pset
            if self._ob is None:
                ob = N.fs_obstacles()
                self._t_offsets = torch.zeros(1, dtype=torch.int32, device=self.device)
                ob.proto_offset = ptr(self._t_offsets)
                ob.plane_stride = padded(n)
                ob.wall_proto = -1
                self._mount = None
                self._protos = []
                self.instances_per_env = 0
                self._ob = ob
            self._ob.scene = pset.native()
            # the loaded rows are not described by the instance tables
            self._ob.inst_box = None
            self._ob.clear = None
            self._ob.worklist = None
            self._ob.reset_list = None
            self._ob.walk_slots = None
            self._clear = None
            self._reset_list = None
            self._desc.obstacles = C.pointer(self._ob)
        if mounts is not None:
            if self._mount is None:
                raise ValueError("world has no camera mounts")
            mp, mq = (np.asarray(m, dtype=np.float64) for m in mounts)
            self._mount[0:3, :n].copy_(torch.from_numpy(mp.T.copy()))
            self._mount[3:7, :n].copy_(torch.from_numpy(mq.T.copy()))
        if state is not None:
            self._state[:, :n].copy_(torch.as_tensor(np.asarray(state), dtype=torch.float32))
        if getattr(self, "_clear", None) is not None and (state is not None or scene is not None):
            self._clear[3].fill_(-1.0)        # rewritten positions: the cache is stale
        if goals is not None:
            self._goal[:, :n].copy_(torch.as_tensor(np.asarray(goals), dtype=torch.float32))
        if pending is not None:
            # (the next streaming step skips and lists every env pending then)
            self._pending[:n].copy_(torch.as_tensor(np.asarray(pending, dtype=np.uint8)))
        if steps is not None:
            self._steps[:n].copy_(torch.as_tensor(np.asarray(steps, dtype=np.int32)))


def _struct_tensor(ctype, records: list, device) -> torch.Tensor:
    """ctypes records -> one uint8 device tensor (at least one byte)."""
    arr = (ctype * max(len(records), 1))(*records)
    raw = np.frombuffer(bytes(arr), dtype=np.uint8).copy()
    return torch.from_numpy(raw).to(device)
