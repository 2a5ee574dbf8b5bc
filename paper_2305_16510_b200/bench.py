"""Benchmark harness of the control step and the depth camera -- the B200
counterpart of flocksim.bench (pkg/src/flocksim/bench.py:1-236).

Same names, arguments, validation and report fields as the reference:
`bench_dynamics` times the controller + integrator pipeline on the batch
`make_bench_batch` draws (bench.py:117-143, 152-173), `bench_render` times
depth rendering of the cluttered `bench_scene_config` scene (bench.py:184-236),
and both return a `BenchReport` (bench.py:51-99).  What differs is where the
work runs: the batch lives in HBM as fp32 planes, the steps run as one
persistent `fs_step_many` launch (or one fused `fs_step` launch per step for
batches below the streaming kernel's size), and `wall_seconds` is the device
time of the timed steps measured with CUDA events on the launching stream,
after a synchronize on both sides.  `workers` is accepted for API parity: the
GPU partitions the batch itself (the reference's `workers` only splits
step_batch over host threads, bench.py:146-149).

`state_checksum` hashes the fp32 state, so it is reproducible run to run and
across launch paths and shardings (the kernels are deterministic), but it is
not the reference's float64 checksum: the two agree to the parity bar
(SURVEY.md 8(c)), not bitwise.
"""

from __future__ import annotations

import hashlib
import json
import os
import platform
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from ._tensors import default_device
from .control import (AttitudeCommands, CommandBatch, ControlGains, ControlLimits,
                      VelocityCommands, fused_step)
from .dynamics import RigidStateBatch, RobotParams

DEFAULT_DT = 0.01
WARMUP_STEPS = 100
MODES = ("attitude", "velocity")


def machine_descriptor(device=None) -> str:
    """bench.py:46-49, plus the GPU the steps ran on."""
    gpu = ""
    if torch.cuda.is_available():
        dev = device if device is not None else default_device()
        gpu = f", {torch.cuda.get_device_name(dev)}"
    return (f"{platform.system()} {platform.machine()}, {os.cpu_count()} cores, "
            f"python {platform.python_version()}, numpy {np.__version__}, "
            f"torch {torch.__version__}{gpu}")


@dataclass
class BenchReport:
    """Timing summary; steps_per_second aggregates across environments
    (bench.py:51-99)."""

    num_envs: int
    total_steps: int          # per-env iterations
    wall_seconds: float       # device time of the timed steps
    steps_per_second: float   # total_steps * num_envs / wall_seconds
    sim_to_real_ratio: float  # steps_per_second * dt
    dt: float
    checksum: str
    machine: str = field(default_factory=machine_descriptor)
    frames_per_second: float | None = None
    resolution: tuple | None = None
    workers: int = 1
    mode: str = ""
    engine: str = ""          # how the timed steps were launched

    def to_dict(self) -> dict:
        d = dict(self.__dict__)
        if self.resolution is not None:
            d["resolution"] = list(self.resolution)
        return d

    def write_json(self, path) -> None:
        Path(path).write_text(json.dumps(self.to_dict(), indent=2) + "\n")

    def summary(self) -> str:
        lines = [f"envs:             {self.num_envs}"]
        if self.mode:
            lines.append(f"mode:             {self.mode}")
        if self.frames_per_second is not None:
            lines += [
                f"frames per env:   {self.total_steps}",
                f"wall time:        {self.wall_seconds:.3f} s",
                f"resolution:       {self.resolution[0]}x{self.resolution[1]}",
                f"render rate:      {self.frames_per_second:,.1f} frames/s",
            ]
        else:
            lines += [
                f"steps per env:    {self.total_steps}",
                f"wall time:        {self.wall_seconds:.3f} s",
                f"aggregate rate:   {self.steps_per_second:,.0f} env-steps/s",
                f"sim-to-real:      {self.sim_to_real_ratio:,.1f}x",
                f"dt per step:      {self.dt * 1e3:.0f} ms",
            ]
        lines += [
            f"workers:          {self.workers}",
            f"engine:           {self.engine}",
            f"checksum:         {self.checksum}",
            f"machine:          {self.machine}",
        ]
        return "\n".join(lines)


def state_checksum(states: RigidStateBatch) -> str:
    """sha256 of p, q, v, omega as row-major fp32 arrays (bench.py:102-106)."""
    h = hashlib.sha256()
    for arr in (states.p, states.q, states.v, states.omega):
        h.update(np.ascontiguousarray(arr.detach().cpu().numpy()).tobytes())
    return h.hexdigest()


def image_checksum(depth, seg) -> str:
    """bench.py:109-113 on the device images (copied to the host)."""
    h = hashlib.sha256()
    for a in (depth, seg):
        a = a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _check_mode(mode: str) -> None:
    if mode not in MODES:
        raise ValueError(f"mode must be 'attitude' or 'velocity', got '{mode}'")


def make_bench_batch(num_envs: int, seed: int, mode: str, params: RobotParams,
                     device=None) -> tuple[RigidStateBatch, CommandBatch]:
    """Initial states and the fixed command of the dynamics benchmark
    (bench.py:117-143): the reference's own NumPy draws, in the same order,
    moved to the device as fp32 planes."""
    _check_mode(mode)
    from . import se3
    dev = device if device is not None else default_device()
    rng = np.random.default_rng(seed)
    n = num_envs
    p = rng.uniform(-1.0, 1.0, (n, 3))
    rot = rng.uniform(-0.1, 0.1, (n, 3))
    v = rng.uniform(-0.2, 0.2, (n, 3))
    w = rng.uniform(-0.1, 0.1, (n, 3))
    q = se3.exp_so3(torch.as_tensor(rot, dtype=torch.float64, device=dev))
    states = RigidStateBatch(p=p, q=q, v=v, omega=w, device=dev)
    if mode == "attitude":
        cmds = CommandBatch.all_attitude(AttitudeCommands(
            roll=np.full(n, 0.05), pitch=np.full(n, -0.05), yaw_rate=np.full(n, 0.2),
            thrust=np.full(n, params.hover_thrust), device=dev))
    else:
        cmds = CommandBatch.all_velocity(VelocityCommands(
            v=np.tile([0.5, 0.3, 0.1], (n, 1)), yaw_rate=np.full(n, 0.2), device=dev))
    return states, cmds


def _pipeline_step(states, cmds, gains, params, limits, dt, workers=1):
    """control_batch + step_batch (bench.py:146-149) as one fused kernel."""
    out, _ = fused_step(states, cmds, gains, params, dt, limits, want_flags=False)
    return out


def _fleet_for(states: RigidStateBatch, cmds: CommandBatch, mode: str, dt: float, params,
               gains, limits):
    """A device fleet holding exactly this batch (the engine of the timed loop)."""
    from .fleet import Fleet
    n = states.n
    f = Fleet(n, mode=mode, dt=dt, params=params, gains=gains, limits=limits,
              device=states.device)
    f.state[:, :n].copy_(states.buf[:, :n])
    _, view = cmds.kernel_mode()
    f.cmd[:4, :n].copy_(view[:, :n])
    return f


def bench_dynamics(num_envs: int, steps: int, mode: str = "attitude", seed: int = 0,
                   workers: int = 1, dt: float = DEFAULT_DT, warmup: int = WARMUP_STEPS,
                   device=None) -> BenchReport:
    """Time the controller + integrator pipeline on an obstacle-free batch
    (bench.py:152-173).  Arguments are validated before any device work."""
    if num_envs < 1:
        raise ValueError("num_envs must be >= 1")
    _check_mode(mode)
    if not 0.0 < dt <= 0.1:
        raise ValueError(f"dt must be in (0, 0.1], got {dt}")
    params, gains, limits = RobotParams(), ControlGains(), ControlLimits()
    states, cmds = make_bench_batch(num_envs, seed, mode, params, device)
    fleet = _fleet_for(states, cmds, mode, dt, params, gains, limits)
    persistent = fleet.chainable
    engine = ("fs_step_many (one persistent launch)" if persistent
              else "fs_step (one fused launch per step)")
    dev = fleet.device
    with torch.cuda.device(dev):
        if warmup > 0:
            fleet.rollout(warmup, persistent=persistent)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if steps > 0:
            fleet.rollout(steps, persistent=persistent)
        e1.record()
        torch.cuda.synchronize(dev)
        wall = e0.elapsed_time(e1) * 1e-3
    rate = steps * num_envs / wall if wall > 0 else float("inf")
    return BenchReport(num_envs=num_envs, total_steps=steps, wall_seconds=wall,
                       steps_per_second=rate, sim_to_real_ratio=rate * dt, dt=dt,
                       checksum=state_checksum(fleet.states()), workers=workers, mode=mode,
                       engine=engine, machine=machine_descriptor(dev))


_BENCH_SPHERE = ('<robot name="s{i}"><link name="l"><collision><geometry>'
                 '<sphere radius="{r}"/></geometry></collision></link></robot>')
_BENCH_BOX = ('<robot name="b{i}"><link name="l"><collision><geometry>'
              '<box size="{x} {y} {z}"/></geometry></collision></link></robot>')
_BENCH_CYL = ('<robot name="c{i}"><link name="l"><collision><geometry>'
              '<cylinder radius="{r}" length="{h}"/></geometry></collision>'
              '</link></robot>')


def bench_scene_config(num_envs: int, seed: int):
    """The cluttered render-benchmark scene (bench.py:184-214): 3 sphere, 3 box
    and 2 pillar prototypes; 5 + 5 + 4 instances per env in walled 10x10x5 m
    envs.  Returns (SimConfig, pools)."""
    from .assets import AssetClassConfig, parse_urdf_subset
    from .world import EnvConfig, SimConfig
    pools = {
        "spheres": [parse_urdf_subset(_BENCH_SPHERE.format(i=i, r=0.3 + 0.15 * i),
                                      class_name="spheres") for i in range(3)],
        "boxes": [parse_urdf_subset(
            _BENCH_BOX.format(i=i, x=0.4 + 0.2 * i, y=0.5, z=0.8 + 0.3 * i),
            class_name="boxes") for i in range(3)],
        "pillars": [parse_urdf_subset(_BENCH_CYL.format(i=i, r=0.15 + 0.05 * i, h=3.0),
                                      class_name="pillars") for i in range(2)],
    }
    classes = [
        AssetClassConfig(name="spheres", count_per_env=5, segmentation_id=2,
                         position_min=[0.1, 0.1, 0.1], position_max=[0.9, 0.9, 0.9]),
        AssetClassConfig(name="boxes", count_per_env=5, segmentation_id=3,
                         position_min=[0.1, 0.1, 0.0], position_max=[0.9, 0.9, 0.6],
                         euler_min=[0, 0, -3.1], euler_max=[0, 0, 3.1]),
        AssetClassConfig(name="pillars", count_per_env=4, segmentation_id=4,
                         frozen=(None, None, 1.5)),
    ]
    cfg = SimConfig(env=EnvConfig(num_envs=num_envs, bounds=[10.0, 10.0, 5.0], seed=seed,
                                  wall_enabled=True, wall_segmentation_id=1),
                    asset_classes=classes)
    return cfg, pools


def bench_render(num_envs: int, frames: int, cam_cfg=None, seed: int = 0, workers: int = 1,
                 device=None) -> BenchReport:
    """Time depth rendering of a static cluttered scene (bench.py:217-236);
    one warm-up frame (checksummed) is not timed."""
    if num_envs < 1 or frames < 1:
        raise ValueError("num_envs and frames must be >= 1")
    from .camera import CameraConfig, render
    from .world import World
    cam = cam_cfg if cam_cfg is not None else CameraConfig()
    cfg, pools = bench_scene_config(num_envs, seed)
    world = World.create(cfg, pools=pools, device=device)
    img = render(world, cam)
    checksum = image_checksum(img.depth, img.segmentation)
    dev = world.device
    with torch.cuda.device(dev):
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(frames):
            img = render(world, cam)
        e1.record()
        torch.cuda.synchronize(dev)
        wall = e0.elapsed_time(e1) * 1e-3
    fps = frames * num_envs / wall if wall > 0 else float("inf")
    return BenchReport(num_envs=num_envs, total_steps=frames, wall_seconds=wall,
                       steps_per_second=fps, sim_to_real_ratio=0.0, dt=0.0, checksum=checksum,
                       frames_per_second=fps, resolution=(cam.width, cam.height),
                       workers=workers, mode="render", engine="fs_render",
                       machine=machine_descriptor(dev))


__all__ = ["DEFAULT_DT", "WARMUP_STEPS", "BenchReport", "machine_descriptor", "state_checksum",
           "image_checksum", "make_bench_batch", "bench_dynamics", "bench_scene_config",
           "bench_render"]
