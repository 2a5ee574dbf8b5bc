#!/usr/bin/env python
"""Benchmark: fused controller + dynamics vehicle-steps/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
                    [--impl ours|reference]

Metric (BASELINE.json): vehicle-steps/sec (controller + dynamics), one
vehicle-step = one vehicle advanced by one control + integration step
(the reference's steps_per_second, bench.py:59,169).

A bench "step" is one control step of the whole shard: ONE fused kernel
launch that reads every vehicle's state (52 B) and command (16 B) from HBM
and writes the new state (52 B) back -- 120 algorithmic bytes per
vehicle-step.  Default workload = BASELINE config 2
(velocity mode, 2^22 vehicles per GPU, dt = 0.01, 1000 steps); the state +
command working set (285 MB) exceeds the 126 MB L2, so no flush is needed.
Multi-GPU: one process per GPU (torchrun), each owns a contiguous 2^22-vehicle
shard (weak scaling); no per-step collective; the per-rollout episode
statistics are reduced with NCCL once at the end (outside the timed loop).

--impl reference: the reference's CPU algorithm (oracle/flocksim_oracle.py,
a pinned float64 NumPy restatement of flocksim's control_batch + step_batch;
the reference itself is Python and does not travel to the GPU box) on all
host cores, on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "vehicle-steps/sec (controller+dynamics)"
UNIT = "vehicle-steps/s"

# BASELINE.json configs; n is per GPU (weak scaling) except cfg0.
CONFIGS = {
    # cfg0 is one control evaluation over 1024 quads; the K timed steps repeat
    # that evaluation (control only: the state does not change), so the time
    # per step is the launch-bound kernel, not one graph launch's overhead
    "cfg0": dict(mode="position", n=1024, steps=1000, dt=0.01, integrate=False, airframe="quad",
                 bytes=84, desc="Lee position controller, single step (evaluated K times), "
                                 "1024 quads, X-quad rotor thrusts"),
    "cfg1": dict(mode="attitude", n=1 << 20, steps=100, dt=0.01, integrate=True, bytes=120,
                 desc="Lee attitude controller + integration, 2^20 quads, 100 steps"),
    "cfg2": dict(mode="velocity", n=1 << 22, steps=1000, dt=0.01, integrate=True, bytes=120,
                 desc="Lee velocity controller (vehicle frame) closed loop, 2^22 quads per GPU, "
                      "1000 steps"),
    "cfg3": dict(mode="position", n=1 << 21, steps=1000, dt=0.01, integrate=True, bytes=121,
                 reset_prob=0.01, stats=True,
                 desc="Lee position controller closed loop, 2^21 quads per GPU (2^24 on 8), "
                      "1% Bernoulli resets per step, NCCL-reduced episode statistics"),
    "world": dict(mode="velocity", n=1 << 22, steps=500, dt=0.01, integrate=True, bytes=211,
                  world=True,
                  desc="free-space World.step (SURVEY 8(f) rank 1): auto-reset, velocity control, "
                       "integration, box collision, counters, reward, 16-float observations; "
                       "2^22 envs per GPU"),
    "vecenv": dict(mode="velocity", n=1 << 22, steps=500, dt=0.01, integrate=True, bytes=211,
                   world=True, actions=True,
                   desc="flocksim_rl VecEnvHandle.step (SURVEY 8(f) rank 3): (E, 4) fp32 policy "
                        "actions clipped + denormalized inside the World.step kernel; 2^22 envs "
                        "per GPU"),
    "forest": dict(mode="velocity", n=1 << 21, steps=200, dt=0.01, integrate=True, bytes=None,
                   world=True, forest=True,
                   desc="obstacle World.step (SURVEY 8(f) rank 4): forest.yaml layout (10 "
                        "depth-3 trees + 6 walls = 76 primitives per env), velocity control, "
                        "integration, primitive SDF collision (AABB broad phase), reward, "
                        "observations; 2^21 envs per GPU"),
    "render": dict(mode="velocity", n=1 << 10, steps=20, dt=0.01, integrate=True, bytes=None,
                   render=True, metric="depth frames/sec (480x270, forest scene)",
                   unit="frames/s",
                   desc="depth + segmentation camera (SURVEY 8(f) rank 4; PAPER.md:140 setting): "
                        "2^10 robots, 480x270 pixels, forest.yaml scene (76 primitives per "
                        "env), float64 ray-primitive arithmetic"),
    "cfg4": dict(mode="position", n=1 << 23, steps=500, dt=0.005, integrate=True, bytes=160,
                 hetero=True, airframe="quad+hex", rotor_dynamics=True,
                 desc="heterogeneous fleet 2^23: half X-quads, half hexarotors, per-vehicle "
                      "mass/inertia, position control, 500 steps"),
}
DEFAULT_CONFIG = "cfg2"
# BASELINE.md "Published numbers for this path": > 3.8e6 aggregate simulation
# steps/s (controllers + physics, 2^17 robots, 2x RTX 3090).
# Not the same configuration (2^17 robots, PhysX) -- the closest published
# figure; vs_baseline_basis in the line says so.
PUBLISHED_STEPS_PER_S = 3.8e6
HBM_FALLBACK_GBS = 6650.0
SPEC_HBM_GBS = 8000.0          # B200 HBM3e data-sheet bandwidth


# ----------------------------------------------------------------------------
# helpers
# ----------------------------------------------------------------------------

def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


def _profile_traffic(config):
    """dram bytes/launch of the fused kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            s = json.load(f)
        return s.get(config, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nvml is not None:
            self._thread = threading.Thread(target=self._run, daemon=True)
            self._thread.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._thread is not None:
            self._thread.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------
# CPU baseline / reference arm (oracle port on all host cores)
# ----------------------------------------------------------------------------

_W = {}


def _cpu_worker_init(mode, n, seed):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np
    from oracle import flocksim_oracle as O
    from oracle.workload import config_batch
    s, m, att, vel, pos = config_batch(mode, n, seed)
    _W.update(O=O, s=s, m=m, att=att, vel=vel, pos=pos, mode=mode, np=np)


def _cpu_worker_step(nsteps):
    O, w = _W["O"], _W
    t0 = time.perf_counter()
    for _ in range(nsteps):
        if w["mode"] == "position":
            f, mom, _ = O.position_control(w["s"], w["pos"][0:3], w["pos"][3], O.Gains(),
                                           O.Robot(), O.Limits())
            w["s"], _, _ = O.integrate(w["s"], f, mom, O.Robot(), 0.01)
        else:
            w["s"], _ = O.step(w["s"], w["m"], w["att"], w["vel"], O.Gains(), O.Robot(), 0.01)
    return time.perf_counter() - t0


def _forest_layout(n, seed):
    """Host float64 forest scene for the CPU legs: forest.yaml's classes (10
    depth-3 trees from assetgen seeds 0-3, trunks on the ground, random yaw)
    plus walls, compiled with the oracle's compile_rows."""
    import numpy as np

    from oracle import scene_oracle as S
    from paper_2305_16510_b200 import assets
    from paper_2305_16510_b200.world import make_wall_prototype
    kinds = {"box": S.BOX, "cylinder": S.CYL, "sphere": S.SPH}
    protos = [assets.generate_tree(assets.TreeConfig(seed=t))[0] for t in range(4)]
    walls = make_wall_prototype([12.0, 12.0, 6.0], 0.1)
    rng = np.random.default_rng(seed)
    rows = []
    for _ in range(n):
        row = []
        for _ in range(10):
            pr = protos[rng.integers(0, 4)]
            ip = np.array([rng.uniform(0.05, 0.95) * 12.0, rng.uniform(0.05, 0.95) * 12.0, 0.0])
            iq = S.rot_zyx(0.0, 0.0, rng.uniform(-3.14159, 3.14159))
            row += [(kinds[p.kind], p.dims, p.position, p.rotation, ip, iq, 2, True)
                    for p in pr.primitives]
        row += [(S.BOX, p.dims, p.position, p.rotation, np.zeros(3), np.array([1.0, 0, 0, 0]),
                 1, True) for p in walls.primitives]
        rows.append(row)
    return S.compile_rows(rows)


def _forest_worker_init(n, seed):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np

    from oracle import flocksim_oracle as O
    from oracle import scene_oracle as S
    from oracle import world_oracle as WO
    ps = _forest_layout(n, seed)
    rng = np.random.default_rng(seed + 1)
    s = np.zeros((13, n))
    s[0:3] = rng.uniform([1.8, 1.8, 1.5], [10.2, 10.2, 3.6], (n, 3)).T
    s[3] = 1.0
    vel = np.concatenate([rng.normal(size=(3, n)), rng.uniform(-1, 1, (1, n))])
    env = WO.EnvCfg(bounds=np.array([12.0, 12.0, 6.0]), episode_max_steps=10 ** 9)
    _W.update(kind="forest", O=O, S=S, WO=WO, ps=ps, s=s, goals=s[0:3].copy(), vel=vel, env=env,
              n=n, np=np)


def _render_worker_init(n, seed):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np

    from oracle import scene_oracle as S
    ps = _forest_layout(n, seed)
    rng = np.random.default_rng(seed + 1)
    p = rng.uniform([1.8, 1.8, 1.5], [10.2, 10.2, 3.6], (n, 3))
    q = S.rot_zyx(0.0, 0.0, rng.uniform(-3.1, 3.1, n))
    mq = S.rot_zyx(-np.pi / 2, 0.0, -np.pi / 2)
    _W.update(kind="render", S=S, ps=ps, p=p, q=q, mp=np.tile([0.1, 0.0, 0.0], (n, 1)),
              mq=np.tile(mq, (n, 1)), n=n)


def _scene_worker_step(nsteps):
    w = _W
    t0 = time.perf_counter()
    for _ in range(nsteps):
        if w["kind"] == "render":
            w["S"].render(w["p"], w["q"], w["mp"], w["mq"], w["ps"], 480, 270, 1.57, 10.0)
        else:
            np, S, WO, O = w["np"], w["S"], w["WO"], w["O"]
            n = w["n"]
            out = WO.world_step(w["s"], w["goals"], np.zeros(n, bool), np.zeros(n, np.int64),
                                np.ones(n, np.uint8), np.zeros((4, n)), w["vel"], O.Robot(),
                                O.Gains(), O.Limits(), w["env"], WO.RewardCfg(), None,
                                hit_fn=lambda pts: S.min_distance(w["ps"], pts) < 0.2)
            w["s"] = out["state"]
    return time.perf_counter() - t0


_THREAD_VARS = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")


def _spawn_pool(cores, init, initargs):
    """Fresh (spawned) single-threaded worker processes: a forked child of a
    process that already initialized torch / a threaded BLAS would inherit
    its thread pools and oversubscribe the cores."""
    import multiprocessing as mp
    saved = {k: os.environ.get(k) for k in _THREAD_VARS}
    for k in _THREAD_VARS:
        os.environ[k] = "1"
    try:
        return mp.get_context("spawn").Pool(cores, initializer=init, initargs=initargs)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


class CpuScene:
    """Process-sharded oracle for the scene workloads (forest World.step or
    the depth camera): one process per core, `per_core` envs each."""

    def __init__(self, kind, per_core, cores=None, seed=0):
        self.cores = cores or os.cpu_count() or 1
        self.per_core = per_core
        init = _render_worker_init if kind == "render" else _forest_worker_init
        self.pool = _spawn_pool(self.cores, init, (per_core, seed))
        self.pool.map(_scene_worker_step, [1] * self.cores)

    @property
    def n(self):
        return self.cores * self.per_core

    def step(self, nsteps=1):
        t0 = time.perf_counter()
        self.pool.map(_scene_worker_step, [nsteps] * self.cores, chunksize=1)
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def scene_cpu_run(kind, steps, warmup):
    per_core = 1 if kind == "render" else 2048
    fleet = CpuScene(kind, per_core)
    try:
        for _ in range(warmup):
            fleet.step(1)
        wall = sum(fleet.step(1) for _ in range(steps))
    finally:
        fleet.close()
    what = ("480x270 depth+segmentation frames of forest envs (76 primitives), float64 NumPy "
            "restatement of flocksim camera.render (pinned to the reference)" if kind == "render"
            else "forest World.step envs (76 primitives), float64 NumPy restatement of flocksim "
                 "World.step + check_collisions (pinned to the reference)")
    unit = "frames/s" if kind == "render" else "env-steps/s"
    return {"value": fleet.n * steps / wall, "unit": unit, "cores": fleet.cores, "kind": "port",
            "sample": f"{fleet.n} {what}, {per_core}/core x {steps} steps after {warmup} "
                      "warm-up, process-sharded", "wall_s": wall}


class CpuFleet:
    """Process-sharded float64 oracle (one process per core, contiguous
    shards as dynamics.py:267-283 partitions threads)."""

    def __init__(self, mode, per_core, cores=None, seed=0):
        self.cores = cores or os.cpu_count() or 1
        self.per_core = per_core
        self.pool = _spawn_pool(self.cores, _cpu_worker_init, (mode, per_core, seed))
        self.pool.map(_cpu_worker_step, [1] * self.cores)     # warm-up, touch data

    @property
    def n(self):
        return self.cores * self.per_core

    def step(self, nsteps=1):
        t0 = time.perf_counter()
        self.pool.map(_cpu_worker_step, [nsteps] * self.cores, chunksize=1)
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def cpu_baseline(mode, steps=5, per_core=1 << 14, warmup=2):
    """The reference algorithm (pinned float64 oracle port) on all host cores,
    the same process-sharded machinery as --impl reference: a bounded sample
    (per_core vehicles per core), warmed up, then `steps` timed steps."""
    fleet = CpuFleet(mode, per_core)
    try:
        for _ in range(warmup):
            fleet.step(1)
        wall = sum(fleet.step(1) for _ in range(steps))
    finally:
        fleet.close()
    return {"value": fleet.n * steps / wall, "unit": UNIT, "cores": fleet.cores, "kind": "port",
            "sample": f"{fleet.n} vehicles ({per_core}/core) x {steps} steps after {warmup} "
                      f"warm-up, {mode} mode, float64 NumPy restatement of flocksim "
                      "control_batch+step_batch (pinned to the reference), process-sharded"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if cfg.get("forest") or cfg.get("render"):
        kind = "render" if cfg.get("render") else "forest"
        cb = scene_cpu_run(kind, args.steps, args.warmup)
        line = {
            "impl": "reference", "metric": cfg.get("metric", "env-steps/sec (World.step)"),
            "value": cb["value"], "unit": cb["unit"], "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * cb["wall_s"] / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, "desc": cfg["desc"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line))
        return 0
    mode = "velocity" if cfg["mode"] == "mixed" else cfg["mode"]
    per_core = 1 << 14
    fleet = CpuFleet(mode, per_core)
    try:
        for _ in range(args.warmup):
            fleet.step(1)
        t = 0.0
        for _ in range(args.steps):
            t += fleet.step(1)
    finally:
        fleet.close()
    value = fleet.n * args.steps / t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "sample_vehicles": fleet.n},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": fleet.cores, "kind": "port",
                         "sample": f"{fleet.n} vehicles ({per_core}/core) per step, {mode} "
                                   "mode, float64 NumPy restatement of flocksim "
                                   "control_batch+step_batch (pinned bitwise to the reference's "
                                   "golden vectors), process-sharded over all host cores"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------

class WorldRunner:
    """Bench adapter: a device World stepped with fixed velocity commands, or
    (actions=True) with fixed (E, 4) fp32 policy actions through the fused
    action path (fs_vecenv_step)."""

    def __init__(self, n, first_id, seed, device, episode_max_steps=1000, actions=False,
                 forest=False, camera=False):
        import ctypes as C

        import torch

        from paper_2305_16510_b200 import world as W
        from paper_2305_16510_b200.control import CommandBatch, VelocityCommands
        self.C, self.torch = C, torch
        if forest:
            cfg, pools = forest_sim_config(n, seed, camera, episode_max_steps)
        else:
            cfg, pools = W.SimConfig(env=W.EnvConfig(num_envs=n, seed=seed,
                                                     episode_max_steps=episode_max_steps)), None
        self.world = W.World(cfg, pools=pools, device=device, first_env=first_id)
        g = torch.Generator(device="cpu").manual_seed(seed)
        v = torch.randn(n, 3, generator=g)
        yr = torch.rand(n, generator=g) * 2 - 1
        self.cmds = CommandBatch.all_velocity(VelocityCommands(v=v.to(device), yaw_rate=yr.to(device),
                                                               validate=False))
        self.actions = None
        if actions:
            self.actions = (torch.rand(n, 4, generator=g) * 2.4 - 1.2).to(device)
        self.n, self.device, self.stats_slots = n, device, None

    def step(self, stream=None):
        if self.actions is not None:
            self.world.step_actions_async(self.actions, stream)
        else:
            self.world.step_async(self.cmds, stream)

    control = step

    def capture(self, steps, integrate=True, chained=False, persistent=False):
        """(World.step is one launch per step: `chained` / `persistent` are ignored)"""
        torch = self.torch
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                h = self.C.c_void_p(s.cuda_stream)
                for _ in range(steps):
                    self.step(h)
        torch.cuda.current_stream(self.device).wait_stream(s)
        return g


def forest_sim_config(n, seed, camera=False, episode_max_steps=1000):
    """pkg/configs/forest.yaml's world (12 x 12 x 6 m walled envs, 10 trees per
    env from assetgen tree seeds 0-3 at default depth 3, a 480x270 forward
    camera) with n envs; returns (SimConfig, pools)."""
    from paper_2305_16510_b200 import assets
    from paper_2305_16510_b200 import world as W
    from paper_2305_16510_b200.camera import CameraConfig
    env = W.EnvConfig(num_envs=n, seed=seed, bounds=[12.0, 12.0, 6.0],
                      episode_max_steps=episode_max_steps, control_mode="velocity",
                      wall_enabled=True, wall_segmentation_id=1,
                      goal_min=[0.15, 0.15, 0.25], goal_max=[0.85, 0.85, 0.6],
                      spawn_min=[0.15, 0.15, 0.25], spawn_max=[0.85, 0.85, 0.6])
    trees = assets.AssetClassConfig(name="trees", count_per_env=10,
                                    position_min=[0.05, 0.05, 0.0],
                                    position_max=[0.95, 0.95, 0.0], frozen=(None, None, 0.0),
                                    euler_min=[0.0, 0.0, -3.14159],
                                    euler_max=[0.0, 0.0, 3.14159], segmentation_id=2)
    cam = CameraConfig(width=480, height=270, hfov=1.57, max_range=10.0,
                       mount_position=[0.1, 0.0, 0.0], randomize_position=[0.01] * 3,
                       randomize_euler=[0.02] * 3) if camera else None
    pools = {"trees": [assets.generate_tree(assets.TreeConfig(seed=t))[0] for t in range(4)]}
    return W.SimConfig(env=env, asset_classes=[trees], camera=cam), pools


class RenderRunner(WorldRunner):
    """Bench adapter for the depth camera: a forest World with its camera;
    one bench step = camera.render of every env into preallocated images
    (one fs_render launch)."""

    def __init__(self, n, first_id, seed, device):
        super().__init__(n, first_id, seed, device, forest=True, camera=True)
        from paper_2305_16510_b200.camera import render
        self.render = render
        self.cam = self.world.camera
        self.out = render(self.world, self.cam)

    def step(self, stream=None):
        self.render(self.world, self.cam, out=self.out)

    control = step


def make_fleet(cfg, n, first_id, seed, device):
    if cfg.get("render"):
        return RenderRunner(n, first_id, seed, device)
    if cfg.get("world"):
        return WorldRunner(n, first_id, seed, device, actions=cfg.get("actions", False),
                           forest=cfg.get("forest", False))
    from paper_2305_16510_b200.allocation import HEXAROTOR, QUAD_X
    from paper_2305_16510_b200.fleet import Fleet
    airframes, split = None, 0
    if cfg.get("airframe") == "quad":
        airframes = (QUAD_X, QUAD_X)
    elif cfg.get("airframe") == "quad+hex":
        airframes, split = (QUAD_X, HEXAROTOR), cfg["global_n"] // 2
    return Fleet(n, mode=cfg["mode"], dt=cfg["dt"], seed=seed, first_id=first_id,
                 airframes=airframes, airframe_split=split,
                 rotor_dynamics=cfg.get("rotor_dynamics", False), hetero=cfg.get("hetero", False),
                 reset_prob=cfg.get("reset_prob", 0.0), want_stats=cfg.get("stats", False),
                 device=device)


def measure_render_e2e(runner, device, steps, chunks=8):
    """camera.render as a NumPy-side caller uses it: robot states copied in
    from pinned host memory, every env rendered, depth + segmentation copied
    back to pinned host memory (the reference returns host arrays).  The envs
    are cut into `chunks` ranges on their own streams, so the read-back of
    one range overlaps the rendering of the next."""
    import torch
    world, out, cam = runner.world, runner.out, runner.cam
    n = world.num_envs
    host_state = torch.empty(world._state.shape, dtype=torch.float32, pin_memory=True)
    host_state.copy_(world._state)
    host_depth = torch.empty(out.depth.shape, dtype=torch.float32, pin_memory=True)
    host_seg = torch.empty(out.segmentation.shape, dtype=torch.int32, pin_memory=True)
    streams = [torch.cuda.Stream(device) for _ in range(chunks)]
    bounds = [(n * k) // chunks for k in range(chunks + 1)]
    main = torch.cuda.current_stream(device)

    def one():
        world._state.copy_(host_state, non_blocking=True)
        for k, s in enumerate(streams):
            s.wait_stream(main)
            a, b = bounds[k], bounds[k + 1]
            with torch.cuda.stream(s):
                runner.render(world, cam, out=out, envs=(a, b - a))
                host_depth[a:b].copy_(out.depth[a:b], non_blocking=True)
                host_seg[a:b].copy_(out.segmentation[a:b], non_blocking=True)
        for s in streams:
            main.wait_stream(s)

    one()
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize(device)
    wall = time.perf_counter() - t0
    return {"value": n * steps / wall, "unit": "frames/s",
            "h2d_bytes_per_step": int(host_state.numel() * 4),
            "d2h_bytes_per_step": int(host_depth.numel() * 4 + host_seg.numel() * 4),
            "steps": steps,
            "path": f"state planes H2D from pinned host, camera.render (fs_render) of {chunks} "
                    f"env ranges on {chunks} streams, each range's depth + segmentation D2H to "
                    "pinned host as soon as it is rendered"}


def measure_e2e(cfg, n, device, steps, chunks=8, nstreams=8):
    """Drop-in usage through the C ABI with HOST buffers (fs_step_host): every
    step copies the state + commands from pinned host memory, runs the fused
    step and copies the new state back -- the reference-facing call on
    NumPy-resident data.  Chunks of the batch are pipelined over `nstreams`
    streams (one cudaMemcpy2DAsync per array per chunk) so H2D, compute and
    D2H overlap.  8 chunks on 8 streams: a few large 2-D copies keep PCIe
    near its full-duplex rate (tools/e2e_sweep.py: 32 x 4 reached 5.9e8,
    8 x 8 7.1e8 vehicle-steps/s; the H2D-bound ceiling is ~7.25e8)."""
    import ctypes as C

    import torch

    from paper_2305_16510_b200 import _native as N
    from paper_2305_16510_b200._tensors import alloc_planes, stride0
    from paper_2305_16510_b200.control import ControlGains, ControlLimits
    from paper_2305_16510_b200.dynamics import RobotParams

    if cfg["mode"] == "mixed" or cfg.get("hetero") or cfg.get("airframe") or \
            cfg.get("reset_prob") or cfg.get("stats") or cfg.get("world") or cfg.get("render"):
        return None
    lib = N.load()
    f = make_fleet(dict(cfg, global_n=n), n, 0, 1234, device)
    host_state = torch.empty(f.state.shape, dtype=torch.float32, pin_memory=True)
    host_cmd = torch.empty(f.cmd.shape, dtype=torch.float32, pin_memory=True)
    host_state.copy_(f.state)
    host_cmd.copy_(f.cmd)
    dev_state = alloc_planes(13, n, device)
    dev_cmd = alloc_planes(4, n, device)
    robot, gains, limits = RobotParams().native(), ControlGains().native(), ControlLimits().native()
    streams = [torch.cuda.Stream(device) for _ in range(nstreams)]
    handles = (C.c_void_p * nstreams)(*[s.cuda_stream for s in streams])
    d = N.fs_step_desc()
    d.n = n
    d.state_in = d.state_out = C.c_void_p(host_state.data_ptr())
    d.state_in_stride = d.state_out_stride = stride0(host_state)
    d.mode = f.mode
    d.integrate = 1 if cfg["integrate"] else 0
    d.cmd = C.c_void_p(host_cmd.data_ptr())
    d.cmd_stride = stride0(host_cmd)
    d.dt = cfg["dt"]

    def one_step():
        N.check(lib.fs_step_host(C.byref(d), robot, gains, limits, None,
                                 C.c_void_p(dev_state.data_ptr()), C.c_void_p(dev_cmd.data_ptr()),
                                 stride0(dev_state), chunks, handles, nstreams), "fs_step_host")

    for _ in range(2):
        one_step()
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    torch.cuda.synchronize(device)
    wall = time.perf_counter() - t0
    return {"value": n * steps / wall, "unit": UNIT,
            "h2d_bytes_per_step": int(n * 17 * 4), "d2h_bytes_per_step": int(n * 13 * 4),
            "steps": steps,
            "path": f"fs_step_host C ABI on pinned host state+commands, {chunks} chunks x "
                    f"{nstreams} streams (cudaMemcpy2DAsync per array per chunk)"}


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2305_16510_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}))
        return 1
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=device)
    N.load()
    for key, val in ((N.FS_TUNE_PREC, args.prec), (N.FS_TUNE_NCW, args.ncw),
                     (N.FS_TUNE_KERNEL, args.kernel), (N.FS_TUNE_VPT, args.vpt),
                     (N.FS_TUNE_CHAIN_RELEASE, args.chain_release),
                     (N.FS_TUNE_L2_KEEP_MB, args.l2_keep_mb)):
        if val is not None:
            N.set_tuning(key, val)

    n = args.n or cfg["n"]
    global_n = n * world
    cfg = dict(cfg, global_n=global_n)
    fleet = make_fleet(cfg, n, rank * n, args.seed, device)
    K, W = args.steps, args.warmup
    if not cfg["integrate"]:
        step_fn = fleet.control
    else:
        step_fn = fleet.step
    for _ in range(W):
        step_fn()
    torch.cuda.synchronize(device)
    if cfg.get("stats"):
        fleet.stats_slots.zero_()

    # re-spawns are drawn inside the step kernel (cfg3); an obstacle World.step
    # is the warp-cooperative auto-reset kernel + the step kernel
    launches_per_step = 2 if cfg.get("forest") else 1
    fleet_cfg = not (cfg.get("world") or cfg.get("render"))
    persistent = (args.launch == "persistent" and fleet_cfg and cfg["integrate"] and not args.eager
                  and getattr(fleet, "chainable", False))
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    graph = None
    if not args.eager:
        # the K launches are captured once and replayed as one CUDA graph: no
        # host launch gaps inside the timed region
        graph = fleet.capture(K, integrate=cfg["integrate"], chained=args.launch == "chained",
                              persistent=persistent)
        if cfg.get("stats"):
            fleet.stats_slots.zero_()
        torch.cuda.synchronize(device)
    else:
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(device)
    with ClockSampler(local) as clk:
        t_start.record()
        if graph is not None:
            graph.replay()
        else:
            for k in range(K):
                starts[k].record()
                step_fn()
                ends[k].record()
        t_end.record()
        torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    if graph is not None:
        kern_ms = [elapsed_ms / K]       # per-step device time (kernels back to back)
    else:
        kern_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())

    stats = None
    if cfg.get("stats"):
        from paper_2305_16510_b200.fleet import summarize_stats
        tot = fleet.stats_local()
        if world > 1:
            dist.all_reduce(tot)          # int64 sums: identical for any GPU count
        stats = summarize_stats(tot.cpu())

    # the same K steps as K separate fs_step launches (one CUDA graph), next
    # to the persistent launch's number
    per_step = None
    if persistent:
        g2 = fleet.capture(K, integrate=True, chained=False, persistent=False)
        torch.cuda.synchronize(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g2.replay()
        e1.record()
        torch.cuda.synchronize(device)
        pms = e0.elapsed_time(e1)
        per_step = {"value": global_n * K / (pms * 1e-3), "unit": UNIT, "ms_per_step": pms / K,
                    "note": "K fs_step launches (one per step) replayed as one CUDA graph"}
        del g2

    # K-step rollout with the vehicles held in registers (fs_rollout)
    fused = None
    if cfg["integrate"] and not args.no_fused and not cfg.get("world") and not cfg.get("render"):
        fleet.reset_fleet()
        fleet.rollout(1, fused=True)
        torch.cuda.synchronize(device)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fleet.rollout(K, fused=True)
        e1.record()
        torch.cuda.synchronize(device)
        fms = e0.elapsed_time(e1)
        fused = {"value": global_n * K / (fms * 1e-3), "unit": UNIT, "ms_total": fms,
                 "note": "one fs_rollout launch, state in registers for all K steps "
                         "(commands held constant, as in the config); compute-bound, not the "
                         "headline"}

    e2e = None
    if not args.no_e2e:
        e2e = measure_e2e(cfg, n, device, max(3, min(K, args.e2e_steps)))
        if e2e is not None and world > 1:
            et = torch.tensor([e2e["value"]], dtype=torch.float64, device=device)
            dist.all_reduce(et)
            e2e["value"] = float(et.item())

    bytes_per = cfg["bytes"]
    if cfg.get("forest"):
        # World.step's 211 B + the instance broad phase (one 32-B record per
        # obstacle instance); the narrow phase of instances within reach (slot
        # records, 32-96 B each) is data dependent and comes on top
        bytes_per = 211 + 32 * fleet.world.instances_per_env
    elif cfg.get("render"):
        cam = fleet.cam
        bytes_per = cam.width * cam.height * 8     # depth f32 + segmentation i32 written
    avg_kernel_s = statistics.mean(kern_ms) * 1e-3
    peak, peak_kind = _peaks()
    achieved = bytes_per * n / avg_kernel_s / 1e9
    value = global_n * K / (elapsed_ms * 1e-3)

    if cfg.get("render") and not args.no_e2e:
        e2e = measure_render_e2e(fleet, device, max(3, min(K, args.e2e_steps)))
        if e2e is not None and world > 1:
            et = torch.tensor([e2e["value"]], dtype=torch.float64, device=device)
            dist.all_reduce(et)
            e2e["value"] = float(et.item())

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        if cfg.get("forest") or cfg.get("render"):
            cpu = scene_cpu_run("render" if cfg.get("render") else "forest", 2, 1)
            cpu.pop("wall_s")
        else:
            cpu = cpu_baseline("velocity" if cfg["mode"] == "mixed" else cfg["mode"])

    if rank == 0:
        unit = cfg.get("unit", "env-steps/s" if cfg.get("world") else UNIT)
        line = {
            "metric": cfg.get("metric", "env-steps/sec (World.step)" if cfg.get("world")
                              else METRIC),
            "value": value, "unit": unit, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": elapsed_ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": (value / PUBLISHED_STEPS_PER_S if fleet_cfg
                                               else None),
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "vehicles_per_gpu": n,
                       "vehicles_total": global_n, "mode": cfg["mode"], "dt": cfg["dt"],
                       "l2": ("per-step traffic larger than L2 (> 126 MB per GPU)"
                              if n * bytes_per > 126e6 else "working set fits L2 (L2-assisted)"),
                       "launch": (("one fs_render launch per step (every env's image)"
                                   if cfg.get("render") else
                                   "auto-reset kernel + World.step kernel per step"
                                   if cfg.get("forest") else
                                   "one World.step kernel per step" if cfg.get("world") else
                                   ("one persistent fs_step_many launch streams all K steps: "
                                    "every step reads state + commands from HBM and writes the "
                                    "state back, the tile pipeline runs on across steps"
                                    if persistent else
                                    "one fused fs_step kernel per control step, in place")
                                   + (" (Bernoulli re-spawns drawn in-kernel)"
                                      if cfg.get("reset_prob") else ""))
                                  + ("; captured as one CUDA graph" if not args.eager
                                     else "; eager launches"))},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_kind,
                         "spec_peak": SPEC_HBM_GBS, "spec_frac": achieved / SPEC_HBM_GBS,
                         "traffic": _profile_traffic(args.config),
                         ("bytes_per_frame" if cfg.get("render") else "bytes_per_vehicle_step"):
                             bytes_per,
                         "kernel_ms_avg": avg_kernel_s * 1e3},
            "clocks": clk.summary(),
            "gpu_launches": 1 if persistent else K * launches_per_step,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "rollout_fused": fused,
        }
        if per_step is not None:
            line["per_step_launches"] = per_step
        if fleet_cfg:
            line["vs_baseline_basis"] = ("value / 3.8e6: BASELINE.md's published aggregate "
                                         "steps/s (Aerial Gym paper, PAPER.md:140: 2^17 robots, "
                                         "controllers + PhysX, 2x RTX 3090); a different "
                                         "configuration, the closest published figure")
        if stats is not None:
            line["episode_stats"] = stats
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override vehicles per GPU")
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fused", action="store_true")
    ap.add_argument("--eager", action="store_true",
                    help="launch the K steps eagerly (per-launch events) instead of a CUDA graph")
    ap.add_argument("--prec", type=int, default=None,
                    help="controller precision: 0 fp32, 1 fp64 front end, 2 fp64 controller")
    ap.add_argument("--ncw", type=int, default=None, help="stream kernel consumer warps (8/16)")
    ap.add_argument("--kernel", type=int, default=None, help="0 auto, 1 simple, 2 stream")
    ap.add_argument("--vpt", type=int, default=None, help="stream vehicles per thread (1/2)")
    ap.add_argument("--launch", default="persistent", choices=["persistent", "chained", "steps"],
                    help="how the K timed steps are launched (all inside one CUDA graph): one "
                         "persistent fs_step_many launch, K chained fs_step launches "
                         "(programmatic dependents), or K plain fs_step launches")
    ap.add_argument("--l2-keep-mb", type=int, default=None,
                    help="MiB of tiles the streaming kernel keeps L2-resident across steps")
    ap.add_argument("--chain-release", type=int, default=None,
                    help="chained steps: 1 = gpu-scope fence before publishing a tile")
    args = ap.parse_args(argv)
    cfg = CONFIGS[args.config]
    if args.steps is None:
        args.steps = cfg["steps"] if args.impl == "ours" else 10
    args.warmup = max(3, args.warmup) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
