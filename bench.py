#!/usr/bin/env python
"""Benchmark: fused controller + dynamics vehicle-steps/s on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
                    [--impl ours|reference]

Metric (BASELINE.json): vehicle-steps/sec (controller + dynamics), one
vehicle-step = one vehicle advanced by one control + integration step
(the reference's steps_per_second, bench.py:59,169).

A bench "step" is one control step of the whole fleet: every vehicle's state
(52 B) and command (16 B) read from HBM and the new state (52 B) written
back -- 120 algorithmic bytes per vehicle-step.  Default
workload = BASELINE config 2 (velocity mode, 2^22 vehicles IN TOTAL, dt =
0.01, 1000 steps).

Multi-GPU: `--gpus N` runs one process per GPU.  Launched without a torchrun
environment, bench.py re-executes itself under torch.distributed.run with N
ranks (127.0.0.1 rendezvous); under the driver's torchrun it uses the ranks
it is given and checks WORLD_SIZE == N.  The fleet configs are sharded the
way BASELINE.json states them: the configured total (2^22 for config 2) is
cut into the reference's contiguous blocks [(n k)//N, (n (k+1))//N)
(dynamics.py:267-283), one per GPU ("scaling": "strong").  Vehicles are
independent, so no collective runs per step; the episode statistics are
reduced with one NCCL all-reduce of three int64 per rollout.  The line's
`north_star` object measures BASELINE.json's north-star target on the same
GPUs: config 3 (position control, 1 % Bernoulli re-spawns, statistics) at
2^24 vehicles in total, 2^24/N per GPU.

--impl reference: the UNMODIFIED reference (flocksim, built into
oracle/_ref by oracle/build_ref.py) on all host cores: control_batch +
step_batch process-sharded over the cores, plus its own bench_dynamics at
workers=1 and workers=cores, on a bounded sample of the same workload.  The
position-mode configs (0, 3, 4) have no reference code: their CPU leg is the
builder's float64 extension oracle (kind "port").
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

# BASELINE.json configs.  `n_total`: the fleet is that many
# vehicles in total, sharded over the GPUs (strong scaling, as BASELINE.json
# states configs 2 and 3); the World / camera workloads keep `n`
# per GPU (weak scaling).
CONFIGS = {
    # cfg0 is one control evaluation over 1024 quads; the K timed steps repeat
    # that evaluation (control only: the state does not change), so the time
    # per step is the launch-bound kernel, not one graph launch's overhead
    "cfg0": dict(mode="position", n=1024, n_total=1024, steps=1000, dt=0.01, integrate=False,
                 airframe="quad",
                 bytes=84, desc="Lee position controller, single step (evaluated K times), "
                                 "1024 quads, X-quad rotor thrusts"),
    "cfg1": dict(mode="attitude", n=1 << 20, n_total=1 << 20, steps=100, dt=0.01, integrate=True,
                 bytes=120,
                 desc="Lee attitude controller + integration, 2^20 quads in total, 100 steps"),
    "cfg2": dict(mode="velocity", n=1 << 22, n_total=1 << 22, steps=1000, dt=0.01, integrate=True,
                 bytes=120,
                 desc="Lee velocity controller (vehicle frame) closed loop, 2^22 quads in total "
                      "sharded evenly over the GPUs, 1000 steps"),
    "cfg3": dict(mode="position", n=1 << 24, n_total=1 << 24, steps=1000, dt=0.01, integrate=True,
                 bytes=121, reset_prob=0.01, stats=True,
                 desc="Lee position controller closed loop, 2^24 quads in total (2^21 per GPU on "
                      "8), 1% Bernoulli resets per step, NCCL-reduced episode statistics"),
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
    "cfg4": dict(mode="position", n=1 << 23, n_total=1 << 23, steps=500, dt=0.005, integrate=True,
                 bytes=160, out_bytes=24,
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


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region
    (every millisecond)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period_s: float = 0.001):
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
    """Port worker: the builder's float64 oracle (position-mode configs have
    no reference code)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import numpy as np
    from oracle import flocksim_oracle as O
    from oracle.workload import config_batch
    s, m, att, vel, pos = config_batch(mode, n, seed)
    _W.update(kind="port", O=O, s=s, m=m, att=att, vel=vel, pos=pos, mode=mode, np=np)


def _ref_worker_init(mode, n, seed):
    """Reference worker: the UNMODIFIED flocksim (oracle/_ref wheels) on a
    shard of BASELINE-distributed vehicles (oracle/workload.config_batch),
    stepped with its public control_batch + step_batch (the body of
    bench._pipeline_step, bench.py:146-149)."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import ref
    from oracle.workload import config_batch
    fc, fd = ref.flocksim("control"), ref.flocksim("dynamics")
    s, _, att, vel, _ = config_batch(mode, n, seed)
    states = fd.RigidStateBatch(p=s[0:3].T.copy(), q=s[3:7].T.copy(), v=s[7:10].T.copy(),
                                omega=s[10:13].T.copy())
    if mode == "attitude":
        cmds = fc.CommandBatch.all_attitude(fc.AttitudeCommands(
            roll=att[0], pitch=att[1], yaw_rate=att[2], thrust=att[3]))
    else:
        cmds = fc.CommandBatch.all_velocity(fc.VelocityCommands(v=vel[0:3].T.copy(),
                                                                yaw_rate=vel[3]))
    _W.update(kind="reference", fc=fc, fd=fd, states=states, cmds=cmds,
              params=fd.RobotParams(), gains=fc.ControlGains(), limits=fc.ControlLimits())


def _cpu_worker_step(nsteps):
    w = _W
    t0 = time.perf_counter()
    if w["kind"] == "reference":
        fc, fd = w["fc"], w["fd"]
        for _ in range(nsteps):
            wrench, _ = fc.control_batch(w["states"], w["cmds"], w["gains"], w["params"],
                                         w["limits"])
            w["states"], _ = fd.step_batch(w["states"], w["params"], wrench, 0.01)
        return time.perf_counter() - t0
    O = w["O"]
    for _ in range(nsteps):
        if w["mode"] == "position":
            f, mom, _ = O.position_control(w["s"], w["pos"][0:3], w["pos"][3], O.Gains(),
                                           O.Robot(), O.Limits())
            w["s"], _, _ = O.integrate(w["s"], f, mom, O.Robot(), 0.01)
        else:
            w["s"], _ = O.step(w["s"], w["m"], w["att"], w["vel"], O.Gains(), O.Robot(), 0.01)
    return time.perf_counter() - t0


def _ref_bench_dynamics(num_envs, steps, mode, workers):
    """The reference's own harness, unmodified (flocksim.bench.bench_dynamics,
    bench.py:152-173): its near-hover batch, workers threads for step_batch."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import ref
    rep = ref.flocksim("bench").bench_dynamics(num_envs=num_envs, steps=steps, mode=mode,
                                               workers=workers, warmup=1)
    return rep.steps_per_second


def reference_available() -> bool:
    try:
        from oracle import ref
        return ref.available()
    except Exception:
        return False


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
    """Process-sharded CPU leg (one single-threaded process per core,
    contiguous shards as dynamics.py:267-283 partitions threads): the
    reference itself (kind "reference") or the float64 oracle port."""

    def __init__(self, mode, per_core, cores=None, seed=0, kind="reference"):
        self.cores = cores or os.cpu_count() or 1
        self.per_core = per_core
        self.kind = kind
        init = _ref_worker_init if kind == "reference" else _cpu_worker_init
        self.pool = _spawn_pool(self.cores, init, (mode, per_core, seed))
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


def _cpu_kind(mode):
    """'reference' for the modes the reference implements, else 'port'."""
    return "reference" if mode in ("attitude", "velocity") and reference_available() else "port"


def cpu_baseline(mode, steps=10, per_core=1 << 16, warmup=2, with_harness=True):
    """The CPU path on all host cores, process-sharded: the unmodified
    reference's control_batch + step_batch (attitude / velocity), else the
    float64 extension oracle.  A bounded sample: per_core vehicles per core,
    warmed up, then `steps` timed steps.  With the reference, its own
    bench_dynamics harness is also timed at workers=1 and workers=cores."""
    kind = _cpu_kind(mode)
    fleet = CpuFleet(mode, per_core, kind=kind)
    try:
        for _ in range(warmup):
            fleet.step(1)
        wall = sum(fleet.step(1) for _ in range(steps))
    finally:
        fleet.close()
    what = ("the unmodified reference (flocksim from oracle/_ref): control_batch + step_batch"
            if kind == "reference" else
            "the float64 extension oracle (oracle/flocksim_oracle.py; no reference code for this "
            "mode)")
    out = {"value": fleet.n * steps / wall, "unit": UNIT, "cores": fleet.cores, "kind": kind,
           "n": fleet.n,
           "sample": f"{fleet.n} vehicles ({per_core}/core, BASELINE {mode}-mode distributions) "
                     f"x {steps} steps after {warmup} warm-up, {what}, one single-threaded "
                     f"process per core", "wall_s": wall}
    if kind == "reference" and with_harness:
        import multiprocessing as mp
        ne, st = 1 << 16, 3
        res = {}
        for w in (1, fleet.cores):
            with mp.get_context("spawn").Pool(1) as pool:
                res[f"workers_{w}"] = pool.apply(_ref_bench_dynamics, (ne, st, mode, w))
        out["reference_bench_dynamics"] = dict(
            res, unit=UNIT, num_envs=ne, steps=st,
            note="flocksim.bench.bench_dynamics as shipped (its near-hover batch; only "
                 "step_batch is threaded, bench.py:146-149)")
    return out


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
    cb = cpu_baseline(mode, steps=args.steps, warmup=args.warmup)
    value = cb["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * cb["wall_s"] / args.steps, "higher_is_better": True,
        "scaling": "strong" if cfg.get("n_total") else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "sample_vehicles": cb["n"],
                   "note": "a bounded sample of the workload on the host cores (the configured "
                           "fleet takes seconds per step on CPU)"},
        "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if "reference_bench_dynamics" in cb:
        line["reference_bench_dynamics"] = cb["reference_bench_dynamics"]
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


def measure_e2e(cfg, n, device, steps, chunks=8, nstreams=8, first_id=0):
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
    f = make_fleet(dict(cfg, global_n=n), n, first_id, 1234, device)
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
    return {"value": n * steps / wall, "unit": UNIT, "wall_s": wall,
            "h2d_bytes_per_step": int(n * 17 * 4), "d2h_bytes_per_step": int(n * 13 * 4),
            "steps": steps,
            "path": f"fs_step_host C ABI on pinned host state+commands, {chunks} chunks x "
                    f"{nstreams} streams (cudaMemcpy2DAsync per array per chunk)"}


def _traffic(config, n_per_gpu, persistent=True):
    """Per-step DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of
    the dominant kernel at this shard size and launch shape, from a committed
    ncu capture (profiles/traffic.json, tools/traffic_table.py), or None when
    no capture exists."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        e = t.get(f"{config}@{int(n_per_gpu)}" + ("" if persistent else "/steps"))
        return (float(e["dram_bytes_per_step"]), e.get("source")) if e else (None, None)
    except Exception:
        return None, None


def _l2_label(traffic, algorithmic, working_set):
    """Derived from measured DRAM bytes when a capture exists (DRAM < 0.9 x
    the algorithmic bytes = L2-assisted), else stated as unmeasured."""
    if traffic is not None and algorithmic:
        r = traffic / algorithmic
        what = "L2-assisted" if r < 0.9 else "streams from HBM"
        return f"{what}: ncu DRAM bytes = {r:.3f} x the algorithmic bytes per step"
    return (f"no ncu capture at this shard size; working set {working_set / 1e6:.0f} MB per GPU "
            "vs the 126 MB L2 (a size estimate, not a measurement)")


def _shard(cfg, args, world, rank):
    """(n, first_id, global_n, scaling) of this rank."""
    from paper_2305_16510_b200.parallel import shard_bounds
    if cfg.get("n_total"):
        total = args.n or cfg["n_total"]
        lo, hi = shard_bounds(total, world, rank)
        return hi - lo, lo, total, "strong"
    n = args.n or cfg["n"]
    return n, rank * n, n * world, "weak"


def _time_fleet(fleet, cfg, args, K, W, world, device, dist, persistent):
    """Warm up, capture the K steps (one CUDA graph), time the replay with
    CUDA events between barriers; returns (max-over-ranks ms, per-step kernel
    ms list, clock summary)."""
    import torch
    step_fn = fleet.step if cfg["integrate"] else fleet.control
    for _ in range(W):
        step_fn()
    torch.cuda.synchronize(device)
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    graph = None
    if not args.eager:
        graph = fleet.capture(K, integrate=cfg["integrate"], chained=args.launch == "chained",
                              persistent=persistent)
        torch.cuda.synchronize(device)
    else:
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    if getattr(fleet, "stats_slots", None) is not None:
        fleet.stats_slots.zero_()
    if _dist_on(world):
        dist.barrier()
    torch.cuda.synchronize(device)
    with ClockSampler(device.index or 0) as clk:
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
    if _dist_on(world):
        dist.barrier()
    elapsed_ms = t_start.elapsed_time(t_end)
    kern_ms = [elapsed_ms / K] if graph is not None else \
        [a.elapsed_time(b) for a, b in zip(starts, ends)]
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=device)
    if _dist_on(world):
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    del graph
    return float(t.item()), kern_ms, clk.summary()


def _north_star(args, world, rank, local, device, dist, peak):
    """BASELINE.json north star on these GPUs: config 3 semantics (position
    control, 1 % Bernoulli re-spawns, episode statistics) at 2^24 vehicles in
    total, 2^24 / N per GPU, K steps in one persistent launch per GPU, the
    statistics all-reduced over NCCL (int64, identical for any N)."""
    import torch
    from paper_2305_16510_b200.fleet import summarize_stats
    cfg = dict(CONFIGS["cfg3"])
    K = args.north_star_steps
    from paper_2305_16510_b200.parallel import shard_bounds
    lo, hi = shard_bounds(cfg["n_total"], world, rank)
    n = hi - lo
    fleet = make_fleet(dict(cfg, global_n=cfg["n_total"]), n, lo, args.seed, device)
    persistent = args.launch == "persistent" and fleet.chainable and not args.eager
    ms, kern, clocks = _time_fleet(fleet, cfg, args, K, 3, world, device, dist, persistent)
    tot = fleet.stats_local()
    if _dist_on(world):
        dist.all_reduce(tot)          # the one collective: three int64 sums
    stats = summarize_stats(tot.cpu())
    alt = None
    if persistent:                    # the faster launch shape at this shard size
        ams, akern, aclocks = _time_fleet(fleet, cfg, args, K, 3, world, device, dist, False)
        alt = {"persistent_ms_per_step": ms / K, "per_step_launches_ms_per_step": ams / K}
        if ams < ms:
            ms, kern, clocks, persistent = ams, akern, aclocks, False
    value = cfg["n_total"] * K / (ms * 1e-3)
    per_gpu_gbs = cfg["bytes"] * n / (statistics.mean(kern) * 1e-3) / 1e9
    f = torch.tensor([per_gpu_gbs], dtype=torch.float64, device=device)
    if _dist_on(world):
        dist.all_reduce(f, op=dist.ReduceOp.MIN)
    traffic, src = _traffic("cfg3", n, persistent)
    del fleet
    torch.cuda.empty_cache()
    return {"metric": METRIC, "value": value, "unit": UNIT, "target": 1e11,
            "meets_target": value >= 1e11, "vehicles_total": cfg["n_total"],
            "vehicles_per_gpu": n, "n_gpus": world, "steps": K, "ms_per_step": ms / K,
            "hbm_frac_per_gpu_min": float(f.item()) / peak, "hbm_frac_target": 0.70,
            "bytes_per_vehicle_step": cfg["bytes"], "traffic_per_step": traffic,
            "traffic_source": src,
            "l2": _l2_label(traffic, cfg["bytes"] * n, n * 68),
            "episode_stats": dict(stats, reduced_over_ranks=world,
                                  collective="NCCL all_reduce(SUM) of 3 int64"
                                  if _dist_on(world) else "none (1 rank)"),
            "launch": ("one persistent fs_step_many launch per GPU" if persistent else
                       "K fs_step launches per GPU") +
                      " (in-kernel re-spawns and statistics), captured as a CUDA graph",
            "launch_shapes": alt,
            "roofline_issue": _issue_roofline("cfg3", n * K / (ms * 1e-3)),
            "clocks": clocks,
            "desc": "BASELINE north star: config 3 (Lee position control, 1% Bernoulli re-spawns "
                    "per step, per-rollout mean position error and crash count reduced over the "
                    "GPUs) at 2^24 vehicles in total"}


def measure_e2e_numpy(cfg, n, device, steps, first_id=0):
    """The reference-facing drop-in on the reference's own data types: float64
    NumPy state / command dataclasses (duck-typed SimpleNamespace records
    with flocksim's field names) in, new ones out, through
    paper_2305_16510_b200.compat.pipeline_step -- what a flocksim caller
    swapped onto the B200 path sees, including the float64 <-> fp32 packing
    on the host (compat.HostSession, fs_step_host_ex)."""
    import types

    import numpy as np
    import torch

    from paper_2305_16510_b200 import compat
    from paper_2305_16510_b200.control import ControlGains, ControlLimits
    from paper_2305_16510_b200.dynamics import RobotParams
    if cfg["mode"] not in ("attitude", "velocity") or cfg.get("reset_prob") or cfg.get("stats") \
            or cfg.get("hetero") or cfg.get("airframe") or cfg.get("world") or cfg.get("render"):
        return None
    f = make_fleet(dict(cfg, global_n=n), n, first_id, 1234, device)
    st = f.state[:, :n].double().cpu().numpy()
    cm = f.cmd[:, :n].double().cpu().numpy()
    del f
    NS = types.SimpleNamespace
    states = NS(p=np.ascontiguousarray(st[0:3].T), q=np.ascontiguousarray(st[3:7].T),
                v=np.ascontiguousarray(st[7:10].T), omega=np.ascontiguousarray(st[10:13].T))
    mode = 1 if cfg["mode"] == "velocity" else 0
    z = np.zeros(n)
    att = NS(roll=cm[0] if mode == 0 else z, pitch=cm[1] if mode == 0 else z,
             yaw_rate=cm[2] if mode == 0 else z, thrust=cm[3] if mode == 0 else z)
    vel = NS(v=np.ascontiguousarray(cm[0:3].T) if mode == 1 else np.zeros((n, 3)),
             yaw_rate=cm[3] if mode == 1 else z)
    cmds = NS(mode=np.full(n, mode, np.uint8), attitude=att, velocity=vel)
    gains, params, limits = ControlGains(), RobotParams(), ControlLimits()
    states = compat.pipeline_step(states, cmds, gains, params, limits, cfg["dt"])   # warm-up
    torch.cuda.synchronize(device)
    t0 = time.perf_counter()
    for _ in range(steps):
        states = compat.pipeline_step(states, cmds, gains, params, limits, cfg["dt"])
    wall = time.perf_counter() - t0
    return {"value": n * steps / wall, "unit": UNIT, "wall_s": wall, "steps": steps,
            "h2d_bytes_per_step": int(n * 17 * 4), "d2h_bytes_per_step": int(n * 14 * 4),
            "path": "compat.pipeline_step (the flocksim drop-in) on float64 NumPy state and "
                    "command records: float64 rows packed into pinned fp32 planes and "
                    "unpacked into new float64 arrays by fs_host_pack_f64 / fs_host_unpack_f64 "
                    "(all host threads), fs_step_host_ex (8 chunks x 8 streams), every step"}


def _dist_on(world):
    """torch.distributed is in use: more than one rank, or FS_BENCH_FORCE_DIST=1
    (a one-rank NCCL run under torchrun: exercises the multi-GPU code path --
    communicator, barriers, max-over-ranks, the statistics all-reduce -- on a
    one-GPU box)."""
    return world > 1 or os.environ.get("FS_BENCH_FORCE_DIST") == "1"


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2305_16510_b200 import _native as N

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"WORLD_SIZE={world} but --gpus {args.gpus}"}))
        return 1
    if not torch.cuda.is_available():
        print(json.dumps({"metric": METRIC, "error": "no CUDA device"}))
        return 1
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    nccl = None
    if _dist_on(world):
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # communicator init lines (nranks, NVLS / NVLink transport) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # (a per-rank file, echoed to stderr below: NCCL_DEBUG_FILE=/dev/stderr
        # reopens -- and truncates -- a redirected stderr; stdout is the JSON line)
        import tempfile
        nlog = os.path.join(tempfile.gettempdir(), f"fs_nccl.{os.getpid()}.log")
        os.environ.setdefault("NCCL_DEBUG_FILE", nlog)
        dist.init_process_group("nccl", device_id=device)
        probe = torch.ones(1, device=device)
        dist.all_reduce(probe)           # forces communicator creation (logged)
        torch.cuda.synchronize(device)
        nccl = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version()),
                "allreduce_probe": float(probe.item())}
        try:
            with open(os.environ["NCCL_DEBUG_FILE"]) as f:
                lines = f.read().splitlines()
            sys.stderr.write("\n".join(lines) + "\n")
            nccl["init_lines"] = [ln.strip() for ln in lines
                                  if "nRanks" in ln or "Init COMPLETE" in ln][:4]
        except OSError:
            pass
    N.load()
    for key, val in ((N.FS_TUNE_PREC, args.prec), (N.FS_TUNE_NCW, args.ncw),
                     (N.FS_TUNE_KERNEL, args.kernel), (N.FS_TUNE_VPT, args.vpt),
                     (N.FS_TUNE_CHAIN_RELEASE, args.chain_release),
                     (N.FS_TUNE_CHAIN_ACQUIRE, args.chain_acquire),
                     (N.FS_TUNE_L2_KEEP_MB, args.l2_keep_mb),
                     (N.FS_TUNE_CLEAR_WALK_CM, args.clear_walk_cm),
                     (N.FS_TUNE_CLEAR_EXACT, args.clear_exact)):
        if val is not None:
            N.set_tuning(key, val)

    n, first_id, global_n, scaling = _shard(cfg, args, world, rank)
    cfg = dict(cfg, global_n=global_n)
    fleet = make_fleet(cfg, n, first_id, args.seed, device)
    K, W = args.steps, args.warmup

    # re-spawns are drawn inside the step kernel (cfg3); an obstacle World.step
    # is the warp-cooperative auto-reset kernel + the step kernel
    # (forest: the auto-reset kernel, the step, the deferred collision test)
    launches_per_step = (3 if getattr(fleet.world, "_worklist", None) is not None else 2) \
        if cfg.get("forest") else 1
    fleet_cfg = not (cfg.get("world") or cfg.get("render"))
    persistent = (args.launch == "persistent" and fleet_cfg and cfg["integrate"] and not args.eager
                  and getattr(fleet, "chainable", False))
    elapsed_ms, kern_ms, clocks = _time_fleet(fleet, cfg, args, K, W, world, device, dist,
                                              persistent)

    stats = None
    if cfg.get("stats"):
        from paper_2305_16510_b200.fleet import summarize_stats
        tot = fleet.stats_local()
        if _dist_on(world):
            dist.all_reduce(tot)          # int64 sums: identical for any GPU count
        stats = summarize_stats(tot.cpu())

    # the same K steps as K separate fs_step launches (one CUDA graph), timed
    # the same way (barriers, max over ranks).  The headline is the faster of
    # the two launch shapes at this shard size: the persistent launch wins
    # when a step streams many rounds of tiles per SM, K launches win on
    # small shards where one step is a few rounds (profiles/r2_launch_sweep)
    per_step = persistent_line = None
    if persistent:
        pms, pkern, pclocks = _time_fleet(fleet, cfg, args, K, W, world, device, dist, False)
        per_step = {"value": global_n * K / (pms * 1e-3), "unit": UNIT, "ms_per_step": pms / K,
                    "note": "K fs_step launches (one per step) replayed as one CUDA graph, "
                            "max over ranks"}
        persistent_line = {"value": global_n * K / (elapsed_ms * 1e-3), "unit": UNIT,
                           "ms_per_step": elapsed_ms / K,
                           "note": "one persistent fs_step_many launch of K steps, max over ranks"}
        if pms < elapsed_ms:
            elapsed_ms, kern_ms, clocks = pms, pkern, pclocks
            persistent = False

    # K-step rollout with the vehicles held in registers (fs_rollout)
    fused = None
    if cfg["integrate"] and not args.no_fused and fleet_cfg:
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

    bytes_per = cfg["bytes"]
    if persistent and cfg.get("out_bytes"):
        # a K-step launch writes the optional outputs (rotor thrusts) in its
        # last step only: they hold the last step's values (flocksim_b200.h)
        bytes_per = cfg["bytes"] - cfg["out_bytes"] + cfg["out_bytes"] / K
    forest_tested = forest_bytes = None
    if cfg.get("forest"):
        wl = getattr(fleet.world, "_worklist", None)
        if wl is not None:
            # algorithmic bytes per env-step, averaged over the run:
            #  * every env: World.step's 211 B + the clearance-cache planes (16 B);
            #  * each env the cache does not clear (forest_tested): its instance
            #    broad phase (32 B per instance) + the cache write (16 B), and the
            #    96-B slot records its test walked (counted by the kernel,
            #    fs_obstacles.walk_slots: data dependent);
            #  * each auto-reset env (rate from the last step's info bits): its
            #    rebuilt scene rows (96 B per slot) + instance boxes (32 B); the
            #    instance poses are not written (computed on demand)
            w = fleet.world
            forest_tested = int(wl[2].item())
            steps_taken = K + W
            t_rate = forest_tested / max(1, steps_taken) / n
            ws = getattr(w, "_walk_slots", None)
            walked = int(ws.item()) if ws is not None else 0
            k_rate = walked / max(1, steps_taken) / n
            r_rate = float(((w._info[:n] & N.FS_INFO_AUTORESET) != 0).float().mean().item())
            j = w.instances_per_env
            bytes_per = (211 + 16 + t_rate * (32 * j + 16) + k_rate * 96 +
                         r_rate * (96 * w.pset.width + 32 * j))
            forest_bytes = {"per_env_base": 227, "tested_fraction": t_rate,
                            "walked_slots_per_env": k_rate, "reset_fraction": r_rate,
                            "scene_width": w.pset.width, "instances": j,
                            "per_env_without_walk": bytes_per - k_rate * 96}
        else:
            # World.step's 211 B + the instance broad phase (one 32-B record per
            # obstacle instance); the narrow phase is data dependent
            bytes_per = 211 + 32 * fleet.world.instances_per_env
    elif cfg.get("render"):
        cam = fleet.cam
        bytes_per = cam.width * cam.height * 8     # depth f32 + segmentation i32 written

    e2e = e2e_np = None
    if not args.no_e2e:
        es = max(3, min(K, args.e2e_steps))
        if cfg.get("render"):
            e2e = measure_render_e2e(fleet, device, es)
        else:
            del fleet
            torch.cuda.empty_cache()
            fleet = None
            e2e = measure_e2e(cfg, n, device, es, first_id=first_id)
            e2e_np = measure_e2e_numpy(cfg, n, device, max(2, min(es, 5)), first_id=first_id)
            if e2e_np is not None:
                wt = torch.tensor([e2e_np.pop("wall_s")], dtype=torch.float64, device=device)
                if _dist_on(world):
                    dist.all_reduce(wt, op=dist.ReduceOp.MAX)
                e2e_np["value"] = global_n * e2e_np["steps"] / float(wt.item())
        if e2e is not None and _dist_on(world):
            et = torch.tensor([e2e.pop("wall_s", 0.0)], dtype=torch.float64, device=device)
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
            e2e["value"] = global_n * e2e["steps"] / float(et.item())
        elif e2e is not None:
            e2e.pop("wall_s", None)
    fleet = None
    torch.cuda.empty_cache()

    avg_kernel_s = statistics.mean(kern_ms) * 1e-3
    peak, peak_kind = _peaks()
    achieved = bytes_per * n / avg_kernel_s / 1e9
    value = global_n * K / (elapsed_ms * 1e-3)
    traffic, traffic_src = _traffic(args.config, n, persistent)

    north = None
    if args.config == DEFAULT_CONFIG and not args.no_north_star:
        north = _north_star(args, world, rank, local, device, dist, peak)

    cpu = None
    if rank == 0 and not args.no_cpu:
        if cfg.get("forest") or cfg.get("render"):
            cpu = scene_cpu_run("render" if cfg.get("render") else "forest", 2, 1)
            cpu.pop("wall_s")
        else:
            cpu = cpu_baseline("velocity" if cfg["mode"] == "mixed" else cfg["mode"])
            cpu.pop("wall_s", None)
            cpu.pop("n", None)
    if _dist_on(world):
        dist.barrier()

    if rank == 0:
        unit = cfg.get("unit", "env-steps/s" if cfg.get("world") else UNIT)
        work_set = n * (68 if fleet_cfg else bytes_per)
        line = {
            "metric": cfg.get("metric", "env-steps/sec (World.step)" if cfg.get("world")
                              else METRIC),
            "value": value, "unit": unit, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": elapsed_ms / K, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": (value / PUBLISHED_STEPS_PER_S if fleet_cfg
                                                else None),
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "vehicles_per_gpu": n,
                       "vehicles_total": global_n, "mode": cfg["mode"], "dt": cfg["dt"],
                       "shards": "contiguous [(n k)//N, (n (k+1))//N) per rank "
                                 "(dynamics.py:267-283)" if scaling == "strong" else
                                 f"{n} per rank",
                       "parallelism": f"dp{world}",
                       "l2": _l2_label(traffic, bytes_per * n, work_set),
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
                         "traffic": traffic, "traffic_source": traffic_src,
                         ("bytes_per_frame" if cfg.get("render") else "bytes_per_vehicle_step"):
                             bytes_per,
                         "kernel_ms_avg": avg_kernel_s * 1e3,
                         "note": "achieved = algorithmic bytes of rank 0's shard / its "
                                 "average step time (CUDA events on the launching stream)"},
            "clocks": clocks,
            "gpu_launches": 1 if persistent else K * launches_per_step,
            "e2e": e2e,
            "e2e_numpy_dropin": e2e_np,
            "cpu_baseline": cpu,
            "rollout_fused": fused,
        }
        if nccl is not None:
            line["nccl"] = nccl
        if per_step is not None:
            line["per_step_launches"] = per_step
            line["persistent_launch"] = persistent_line
        if fleet_cfg:
            line["vs_baseline_basis"] = ("value / 3.8e6: BASELINE.md's published aggregate "
                                         "steps/s (Aerial Gym paper, PAPER.md:140: 2^17 robots, "
                                         "controllers + PhysX, 2x RTX 3090); a different "
                                         "configuration, the closest published figure")
        if stats is not None:
            line["episode_stats"] = stats
        if north is not None:
            line["north_star"] = north
        if cfg.get("render"):
            line["roofline_issue"] = _render_issue_roofline(K, elapsed_ms, n)
        elif args.config in ISSUE_CAPTURES:
            line["roofline_issue"] = _issue_roofline(args.config, n * K / (elapsed_ms * 1e-3))
        if forest_tested is not None:
            line["collision_tests"] = {
                "envs_tested_per_step": forest_tested / max(1, K + W),
                "fraction": forest_tested / max(1, K + W) / n,
                "algorithmic_bytes": forest_bytes,
                "note": "envs per step whose collision test ran (the clearance cache did not "
                        "clear them), averaged over every step the world took (warm-up + timed)"}
        print(json.dumps(line))
    if _dist_on(world):
        dist.destroy_process_group()
    return 0


def _render_issue_roofline(K, elapsed_ms, n):
    """The renderer is bound by instruction issue, not HBM: its fraction of
    the SM issue ceiling (148 SMs x 4 warp-schedulers x 32 lanes x clock),
    from the ncu-measured thread-instructions per ray
    (profiles/ncu_summary.json 'render')."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            r = json.load(f)["render"]
        inst = float(r["thread_inst_per_ray"])
    except Exception:
        return None
    rays = 480 * 270 * n
    achieved = inst * rays / (elapsed_ms / K * 1e-3)
    peak = 148 * 4 * 32 * 1.965e9
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "thread-inst/s",
            "frac": achieved / peak, "inst_per_ray": inst,
            "note": "achieved = ncu thread-instructions per ray x rays per frame batch / the "
                    "measured batch time; peak = 148 SMs x 4 schedulers x 32 lanes x 1.965 GHz"}


# warp-instructions per vehicle-step of the dominant kernel, from committed
# ncu --set full captures (smsp__inst_executed.sum / vehicles / steps)
ISSUE_CAPTURES = {
    "cfg2": ("profiles/raw/r2s2_ncu_raw_cfg2.csv", 1 << 22, 20),
    "cfg3": ("profiles/raw/r2s2_ncu_raw_cfg3_2097152.csv", 1 << 21, 20),
    "cfg4": ("profiles/raw/r1_ncu_raw_cfg4_persistent.csv", 1 << 23, 20),
}


def _issue_roofline(config, vehicle_steps_per_s_per_gpu):
    """The fused step is bound by instruction issue, not HBM, once the
    statistics, re-spawns or rotor allocation are on: its
    fraction of the SM issue ceiling (148 SMs x 4 warp-schedulers x 1.965 GHz
    warp-instructions/s) from the ncu-measured warp-instructions per
    vehicle-step of a committed capture."""
    import csv
    e = ISSUE_CAPTURES.get(config)
    if e is None:
        return None
    try:
        with open(os.path.join(ROOT, e[0])) as f:
            rows = list(csv.reader(f))
        winst = float(rows[2][rows[0].index("smsp__inst_executed.sum")].replace(",", ""))
    except Exception:
        return None
    per_veh = winst / (e[1] * e[2])
    achieved = per_veh * vehicle_steps_per_s_per_gpu
    peak = 148 * 4 * 1.965e9
    return {"bound": "issue", "achieved": achieved, "peak": peak, "unit": "warp-inst/s",
            "frac": achieved / peak, "warp_inst_per_vehicle_step": per_veh,
            "source": f"{e[0]} (ncu --set full: smsp__inst_executed.sum / {e[1]} vehicles / "
                      f"{e[2]} steps)",
            "note": "achieved = warp-instructions per vehicle-step x this GPU's vehicle-steps/s; "
                    "peak = 148 SMs x 4 schedulers x 1.965 GHz"}


def dry_run(args, cfg):
    """CPU check of the multi-rank plumbing (no GPU work): gloo process group,
    every rank's shard bounds, the max-over-ranks timing reduction and the
    int64 statistics all-reduce.  Rank 0 prints one JSON line."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        print(json.dumps({"error": f"WORLD_SIZE={world} but --gpus {args.gpus}"}))
        return 1
    if _dist_on(world):
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    n, first_id, global_n, scaling = _shard(cfg, args, world, rank)
    mine = torch.tensor([rank, n, first_id, global_n], dtype=torch.int64)
    rows = [torch.zeros(4, dtype=torch.int64) for _ in range(world)]
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    stats = torch.tensor([n, rank, 1], dtype=torch.int64)
    if _dist_on(world):
        dist.all_gather(rows, mine)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(stats)
    else:
        rows = [mine]
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "workload": args.config,
                          "scaling": scaling, "vehicles_total": global_n,
                          "shards": [{"rank": int(r[0]), "n": int(r[1]), "first_id": int(r[2])}
                                     for r in rows],
                          "max_over_ranks": float(t.item()),
                          "stats_sum": [int(x) for x in stats]}))
    if _dist_on(world):
        dist.destroy_process_group()
    return 0


def _spawn_ranks(args, argv):
    """Re-execute this script under torch.distributed.run with --gpus ranks
    (the driver's own launch shape: 127.0.0.1 rendezvous, one rank per GPU)."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__), *argv]
    return subprocess.run(cmd).returncode


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
    ap.add_argument("--chain-acquire", type=int, default=None,
                    help="chained steps, load side: bit 0 acquire counter loads, bit 1 proxy "
                         "fence (default 2), bit 2 fence.acq_rel.gpu")
    ap.add_argument("--clear-walk-cm", type=int, default=None,
                    help="obstacle worlds: clearance-cache slot-walk radius (cm)")
    ap.add_argument("--clear-exact", type=int, default=None,
                    help="obstacle worlds: 1 walked slots bound the clearance by their SDF")
    ap.add_argument("--north-star-steps", type=int, default=1000,
                    help="steps of the north_star sub-measurement (config 3 at 2^24 total)")
    ap.add_argument("--no-north-star", action="store_true")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU check of the multi-rank plumbing (gloo): print each rank's shard")
    raw = list(sys.argv[1:] if argv is None else argv)
    args = ap.parse_args(raw)
    cfg = CONFIGS[args.config]
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _spawn_ranks(args, raw)
    if args.dry_run:
        return dry_run(args, cfg)
    if args.steps is None:
        args.steps = cfg["steps"] if args.impl == "ours" else 10
    args.warmup = max(3, args.warmup) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
