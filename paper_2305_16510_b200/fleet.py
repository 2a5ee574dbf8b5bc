"""Device-resident fleet: in-place fused steps, K-step rollouts, CUDA graphs,
sharding and episode statistics.

This is the B200 replacement for the reference's hot loops
(bench_dynamics, bench.py:161-167; World._step_dynamics, world.py:259-275):
the state (13 fp32 planes) and commands (4 or 8 planes) stay in HBM, one
fused kernel advances every vehicle per control step, and nothing returns
to the host inside a rollout.  A shard of a multi-GPU fleet owns the
contiguous global ids [first_id, first_id + n) with the reference's bounds
formula (dynamics.py:269); the device RNG is keyed by global id so every
sharding of a fleet is bitwise identical per vehicle.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as N
from ._tensors import alloc_planes, default_device, ptr, stride0, stream_handle
from .allocation import Airframe, native_pair
from .control import ControlGains, ControlLimits
from .dynamics import RigidStateBatch, RobotParams
from .parallel import shard_bounds  # noqa: F401  (re-export)

STATS_SLOTS = 1024
CHAIN_MIN_N = 1 << 15             # the streaming kernel's minimum batch (chained steps)
FIXED_POINT = float(1 << 20)      # |p - p_d| units in the statistic sums


class Fleet:
    """n vehicles of one shard with their commands, kept in HBM.

    mode: 'attitude' | 'velocity' | 'position' | 'mixed'
    airframes: None, or (first, second) with `airframe_split` (global id)
    hetero: per-vehicle mass and diagonal inertia planes
    """

    MODES = {"attitude": N.FS_MODE_ATTITUDE, "velocity": N.FS_MODE_VELOCITY,
             "mixed": N.FS_MODE_MIXED, "position": N.FS_MODE_POSITION}

    def __init__(self, n: int, mode: str = "velocity", dt: float = 0.01, seed: int = 0,
                 first_id: int = 0, params: RobotParams | None = None,
                 gains: ControlGains | None = None, limits: ControlLimits | None = None,
                 airframes: tuple | None = None, airframe_split: int = 0,
                 rotor_dynamics: bool = False, hetero: bool = False,
                 reset_prob: float = 0.0, want_flags: bool = False, want_wrench: bool = False,
                 want_stats: bool = False, device=None):
        if mode not in self.MODES:
            raise ValueError(f"mode must be one of {sorted(self.MODES)}, got '{mode}'")
        if not 0.0 < dt <= 0.1:
            raise ValueError(f"dt must be in (0, 0.1], got {dt}")
        self.lib = N.load()
        self.device = device if device is not None else default_device()
        self.n, self.mode_name, self.mode = int(n), mode, self.MODES[mode]
        self.dt, self.seed, self.first_id = float(dt), int(seed), int(first_id)
        self.params = params or RobotParams()
        self.gains = gains or ControlGains()
        self.limits = limits or ControlLimits()
        self._robot = self.params.native()
        self._gains = self.gains.native()
        self._limits = self.limits.native()
        self.airframes = airframes
        self._frames = native_pair(*airframes) if airframes else None
        self.airframe_split = int(airframe_split)
        self.rotor_dynamics = bool(rotor_dynamics)
        self.reset_prob = float(reset_prob)
        self.step_index = 0

        nc = 8 if self.mode == N.FS_MODE_MIXED else 4
        self.state = alloc_planes(13, n, self.device)
        self.cmd = alloc_planes(nc, n, self.device)
        self.mode_plane = (torch.zeros(n, dtype=torch.uint8, device=self.device)
                           if self.mode == N.FS_MODE_MIXED else None)
        self.vparams = alloc_planes(4, n, self.device) if hetero else None
        self.rotors = (alloc_planes(N.FS_MAX_ROTORS, n, self.device, zero=True)
                       if airframes else None)
        self.flags = torch.zeros(max(n, 1), dtype=torch.uint8, device=self.device) \
            if want_flags else None
        self.wrench = alloc_planes(4, n, self.device) if want_wrench else None
        self.stats_slots = (torch.zeros((STATS_SLOTS, 3), dtype=torch.int64, device=self.device)
                            if want_stats else None)
        # chained steps (fs_step_desc.tile_sync): per-128-vehicle step counters
        self.chainable = n >= CHAIN_MIN_N
        self.tile_sync = (torch.zeros(max(1, int(self.lib.fs_tile_sync_len(n))),
                                      dtype=torch.int32, device=self.device)
                          if self.chainable else None)
        self.reset_fleet()

    # -- setup ---------------------------------------------------------------
    def reset_fleet(self) -> None:
        """Seeded spawn of every vehicle (fs_init_fleet; BASELINE config draws)."""
        with torch.cuda.device(self.device):
            N.check(self.lib.fs_init_fleet(
                self.n, self.first_id, self.seed, self.mode, ptr(self.state), stride0(self.state),
                ptr(self.cmd), stride0(self.cmd), ptr(self.vparams),
                stride0(self.vparams) if self.vparams is not None else 0, self._robot,
                stream_handle()), "init_fleet")
        if self.stats_slots is not None:
            self.stats_slots.zero_()
        self.step_index = 0

    def states(self) -> RigidStateBatch:
        return RigidStateBatch.from_planes(self.state, self.n)

    # -- stepping ------------------------------------------------------------
    def _desc(self, integrate: bool = True) -> N.fs_step_desc:
        d = N.fs_step_desc()
        d.n = self.n
        d.first_id = self.first_id
        d.state_in = d.state_out = ptr(self.state)
        d.state_in_stride = d.state_out_stride = stride0(self.state)
        d.mode = self.mode
        d.integrate = 1 if integrate else 0
        d.mode_per_vehicle = ptr(self.mode_plane)
        d.cmd = ptr(self.cmd)
        d.cmd_stride = stride0(self.cmd)
        d.vparams = ptr(self.vparams)
        d.vparams_stride = stride0(self.vparams) if self.vparams is not None else 0
        d.airframe_split = self.airframe_split
        d.wrench_out = ptr(self.wrench)
        d.wrench_stride = stride0(self.wrench) if self.wrench is not None else 0
        d.rotor_out = ptr(self.rotors)
        d.rotor_stride = stride0(self.rotors) if self.rotors is not None else 0
        d.flags_out = ptr(self.flags)
        d.rotor_dynamics = 1 if self.rotor_dynamics else 0
        d.dt = self.dt
        d.reset_prob = self.reset_prob
        d.seed = self.seed
        d.step_index = self.step_index
        d.stats_slots = ptr(self.stats_slots)
        d.stats_nslots = STATS_SLOTS if self.stats_slots is not None else 0
        return d

    def step(self, stream=None, chain: int | None = None) -> None:
        """One fused control + integration step of every vehicle, in place.

        chain=k (k >= 0): the k-th step of a chain started by `_chain_start`
        (waits for step k-1's tiles, publishes k+1; see fs_step_desc.tile_sync)."""
        d = self._desc(True)
        if chain is not None:
            d.tile_sync = ptr(self.tile_sync)
            d.sync_wait = chain
            d.sync_post = chain + 1
        N.check(self.lib.fs_step(C.byref(d), self._robot, self._gains, self._limits,
                                 self._frames, stream or stream_handle(self.device)), "fs_step")
        self.step_index += 1

    def _chain_start(self, stream) -> None:
        """Zero the step counters on `stream` (chain step 0 waits for
        nothing; the zeroing is ordered before it like any stream op)."""
        if stream is None:
            self.tile_sync.zero_()
        else:
            h = stream.value if isinstance(stream, C.c_void_p) else int(stream)
            with torch.cuda.stream(torch.cuda.ExternalStream(h, device=self.device)):
                self.tile_sync.zero_()

    def _steps(self, steps: int, stream, chained: bool) -> None:
        if chained and self.chainable and steps > 1:
            self._chain_start(stream)
            for k in range(steps):
                self.step(stream, chain=k)
        else:
            for _ in range(steps):
                self.step(stream)

    def control(self, stream=None) -> None:
        """Control only (no integration): wrench / rotor thrusts / flags."""
        d = self._desc(False)
        N.check(self.lib.fs_step(C.byref(d), self._robot, self._gains, self._limits,
                                 self._frames, stream or stream_handle(self.device)), "fs_control")

    def step_many(self, steps: int, stream=None) -> None:
        """`steps` fused steps in one persistent launch of the streaming
        kernel (fs_step_many): every step reads and writes the fleet in HBM
        like `step`, bitwise the same result, without a launch boundary
        between steps.  Needs the streaming kernel (n >= 2^15)."""
        if not self.chainable:
            raise ValueError(f"step_many needs n >= {CHAIN_MIN_N} (streaming kernel), got {self.n}")
        self._chain_start(stream)
        d = self._desc(True)
        d.tile_sync = ptr(self.tile_sync)
        d.sync_wait, d.sync_post = 0, 1
        N.check(self.lib.fs_step_many(C.byref(d), self._robot, self._gains, self._limits,
                                      self._frames, int(steps),
                                      stream or stream_handle(self.device)), "fs_step_many")
        self.step_index += steps

    def rollout(self, steps: int, fused: bool = False, stream=None, chained: bool = False,
                persistent: bool = False) -> None:
        """`steps` control steps.  fused=False: the state round-trips HBM every
        step (commands may change between steps); persistent: all steps in
        one streaming launch (`step_many`), else one launch per step, chained
        so that consecutive steps overlap -- all bitwise the same result as
        unchained launches.  fused=True: one kernel, vehicles held in
        registers for all steps (fs_rollout)."""
        if fused:
            d = self._desc(True)
            N.check(self.lib.fs_rollout(C.byref(d), self._robot, self._gains, self._limits,
                                        self._frames, int(steps),
                                        stream or stream_handle(self.device)), "fs_rollout")
            self.step_index += steps
        elif persistent and self.chainable:
            self.step_many(steps, stream)
        else:
            self._steps(steps, stream, chained)

    def capture(self, steps: int, integrate: bool = True, chained: bool = False,
                persistent: bool = False) -> torch.cuda.CUDAGraph:
        """Capture `steps` steps into a CUDA graph.  Replaying it advances the
        fleet by `steps` steps (RNG counters baked at capture: call once per
        replay window, or use reset_prob == 0).  chained: the graph zeroes
        the step counters, then runs the per-step launches as one chain;
        persistent: one fs_step_many launch instead."""
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                h = C.c_void_p(s.cuda_stream)
                if integrate and persistent and self.chainable:
                    self.step_many(steps, h)
                elif integrate:
                    self._steps(steps, h, chained)
                else:
                    for _ in range(steps):
                        self.control(h)
        torch.cuda.current_stream(self.device).wait_stream(s)
        return g

    # -- statistics ----------------------------------------------------------
    def stats_local(self) -> torch.Tensor:
        """(3,) int64 on device: [sum |p - p_d| * 2^20, crashes, samples]."""
        if self.stats_slots is None:
            raise RuntimeError("fleet was created without want_stats")
        out = torch.empty(3, dtype=torch.int64, device=self.device)
        with torch.cuda.device(self.device):
            N.check(self.lib.fs_stats_reduce(ptr(self.stats_slots), STATS_SLOTS, ptr(out),
                                             stream_handle()), "stats_reduce")
        return out


def summarize_stats(totals) -> dict:
    """Host summary of reduced [err_fixed, crashes, samples]."""
    t = [int(x) for x in (totals.tolist() if hasattr(totals, "tolist") else totals)]
    ok = max(1, t[2] - t[1])
    return {"mean_position_error_m": t[0] / FIXED_POINT / ok, "crashes": t[1], "samples": t[2]}


__all__ = ["Fleet", "shard_bounds", "summarize_stats", "Airframe", "STATS_SLOTS"]
