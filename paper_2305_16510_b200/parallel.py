"""Multi-GPU plumbing: contiguous vehicle shards, one process per GPU.

The path has no per-step exchange: vehicles are independent
(dynamics.py:18-19), so each rank owns the contiguous global
ids [(n k)//W, (n (k+1))//W) -- the reference's own partition formula
(dynamics.py:269-270) -- and steps them with no collective.  The only
collective is the per-rollout reduction of episode statistics (BASELINE
config 3): three int64 fixed-point sums, whose addition is associative, so
the reduced statistics are bitwise identical for 1/2/4/8 GPUs.  Backend:
NCCL over NVLink on GPUs, gloo for the CPU tests.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard of rank `rank` (dynamics.py:269-270)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    return (n * rank) // world, (n * (rank + 1)) // world


def env_ranks() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None, device: torch.device | None = None) -> tuple[int, int]:
    """Initialise the process group when WORLD_SIZE > 1; returns (rank, world)."""
    rank, world, _ = env_ranks()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        kw = {"device_id": device} if backend == "nccl" and device is not None else {}
        dist.init_process_group(backend, **kw)
    return rank, world


def allreduce_stats(totals: torch.Tensor) -> torch.Tensor:
    """Sum the (3,) int64 episode statistics over ranks, in place."""
    if totals.dtype != torch.int64:
        raise TypeError("statistics must be int64 fixed point")
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(totals, op=dist.ReduceOp.SUM)
    return totals


def max_over_ranks(x: float, device=None) -> float:
    """Max of a scalar over ranks (timing: the slowest rank defines the step)."""
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
