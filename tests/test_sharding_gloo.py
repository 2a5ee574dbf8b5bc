"""Multi-process sharding on CPU (gloo, world_size 2).

The N>1 path of the build: each rank owns the contiguous global ids
shard_bounds(n, W, rank) (dynamics.py:269), steps them with no per-step
collective, and the per-rollout episode statistics (int64 fixed point) are
summed with one all_reduce.  Here the per-rank stepping is the CPU oracle
(position mode, with the device RNG twin's Bernoulli re-spawns), so the test
exercises exactly the host logic the GPU ranks use: the shard bounds, the
global-id RNG keying and the statistics reduction -- and checks that the
2-rank result is bitwise identical to the 1-rank result.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N_VEH = 96
STEPS = 12
SEED = 9
P_RESET = 0.05


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def run_shard(lo, hi):
    """Oracle rollout of global ids [lo, hi): returns int64 [err, crash, count]."""
    from oracle import flocksim_oracle as O
    from oracle import rng_twin as R
    gid = np.arange(lo, hi, dtype=np.uint64)
    s, cmd = R.spawn(SEED, gid, R.INIT_STEP, "position")
    err_sum = crash = count = 0
    for k in range(STEPS):
        reset = R.reset_mask(SEED, gid, k, P_RESET)
        if reset.any():
            s2, c2 = R.spawn(SEED, gid, k, "position")
            s[:, reset], cmd[:, reset] = s2[:, reset], c2[:, reset]
        f, m, _ = O.position_control(s, cmd[0:3], cmd[3], O.Gains(), O.Robot(), O.Limits())
        s_new, clamped, nonfinite = O.integrate(s, f, m, O.Robot(), 0.01)
        s = np.where(reset[None, :], s, s_new)
        live = ~reset
        e = np.sqrt(((s[0:3] - cmd[0:3]) ** 2).sum(axis=0)).astype(np.float32)
        bad = (clamped | nonfinite) & live
        fixed = np.rint(e.astype(np.float64) * 2.0 ** 20).astype(np.int64)
        err_sum += int(fixed[live & ~bad].sum())
        crash += int(bad.sum())
        count += int(live.sum())
    return np.array([err_sum, crash, count], dtype=np.int64), s


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    from paper_2305_16510_b200 import parallel
    r, w = parallel.init(backend="gloo")
    assert (r, w) == (rank, world)
    lo, hi = parallel.shard_bounds(N_VEH, world, rank)
    stats, state = run_shard(lo, hi)
    t = torch.from_numpy(stats.copy())
    parallel.allreduce_stats(t)
    mx = parallel.max_over_ranks(float(rank))
    gathered = [torch.zeros(13, hi - lo + 1, dtype=torch.float64) for _ in range(world)]
    # shard sizes may differ: gather with padding via all_gather_object
    objs = [None] * world
    dist.all_gather_object(objs, (lo, hi, state))
    if rank == 0:
        full = np.zeros((13, N_VEH))
        for lo_, hi_, st in objs:
            full[:, lo_:hi_] = st
        np.savez(out_path, stats=t.numpy(), state=full, maxr=mx)
    dist.barrier()
    dist.destroy_process_group()
    del gathered


@pytest.mark.parametrize("world", [2])
def test_two_rank_rollout_statistics_match_single_rank(tmp_path, world):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = np.load(out)
    single_stats, single_state = run_shard(0, N_VEH)
    assert np.array_equal(res["stats"], single_stats)
    assert np.array_equal(res["state"], single_state)
    assert res["maxr"] == world - 1
    assert single_stats[2] > 0 and single_stats[2] < N_VEH * STEPS   # resets happened


def test_shard_bounds_cover_and_partition():
    from paper_2305_16510_b200.parallel import shard_bounds
    for n in (1, 7, 257, 1 << 20):
        for w in (1, 2, 3, 4, 8):
            b = [shard_bounds(n, w, k) for k in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[k][1] == b[k + 1][0] for k in range(w - 1))
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)
