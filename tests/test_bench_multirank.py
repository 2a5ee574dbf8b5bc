"""CPU tests of bench.py's multi-GPU plumbing and its reference arm.

`bench.py --gpus N` re-executes itself under torch.distributed.run with N
ranks when no torchrun environment is present; `--dry-run` runs the rank
plumbing on gloo with no GPU work (shard bounds from the reference's
partition formula, dynamics.py:267-283; the max-over-ranks timing reduction;
the int64 statistics all-reduce).  `--impl reference` times the unmodified
reference (oracle/_ref) on the host cores.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus,config,total", [(2, "cfg2", 1 << 22), (4, "cfg3", 1 << 24),
                                               (3, "cfg4", 1 << 23)])
def test_bench_spawns_n_ranks_with_reference_shards(gpus, config, total):
    out = _run("--gpus", str(gpus), "--config", config, "--dry-run")
    assert out["n_gpus"] == gpus
    assert out["scaling"] == "strong"
    assert out["vehicles_total"] == total
    shards = sorted(out["shards"], key=lambda r: r["rank"])
    assert [r["rank"] for r in shards] == list(range(gpus))
    for k, r in enumerate(shards):
        assert r["first_id"] == (total * k) // gpus
        assert r["n"] == (total * (k + 1)) // gpus - (total * k) // gpus
    assert sum(r["n"] for r in shards) == total
    assert out["max_over_ranks"] == float(gpus)
    assert out["stats_sum"] == [total, gpus * (gpus - 1) // 2, gpus]


def test_bench_single_rank_dry_run_and_weak_configs():
    out = _run("--dry-run")
    assert out["n_gpus"] == 1 and out["vehicles_total"] == 1 << 22
    out = _run("--gpus", "2", "--config", "world", "--dry-run")
    assert out["scaling"] == "weak"
    assert [r["first_id"] for r in sorted(out["shards"], key=lambda r: r["rank"])] == \
        [0, 1 << 22]


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--dry-run"], capture_output=True, text=True, timeout=300, env=env,
                         cwd=ROOT)
    assert res.returncode == 1
    assert "WORLD_SIZE=1" in res.stdout


def test_reference_arm_times_the_unmodified_reference():
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built (python oracle/build_ref.py)")
    out = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert out["impl"] == "reference"
    assert out["cpu_baseline"]["kind"] == "reference"
    assert out["cpu_baseline"]["cores"] == os.cpu_count()
    assert out["value"] > 0 and out["e2e"]["value"] == out["value"]
    assert out["e2e"]["h2d_bytes_per_step"] == 0
    rb = out["reference_bench_dynamics"]
    assert rb["workers_1"] > 0 and rb[f"workers_{os.cpu_count()}"] > 0
    # position-mode configs have no reference code: the extension oracle
    out = _run("--impl", "reference", "--config", "cfg3", "--steps", "1", "--warmup", "0")
    assert out["cpu_baseline"]["kind"] == "port"


def test_issue_roofline_from_committed_captures():
    """bench.py's roofline_issue: warp-instructions per vehicle-step read from
    the committed ncu captures (profiles/raw), against 148 x 4 x 1.965 GHz."""
    import bench
    for cfg, lo, hi in (("cfg2", 12.0, 20.0), ("cfg3", 16.0, 26.0), ("cfg4", 16.0, 26.0)):
        r = bench._issue_roofline(cfg, 1e10)
        assert r is not None and r["bound"] == "issue", cfg
        assert lo < r["warp_inst_per_vehicle_step"] < hi, (cfg, r)
        assert r["peak"] == pytest.approx(148 * 4 * 1.965e9)
        assert r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert bench._issue_roofline("world", 1e10) is None


def test_force_dist_flag(monkeypatch):
    import bench
    monkeypatch.delenv("FS_BENCH_FORCE_DIST", raising=False)
    assert not bench._dist_on(1) and bench._dist_on(2)
    monkeypatch.setenv("FS_BENCH_FORCE_DIST", "1")
    assert bench._dist_on(1)
