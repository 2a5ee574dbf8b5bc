"""CPU tests of the benchmark-harness mirror (flocksim.bench,
pkg/src/flocksim/bench.py; reference tests pkg/tests/test_bench.py:20-77):
argument validation precedes any device work, and the report object keeps
the reference's fields, JSON and summary."""

import json

import pytest

from paper_2305_16510_b200 import bench as B


def test_reference_names_present():
    for name in ("BenchReport", "bench_dynamics", "bench_render", "image_checksum",
                 "make_bench_batch", "state_checksum", "bench_scene_config",
                 "machine_descriptor", "DEFAULT_DT", "WARMUP_STEPS"):
        assert hasattr(B, name)
    assert B.DEFAULT_DT == 0.01 and B.WARMUP_STEPS == 100


def test_invalid_args_rejected_before_device_work():
    # (no GPU in this container: these must raise ValueError, not a CUDA error)
    with pytest.raises(ValueError):
        B.bench_dynamics(num_envs=0, steps=10)
    with pytest.raises(ValueError, match="mode"):
        B.bench_dynamics(num_envs=4, steps=10, mode="position")
    with pytest.raises(ValueError, match="dt"):
        B.bench_dynamics(num_envs=4, steps=10, dt=0.5)
    with pytest.raises(ValueError):
        B.bench_render(num_envs=0, frames=1)
    with pytest.raises(ValueError):
        B.bench_render(num_envs=1, frames=0)


def test_report_json_and_summary(tmp_path):
    r = B.BenchReport(num_envs=4, total_steps=10, wall_seconds=0.5, steps_per_second=80.0,
                      sim_to_real_ratio=0.8, dt=0.01, checksum="ab", mode="velocity",
                      engine="fs_step_many (one persistent launch)", machine="m")
    path = tmp_path / "report.json"
    r.write_json(path)
    data = json.loads(path.read_text())
    assert data["num_envs"] == 4 and data["checksum"] == "ab"
    assert data["resolution"] is None
    s = r.summary()
    assert "aggregate rate:   80 env-steps/s" in s and "mode:             velocity" in s
    rr = B.BenchReport(num_envs=2, total_steps=3, wall_seconds=1.0, steps_per_second=6.0,
                       sim_to_real_ratio=0.0, dt=0.0, checksum="x", frames_per_second=6.0,
                       resolution=(48, 32), mode="render", machine="m")
    assert rr.to_dict()["resolution"] == [48, 32]
    assert "resolution:       48x32" in rr.summary()
