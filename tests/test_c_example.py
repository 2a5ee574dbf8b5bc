"""The drop-in boundary from plain C (examples/c_abi_step.c): it builds
against include/flocksim_b200.h and the in-tree library with gcc alone (CPU),
and on a B200 K fs_step calls equal one fs_step_many(K) launch bitwise."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EX = os.path.join(ROOT, "examples")


def _build():
    from paper_2305_16510_b200 import build
    build.build()
    if shutil.which("gcc") is None or not os.path.exists("/usr/local/cuda/include/cuda_runtime.h"):
        pytest.skip("gcc or the CUDA headers are not available")
    r = subprocess.run(["make", "-B", "-C", EX], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "warning" not in r.stderr.lower(), r.stderr
    return os.path.join(EX, "c_abi_step")


def test_c_example_builds_with_gcc_alone():
    assert os.access(_build(), os.X_OK)


@pytest.mark.gpu
@pytest.mark.parametrize("n,k", [(1 << 16, 10), (300001, 7), (5000, 3)])
def test_c_example_runs(n, k):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    exe = _build()
    r = subprocess.run([exe, str(n), str(k)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 differing values" in r.stdout or "refused" in r.stdout, r.stdout
