"""Recipe: build the UNMODIFIED reference (flocksim + flocksim_rl) into
wheels under oracle/_ref/ as test infrastructure.

TEST INFRASTRUCTURE.  The reference is pure Python/NumPy, so "building" it
is an offline `pip wheel` of its own sources into a git-ignored directory
(oracle/_ref/ is listed in .gitignore but NOT in .gpurunignore, so it travels
to the GPU box with the snapshot, like the built .so).  It is used only by
tests/, __graft_entry__.smoke() and bench.py's CPU legs: as the CPU baseline
(`cpu_baseline.kind = "reference"`) and as the caller the drop-in adapter
(paper_2305_16510_b200/compat.py) is swapped into.  The product package
never imports it.

    python oracle/build_ref.py          # (also run by __graft_entry__.build())

/root/reference is read-only, so the sources are copied to a temporary
directory first and pip builds from there (--no-index, --no-build-isolation,
--no-deps: numpy / PyYAML / Pillow are already in the image).  The two
pure-Python wheels are imported straight from the archives (zipimport,
oracle/ref.py), so no loose copy of the reference's sources sits in the tree.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = "/root/reference/pkg"
TARGET = os.path.join(HERE, "_ref")
STAMP = os.path.join(TARGET, ".installed_from")


def wheels() -> list:
    if not os.path.isdir(TARGET):
        return []
    return sorted(os.path.join(TARGET, f) for f in os.listdir(TARGET) if f.endswith(".whl"))


def installed() -> bool:
    return any(os.path.basename(w).startswith("flocksim-") for w in wheels())


def build(force: bool = False) -> str | None:
    """Build the reference wheels into oracle/_ref; returns the target, or
    None when /root/reference is absent (on the GPU box the prebuilt wheels
    are used)."""
    if not os.path.isdir(REF_PKG):
        return TARGET if installed() else None
    if installed() and not force:
        return TARGET
    with tempfile.TemporaryDirectory() as tmp:
        src = os.path.join(tmp, "pkg")
        shutil.copytree(REF_PKG, src, ignore=shutil.ignore_patterns("__pycache__", "*.egg-info",
                                                                     "build"))
        stage = os.path.join(tmp, "wheels")
        cmd = [sys.executable, "-m", "pip", "wheel", "--no-index", "--no-build-isolation",
               "--no-deps", "--quiet", "--wheel-dir", stage, src, os.path.join(src, "bindings")]
        res = subprocess.run(cmd, capture_output=True, text=True, cwd=tmp)
        if res.returncode != 0:
            raise RuntimeError(f"reference build failed:\n{res.stdout}\n{res.stderr}")
        if os.path.isdir(TARGET):
            shutil.rmtree(TARGET)
        shutil.move(stage, TARGET)
    with open(STAMP, "w") as f:
        f.write(f"{REF_PKG} via pip wheel --no-index --no-build-isolation --no-deps\n")
    return TARGET


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
