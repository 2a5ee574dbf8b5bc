"""Build the sm_100a shared library in-tree (travels to the GPU box).

    python -m paper_2305_16510_b200.build [--verbose]

Produces paper_2305_16510_b200/lib/libflocksim_b200.so from csrc/*.cu with
nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(OUT_DIR, "libflocksim_b200.so")
SOURCES = ["fs_kernels.cu", "fs_step_att.cu", "fs_step_vel.cu", "fs_step_mix.cu",
           "fs_step_pos.cu", "fs_world.cu", "fs_scene.cu", "fs_se3.cu"]
HEADERS = ["fs_host.h", "fs_math.cuh", "fs_rng.cuh", "fs_step.cuh", "fs_scene.cuh"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo", "-ftz=true",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "flocksim_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile each translation unit in parallel (-c), then link the .so."""
    if not force and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    obj_dir = os.path.join(OUT_DIR, "obj")
    os.makedirs(obj_dir, exist_ok=True)
    base = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    if verbose:
        base += ["-Xptxas", "-v"]
    procs = []
    objs = []
    for src in SOURCES:
        obj = os.path.join(obj_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        procs.append((src, subprocess.Popen(base + ["-c", os.path.join(CSRC, src), "-o", obj],
                                            stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                            text=True)))
    logs = []
    failed = False
    for src, p in procs:
        out, err = p.communicate()
        logs.append(f"== {src}\n{out}{err}")
        failed |= p.returncode != 0
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(logs))
    if verbose:
        sys.stdout.write("\n".join(logs))
    tmp = LIB + ".tmp"
    res = subprocess.run([nvcc(), "-shared", "-Xcompiler", "-fPIC", "-Xlinker", "--no-undefined",
                          *objs, "-o", tmp],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, LIB)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args(argv)
    print(build(force=a.force, verbose=a.verbose))


if __name__ == "__main__":
    main()
