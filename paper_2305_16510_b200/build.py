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


def build(force: bool = False, verbose: bool = False, defines=(), lib: str | None = None) -> str:
    """Compile each translation unit in parallel (-c), then link the .so.
    `defines` / `lib`: a developer variant (-D flags) linked to another path."""
    out_lib = lib or LIB
    if not force and not defines and lib is None and not _stale():
        return LIB
    os.makedirs(OUT_DIR, exist_ok=True)
    obj_dir = os.path.join(OUT_DIR, "obj" if not defines else "obj_variant")
    os.makedirs(obj_dir, exist_ok=True)
    base = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC]
    base += [f"-D{d}" for d in defines]
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
    tmp = out_lib + ".tmp"
    res = subprocess.run([nvcc(), "-shared", "-Xcompiler", "-fPIC", "-Xlinker", "--no-undefined",
                          *objs, "-o", tmp],
                         capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, out_lib)
    return out_lib


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--define", action="append", default=[],
                    help="developer variant: extra -D (requires --lib)")
    ap.add_argument("--lib", default=None, help="output path of a variant library")
    a = ap.parse_args(argv)
    if a.define and not a.lib:
        ap.error("--define needs --lib (the production library is built without variants)")
    print(build(force=a.force, verbose=a.verbose, defines=a.define, lib=a.lib))


if __name__ == "__main__":
    main()
