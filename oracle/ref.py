"""Import the unmodified reference installed by oracle/build_ref.py.

TEST INFRASTRUCTURE: tests/, __graft_entry__.smoke() and bench.py's CPU legs
only.  The reference lives in oracle/_ref/ (git-ignored, travels to the GPU
box); /root/reference itself is never read at run time.
"""

from __future__ import annotations

import importlib
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


class ReferenceUnavailable(ImportError):
    """oracle/_ref is missing (run oracle/build_ref.py in the build container)."""


def _wheels() -> list:
    if not os.path.isdir(REF_DIR):
        return []
    return sorted(os.path.join(REF_DIR, f) for f in os.listdir(REF_DIR) if f.endswith(".whl"))


def available() -> bool:
    return any(os.path.basename(w).startswith("flocksim-") for w in _wheels())


def flocksim(submodule: str | None = None):
    """The reference package (or one of its modules, e.g. 'bench'),
    imported from its wheels in oracle/_ref (zipimport)."""
    if not available():
        raise ReferenceUnavailable(f"{REF_DIR} holds no flocksim wheel "
                                   "(python oracle/build_ref.py)")
    for w in _wheels():
        if w not in sys.path:
            sys.path.insert(0, w)
    mod = importlib.import_module("flocksim" if submodule is None else f"flocksim.{submodule}")
    origin = os.path.realpath(getattr(mod, "__file__", "") or "")
    if not origin.startswith(os.path.realpath(REF_DIR)):
        raise ReferenceUnavailable(f"flocksim resolved to {origin}, not oracle/_ref")
    return mod


def flocksim_rl():
    flocksim()
    return importlib.import_module("flocksim_rl")
