"""Shared fixtures; registers the ``gpu`` marker.

``-m "not gpu"`` tests run in the CPU build container: the oracle against the
golden vectors, host-side logic, the C-ABI symbol table, and the multi-process
(gloo) sharding path.  ``-m gpu`` tests are the parity tests proper and call
the CUDA kernels through the C-ABI library.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture
def golden():
    return load_golden
