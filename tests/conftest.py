"""pytest configuration: the `gpu` marker and shared fixture loaders."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a CUDA B200 (runs on the GPU box via -m gpu)")


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def fields_from(g):
    """Reference-GridProblem fields stored in a golden fixture."""
    nd = g["source"].ndim
    return {
        "u": g["u0"].copy(),
        "source": g["source"].copy(),
        "center": g["center"].copy(),
        "lower": tuple(g[f"lower{a}"].copy() for a in range(nd)),
        "upper": tuple(g[f"upper{a}"].copy() for a in range(nd)),
        "mask": g["mask"].copy() if "mask" in g else None,
    }


@pytest.fixture
def golden():
    return load_golden
