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


def bc_from(g):
    """Boundary spec stored in a golden fixture: per axis ((kind, values), ...)."""
    nd = g["source"].ndim
    out = []
    for ax in range(nd):
        pair = []
        for side in range(2):
            kind = str(g[f"bc{ax}{side}"]) if f"bc{ax}{side}" in g else "fixed"
            vals = g.get(f"bcval{ax}{side}")
            pair.append((kind, vals))
        out.append(tuple(pair))
    return tuple(out)


def rules_from(g):
    """The same spec as this package's BoundaryRule objects."""
    from paper_1511_04292_b200 import grids as G

    out = []
    for pair in bc_from(g):
        rules = []
        for kind, vals in pair:
            rules.append(G.face_dirichlet(vals) if kind == "face_dirichlet"
                         else G.BoundaryRule(kind))
        out.append(tuple(rules))
    return tuple(out)


def tie_origin(uu):
    """The spherical problems' inner-radius tie u_0 = u_1 = u_2 (a
    ``post_sweep`` hook, restated from the reference problems.py:586-589)."""
    uu[1] = uu[2]
    uu[0] = uu[2]


POST_HOOKS = {"tie_origin": tie_origin}


def post_from(g):
    """The post_sweep hook a boundary fixture was generated with, or None."""
    return POST_HOOKS[str(g["post"])] if "post" in g else None
