"""Coefficient classes (srj_plan_set_coef_classes, ABI v6) against the oracle.

Per-cell coefficient arrays that are constant along axis 0 and / or along the
last axis (engine.coef_class) are read from their first slice / first element
of each row by the 3D per-cell sweep kernel (srj_sweep3d.cuh, the CLS
instantiation).  The values read are bitwise the per-cell ones, so every field
and (dmax, rmax) must equal the oracle's step-by-step restatement of ``_wj3``
(``/root/reference/pkg/src/srj/grids.py:379-408``) bit for bit, for every
class combination and masks.  The 2D per-cell kernels read every cell (classes
measured no faster there); the 2D cases pin that broadcast-structured inputs
still match ``_wj2`` (``grids.py:351-376``) on the one-sweep and fused paths,
at shapes off the small-grid cluster kernel (more than 512 rows).
"""

import ctypes

import numpy as np
import pytest

import oracle
from helpers import Cycle, problem_from
from paper_1511_04292_b200 import _lib
from paper_1511_04292_b200 import grids as G
from paper_1511_04292_b200.engine import DeviceGrid, coef_class
from paper_1511_04292_b200.problems import grad_shafranov_fields

pytestmark = pytest.mark.gpu


def _array(rng, shape, cls, lo, hi):
    """Random array of class ``cls`` (bit 1: constant along axis 0, bit 2:
    constant along the last axis)."""
    s = list(shape)
    if cls & 1:
        s[0] = 1
    if cls & 2:
        s[-1] = 1
    a = lo + (hi - lo) * rng.random(s)
    return np.ascontiguousarray(np.broadcast_to(a, shape))


def _fields(rng, shape, classes, masked):
    nd = len(shape)
    c = _array(rng, shape, classes[0], 4.0, 5.0)
    lo = tuple(_array(rng, shape, classes[1 + 2 * a], -1.0, -0.5) for a in range(nd))
    hi = tuple(_array(rng, shape, classes[2 + 2 * a], -1.0, -0.5) for a in range(nd))
    return {"u": rng.standard_normal(tuple(n + 2 for n in shape)),
            "source": rng.standard_normal(shape), "center": c, "lower": lo, "upper": hi,
            "mask": (rng.random(shape) > 0.1) if masked else None}


def _check(f, w, steps, fuse, bc=None):
    p = problem_from(f, bc=bc)
    q = problem_from(f, bc=bc)
    hist, _ = G.srj_solve(p, Cycle(w), 1e-300, max_iters=steps, fuse=fuse, chunk=7)
    if bc is None:
        _, _, norms = oracle.run(q, w, 0, steps)
    else:
        obc = tuple(((lo.kind, lo.values), (hi.kind, hi.values)) for lo, hi in bc)
        _, _, norms = oracle.run_bc(q, obc, w, steps)
    assert np.array_equal(p.u, q.u)
    assert np.array_equal(hist.residual_inf, norms[:, 0] / np.abs(w[np.arange(steps) % len(w)]))
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


W = np.array([17.0, 0.6, 0.8, 0.9, 1.0, 0.7])

SHAPES_2D = [(520, 301), (600, 530), (1030, 67), (515, 2)]


@pytest.mark.parametrize("shape", SHAPES_2D)
@pytest.mark.parametrize("fuse", [1, 2])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_classes_2d_bitwise(shape, fuse, seed):
    rng = np.random.default_rng(1000 * seed + shape[0] + shape[1] + fuse)
    classes = [int(x) for x in rng.integers(0, 4, 5)]
    classes[seed % 5] = 3 - seed % 2 * 2  # every seed has at least one classed array
    f = _fields(rng, shape, classes, masked=seed == 1)
    got = [coef_class(a) for a in [f["center"]] + [x for p in zip(f["lower"], f["upper"]) for x in p]]
    assert any(got)
    _check(f, W, 11, fuse)


@pytest.mark.parametrize("shape", [(9, 13, 70), (20, 33, 129), (40, 17, 5), (6, 8, 2)])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_classes_3d_bitwise(shape, seed):
    rng = np.random.default_rng(77 * seed + sum(shape))
    classes = [int(x) for x in rng.integers(0, 4, 7)]
    classes[seed] = 2
    f = _fields(rng, shape, classes, masked=seed == 2)
    _check(f, W, 9, 1)


def test_spherical_structure_3d():
    """The spherical Poisson builder's structure (problems.py:540-556):
    radial / polar profiles broadcast over the grid, first radial layer
    masked out -- every coefficient array classed."""
    import sys, os

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from coef_class_probe import sph3d_fields

    f = sph3d_fields(24)
    classes = [coef_class(a) for a in [f["center"]] + [x for p in zip(f["lower"], f["upper"]) for x in p]]
    assert classes == [2, 2, 2, 3, 3, 3, 3]
    f["u"] = np.random.default_rng(0).standard_normal(f["u"].shape)
    _check(f, np.array([1.5, 0.8, 0.9]), 12, 1)


@pytest.mark.parametrize("test", ["A", "B"])
def test_grad_shafranov_mirror_classes(test):
    """The reference's Grad-Shafranov problem (problems.py:634-717, MIRROR
    theta faces: one sweep per launch through srj_sweep2d_var) at a size past
    the cluster kernel: center row-constant, radial coefficients constant."""
    f = grad_shafranov_fields(test, 0.2, 600)
    bc = ((G.FIXED, G.FIXED), (G.MIRROR, G.MIRROR))
    _check(f, np.array([30.0, 0.9, 0.7, 1.1]), 10, 0, bc=bc)


def test_masked_constant_stencil_3d():
    """A 3D constant stencil under a mask: the per-cell kernel with every
    array classed constant (read once per row)."""
    rng = np.random.default_rng(5)
    shape = (17, 30, 70)
    f = {"u": rng.standard_normal(tuple(n + 2 for n in shape)), "source": rng.standard_normal(shape),
         "center": np.full(shape, 6.0), "lower": (np.full(shape, -1.0),) * 3,
         "upper": (np.full(shape, -1.0),) * 3, "mask": rng.random(shape) > 0.2}
    _check(f, W, 10, 1)


def test_masked_constant_stencil_classes():
    """A 2D constant stencil under a mask (the per-cell kernels, one sweep
    per launch and fused)."""
    rng = np.random.default_rng(4)
    shape = (700, 450)
    f = {"u": rng.standard_normal((702, 452)), "source": rng.standard_normal(shape),
         "center": np.full(shape, 4.0), "lower": (np.full(shape, -1.0),) * 2,
         "upper": (np.full(shape, -1.0),) * 2, "mask": rng.random(shape) > 0.2}
    for fuse in (1, 2):
        _check(f, W, 8, fuse)


def test_set_coef_classes_errors():
    rng = np.random.default_rng(1)
    f = _fields(rng, (520, 40), [0] * 5, False)
    dev = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"])
    lib = _lib.load()
    bad = (ctypes.c_int32 * 7)(0, 4, 0, 0, 0, 0, 0)
    assert lib.srj_plan_set_coef_classes(dev.plan, bad) == _lib.SRJ_EINVAL
    assert lib.srj_plan_set_coef_classes(dev.plan, None) == _lib.SRJ_EINVAL
    assert lib.srj_plan_set_coef_classes(None, bad) == _lib.SRJ_EINVAL
    ok = (ctypes.c_int32 * 7)(0, 0, 0, 0, 0, 0, 0)
    assert lib.srj_plan_set_coef_classes(dev.plan, ok) == _lib.SRJ_OK
    dev.close()
