"""1-D grids on the GPU path (reference ``_wj1`` / ``_gs1``, grids.py:331-348,
:410-424): the line runs as a 1 x n two-dimensional grid (``grids._LineGrid``).
Golden vectors come from the reference itself (tools/make_golden_1d.py); the
comparison is ``np.array_equal`` (every value equal; the lift can only change
the sign of a zero, see ``_LineGrid``)."""

import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from conftest import fields_from, load_golden, post_from, rules_from  # noqa: E402
from helpers import Cycle, problem_from  # noqa: E402

import oracle  # noqa: E402
from paper_1511_04292_b200 import grids as G  # noqa: E402

pytestmark = pytest.mark.gpu

LINE_CASES = ["line_spherical", "line_var_faces", "line_var_periodic", "line_var_fixed",
              "line_const_solve"]


@pytest.mark.parametrize("name", LINE_CASES)
@pytest.mark.parametrize("fuse", [0, 1])
def test_line_solve_vs_reference(name, fuse):
    """srj_solve on 1-D problems == the reference's srj_solve: field with
    ghosts, both histories, iteration count (tolerance runs stop at the
    reference's step, incl. the spherical problem's mask + tie_origin hook)."""
    g = load_golden(name)
    p = problem_from(fields_from(g), bc=rules_from(g), post=post_from(g))
    hist, interior = G.srj_solve(p, Cycle(g["weights"]), float(g["tol"]),
                                 max_iters=int(g["steps"]), fuse=fuse)
    assert hist.iterations == len(g["residual_inf"])
    assert hist.converged == bool(g["converged"])
    assert np.array_equal(p.u, g["u_final"])
    assert interior.shape == g["source"].shape
    assert np.array_equal(hist.residual_inf, g["residual_inf"])
    assert np.array_equal(hist.true_residual_inf, g["true_residual_inf"])


@pytest.mark.parametrize("name", ["gs_line", "sor_line"])
def test_line_gauss_seidel_vs_reference(name):
    g = load_golden(name)
    p = problem_from(fields_from(g), bc=rules_from(g))
    kw = dict(tol=float(g["tol"]), max_iters=int(g["steps"]))
    if bool(g["sor"]):
        hist, _ = G.sor_solve(p, float(g["omega"]), **kw)
    else:
        hist, _ = G.gauss_seidel_solve(p, **kw)
    assert np.array_equal(p.u, g["u_final"])
    assert np.array_equal(hist.residual_inf, g["residual_inf"])
    assert np.array_equal(hist.true_residual_inf, g["true_residual_inf"])


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 1000, 40_000])
def test_line_sizes_vs_oracle(n):
    """Band edges, a single cell, lines longer than one warp's band: 37 steps
    of a P=6 cycle against the C oracle (oracle_wj1)."""
    rng = np.random.default_rng(n)
    f = {"u": rng.standard_normal(n + 2), "source": rng.standard_normal(n),
         "center": rng.uniform(3.0, 5.0, n), "lower": (-rng.uniform(0.5, 1.0, n),),
         "upper": (-rng.uniform(0.5, 1.0, n),), "mask": (rng.random(n) > 0.2) if n > 2 else None}
    w = load_golden("const2d_p6")["weights"]
    p, q = problem_from(f), problem_from(f)
    hist, _ = G.srj_solve(p, Cycle(w), tol=1e-300, max_iters=37)
    done, _, norms = oracle.run(q, w, 0, 37)
    assert done == hist.iterations == 37
    assert np.array_equal(p.u, q.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


def test_line_single_sweep_and_jacobi():
    """weighted_jacobi_sweep (both traversals) and jacobi_solve on a line."""
    g = load_golden("line_var_fixed")
    f = fields_from(g)
    p, q = problem_from(f), problem_from(f)
    dm, rm = G.weighted_jacobi_sweep(p, 0.8, traversal="reverse")
    odm, orm = oracle.step(q, 0.8)
    assert (dm, rm) == (odm, orm) and np.array_equal(p.u, q.u)
    with pytest.raises(ValueError):
        G.weighted_jacobi_sweep(p, 0.8, traversal="sideways")
    hist, _ = G.jacobi_solve(p, 1e-9, max_iters=5000)
    done, status, norms = oracle.run(q, np.ones(1), 0, 5000, tol=1e-9)
    assert hist.iterations == done and hist.converged == (status == 1)
    assert np.array_equal(p.u, q.u)


def test_line_relative_l2_rule():
    """The BASELINE's relative-L2 rule on a line (not in the reference): the
    check after every cycle sees ||s - A u||_2 / ||s||_2 of a numpy evaluation
    to 1e-12, and the solve stops at the first cycle below the tolerance."""
    g = load_golden("line_const_solve")
    f = fields_from(g)
    p = problem_from(f)
    w = g["weights"]
    hist, _ = G.srj_solve(p, Cycle(w), 1e-8, stop="residual_l2")
    assert hist.converged and hist.iterations % len(w) == 0
    q = problem_from(f)
    ref = math.sqrt(float(np.sum(q.source ** 2)))
    rels = []
    for _ in range(hist.iterations // len(w)):
        oracle.run(q, w, 0, len(w))
        r = q.source - (q.center * q.u[1:-1] + q.lower[0] * q.u[:-2] + q.upper[0] * q.u[2:])
        rels.append(math.sqrt(float(np.sum(r * r))) / ref)
    assert np.array_equal(p.u, q.u)
    assert np.allclose(hist.relative_l2[:, 1], rels, rtol=1e-12, atol=0.0)
    assert rels[-1] < 1e-8 and all(x >= 1e-8 for x in rels[:-1])


def test_line_nonlinear_source_vs_oracle():
    """source_kappa on a line: s(u) = kappa * u^5 re-evaluated every sweep
    (DESIGN section 7), against the oracle's 1-D restatement."""
    n = 777
    rng = np.random.default_rng(5)
    one = np.ones(n)
    h = 1.0 / (n + 1)
    f = {"u": np.ones(n + 2), "source": np.zeros(n), "center": 2.0 / h ** 2 * one,
         "lower": (-one / h ** 2,), "upper": (-one / h ** 2,), "mask": None}
    kappa = 2.0 * math.pi * rng.uniform(0.01, 0.1, n)
    w = load_golden("const2d_p6")["weights"]
    p, q = problem_from(f, kappa=kappa), problem_from(f)
    hist, _ = G.srj_solve(p, Cycle(w), tol=1e-300, max_iters=120)
    done, _, norms = oracle.run(q, w, 0, 120, kappa=kappa)
    assert done == hist.iterations == 120
    assert np.array_equal(p.u, q.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])
