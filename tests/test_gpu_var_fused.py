"""Two fused steps on per-cell coefficient arrays (srj_sweep2d_vtb.cuh, the
default for 2D problems in the reference's own layout) against the oracle.

The reference kernel is ``_wj2`` (``/root/reference/pkg/src/srj/grids.py:351-376``)
applied step by step; the fused kernel must reproduce every step's field and
(dmax, rmax) bit for bit: masks, band edges (60 owned columns per warp band),
strip edges, odd step counts (a final one-step launch) and the nonlinear
source.
"""

import numpy as np
import pytest

import oracle
from helpers import Cycle, problem_from
from paper_1511_04292_b200 import grids as G

pytestmark = pytest.mark.gpu

SHAPES = [(3, 5), (7, 61), (64, 60), (65, 121), (200, 301), (513, 257), (33, 1201)]


def _fields(rng, shape, masked):
    f = {"u": rng.standard_normal(tuple(n + 2 for n in shape)),
         "source": rng.standard_normal(shape),
         "center": 4.0 + rng.random(shape),
         "lower": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(2)),
         "upper": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(2)),
         "mask": (rng.random(shape) > 0.1) if masked else None}
    return f


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("masked", [False, True])
def test_fused_var2d_bitwise(shape, masked):
    rng = np.random.default_rng(shape[0] * 7919 + shape[1] + masked)
    f = _fields(rng, shape, masked)
    w = np.concatenate([[float(rng.uniform(2.0, 30.0))], rng.uniform(0.5, 1.0, 6)])
    steps = 13
    p, q = problem_from(f), problem_from(f)
    hist, _ = G.srj_solve(p, Cycle(w), 1e-300, max_iters=steps, fuse=2, chunk=5)
    _, _, norms = oracle.run(q, w, 0, steps)
    assert np.array_equal(p.u, q.u)
    assert np.array_equal(hist.residual_inf, norms[:, 0] / np.abs(w[np.arange(steps) % len(w)]))
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


@pytest.mark.parametrize("shape", [(40, 70), (300, 130)])
def test_fused_var2d_nonlinear_bitwise(shape):
    rng = np.random.default_rng(sum(shape))
    f = _fields(rng, shape, True)
    f["u"] = 1.0 + 0.01 * rng.standard_normal(f["u"].shape)
    kappa = 0.05 * rng.random(shape)
    w = np.array([3.0, 0.9, 0.7, 1.1])
    steps = 10
    p, q = problem_from(f, kappa=kappa), problem_from(f, kappa=kappa)
    hist, _ = G.srj_solve(p, Cycle(w), 1e-300, max_iters=steps, fuse=2)
    _, _, norms = oracle.run(q, w, 0, steps, kappa=kappa)
    assert np.array_equal(p.u, q.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


def test_fused_var2d_matches_one_step():
    """fuse=2 (srj_sweep2d_vtb) equals fuse=1 (srj_sweep2d_var)."""
    rng = np.random.default_rng(5)
    f = _fields(rng, (301, 257), True)
    w = np.array([25.0, 0.6, 0.8, 0.9, 1.0])
    a, b = problem_from(f), problem_from(f)
    ha, _ = G.srj_solve(a, Cycle(w), 1e-300, max_iters=21, fuse=2)
    hb, _ = G.srj_solve(b, Cycle(w), 1e-300, max_iters=21, fuse=1)
    assert np.array_equal(a.u, b.u)
    assert np.array_equal(ha.residual_inf, hb.residual_inf)
