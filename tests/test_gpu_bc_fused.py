"""Fused multi-sweep launches with MIRROR / FACE_DIRICHLET faces (2D, 3D).

The band kernel relaxes stages 2..T of a launch against the ghost the
reference refreshes after every sweep (grids.py:225-247), computed from the
boundary-adjacent cell inside the stage; the ghost layer itself is refreshed
once per launch.  Each case is compared bit for bit with the oracle's
step-by-step sweep + refresh (``oracle.run_bc``).  Grids are above the
small-grid cluster threshold (2^18 cells) so the band kernel runs; the shapes
put the boundary columns at every lane/cell position of the edge bands and
include grids of one band and of few rows.  3D: the CTA-tile kernel (T=2, 3)
writes each boundary cell's ghost into the next stage's window.
"""

import os

import numpy as np
import pytest

import oracle
from helpers import Cycle, problem_from
from paper_1511_04292_b200 import grids as G

pytestmark = pytest.mark.gpu

W = np.array([7.3, 0.61, 0.93, 0.55, 0.97, 0.72, 0.88, 0.51, 0.99])


def _fields(shape, seed, var=False, masked=False):
    rng = np.random.default_rng(seed)
    nd = len(shape)
    f = {"u": rng.standard_normal(tuple(n + 2 for n in shape)),
         "source": rng.standard_normal(shape), "mask": None}
    if var:
        f["center"] = 2.0 * nd + rng.random(shape)
        f["lower"] = tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd))
        f["upper"] = tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd))
        if masked:
            f["mask"] = rng.random(shape) > 0.1
    else:
        f["center"] = np.full(shape, 2.0 * nd)
        f["lower"] = tuple(np.full(shape, -1.0) for _ in range(nd))
        f["upper"] = tuple(np.full(shape, -1.0) for _ in range(nd))
    return f


def _rule(kind, val):
    return G.face_dirichlet(val) if kind == "face_dirichlet" else G.BoundaryRule(kind)


def _run(shape, bc, fuse, steps, seed, var=False, masked=False):
    f = _fields(shape, seed, var, masked)
    rules = tuple(tuple(_rule(k, v) for k, v in pair) for pair in bc)
    p = problem_from(f, bc=rules)
    q = problem_from(f)
    q.u[...] = p.u  # same refreshed starting ghosts
    hist, _ = G.srj_solve(p, Cycle(W), 1e-300, max_iters=steps, fuse=fuse, chunk=11)
    _, _, norms = oracle.run_bc(q, bc, W, steps)
    assert np.array_equal(p.u, q.u), (shape, bc, fuse)
    metric = norms[:, 0] / np.abs(W[np.arange(steps) % len(W)])
    assert np.array_equal(hist.residual_inf, metric)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


M, F = "mirror", "face_dirichlet"
X = "fixed"


def _vals(n, seed):
    return np.random.default_rng(seed).standard_normal(n)


CASES = [
    # (shape, bc) -- bc per axis: ((lo kind, lo value), (hi kind, hi value))
    ((600, 517), (((M, None), (M, None)), ((M, None), (M, None)))),
    ((533, 601), (((F, 0.75), (F, -1.25)), ((F, 2.0), (F, 0.5)))),
    ((541, 509), (((F, _vals(509, 1)), (M, None)), ((X, None), (F, _vals(541, 2))))),
    ((517, 531), (((X, None), (F, _vals(531, 3))), ((M, None), (X, None)))),
    ((4100, 70), (((M, None), (F, -0.5)), ((F, _vals(4100, 4)), (M, None)))),  # few bands
    ((2900, 100), (((M, None), (M, None)), ((M, None), (F, 1.5)))),
    ((9, 30001), (((M, None), (F, _vals(30001, 5))), ((M, None), (M, None)))),  # few rows
    ((40, 7001), (((F, 0.25), (M, None)), ((F, -3.0), (F, 3.0)))),
]


@pytest.mark.parametrize("fuse", [2, 3, 4])
@pytest.mark.parametrize("case", range(len(CASES)))
def test_fused_mirror_face_dirichlet_constant(case, fuse):
    shape, bc = CASES[case]
    _run(shape, bc, fuse, 13, seed=10 * case + fuse)


@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("case", [0, 2, 4])
def test_fused_mirror_face_dirichlet_per_cell(case, masked):
    shape, bc = CASES[case]
    _run(shape, bc, 3, 10, seed=100 + case, var=True, masked=masked)


def test_default_fuse_neumann_laplace_matches_one_sweep_per_launch():
    """Size-independent property at a production size: the automatic fused
    depth and fuse=1 (one sweep + refresh per launch) agree bit for bit."""
    from paper_1511_04292_b200.problems import laplace_neumann_fields

    f = laplace_neumann_fields(2048)
    rng = np.random.default_rng(7)
    f["u"] = rng.standard_normal(f["u"].shape)
    out = []
    for fuse in (0, 1):
        p = problem_from(dict(f), bc=((G.MIRROR, G.MIRROR),) * 2)
        hist, _ = G.srj_solve(p, Cycle(W), 1e-300, max_iters=45, fuse=fuse)
        out.append((p.u.copy(), hist.residual_inf.copy(), hist.true_residual_inf.copy()))
    for a, b in zip(*out):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SRJ_BC_RANDOM_CASES", "16"))))
def test_random_fused_faces(seed):
    """Random shapes (band-kernel sizes), face kinds, scalar or per-position
    face values, fused depth 2..4 and coefficient mode."""
    rng = np.random.default_rng(500 + seed)
    n0 = int(rng.integers(8, 1200))
    n1 = int(rng.integers(max(8, (1 << 18) // n0 + 1), (1 << 18) // n0 + 900))
    bc = []
    for ax, n_other in ((0, n1), (1, n0)):
        pair = []
        for _ in range(2):
            k = ("fixed", "mirror", "face_dirichlet")[int(rng.integers(0, 3))]
            v = None
            if k == "face_dirichlet":
                v = rng.standard_normal(n_other) if rng.random() < 0.5 else float(rng.standard_normal())
            pair.append((k, v))
        bc.append(tuple(pair))
    if all(k == "fixed" for pair in bc for k, _ in pair):
        bc[1] = (("mirror", None), bc[1][1])
    var = bool(rng.random() < 0.3)
    _run((n0, n1), tuple(bc), int(rng.integers(2, 5)), int(rng.integers(3, 20)), seed=900 + seed,
         var=var, masked=var and bool(rng.random() < 0.5))


CASES_3D = [
    ((37, 30, 70), (((M, None), (M, None)), ((M, None), (M, None)), ((M, None), (M, None)))),
    ((29, 26, 131), (((F, 0.5), (F, _vals((26, 131), 6))), ((M, None), (F, _vals((29, 131), 7))),
                     ((F, _vals((29, 26), 8)), (X, None)))),
    ((45, 13, 66), (((X, None), (M, None)), ((F, -1.0), (X, None)), ((M, None), (F, 2.5)))),
    ((12, 40, 9), (((M, None), (F, 0.25)), ((X, None), (M, None)), ((F, _vals((12, 40), 9)), (M, None)))),
]


@pytest.mark.parametrize("fuse", [2, 3])
@pytest.mark.parametrize("case", range(len(CASES_3D)))
def test_fused_faces_3d(case, fuse):
    shape, bc = CASES_3D[case]
    _run(shape, bc, fuse, 11, seed=300 + 10 * case + fuse)


@pytest.mark.parametrize("seed", range(int(os.environ.get("SRJ_BC_RANDOM_CASES", "16"))))
def test_random_fused_faces_3d(seed):
    """3D: random shapes (tile-edge positions along j and k), face kinds,
    scalar or per-position face values, fused depth 2..3."""
    rng = np.random.default_rng(700 + seed)
    shape = tuple(int(x) for x in (rng.integers(6, 40), rng.integers(3, 40), rng.integers(3, 150)))
    bc = []
    for ax in range(3):
        other = tuple(n for a, n in enumerate(shape) if a != ax)
        pair = []
        for _ in range(2):
            k = ("fixed", "mirror", "face_dirichlet")[int(rng.integers(0, 3))]
            v = None
            if k == "face_dirichlet":
                v = rng.standard_normal(other) if rng.random() < 0.5 else float(rng.standard_normal())
            pair.append((k, v))
        bc.append(tuple(pair))
    if all(k == "fixed" for pair in bc for k, _ in pair):
        bc[2] = (("mirror", None), bc[2][1])
    _run(shape, tuple(bc), int(rng.integers(2, 4)), int(rng.integers(3, 14)), seed=1900 + seed)


@pytest.mark.parametrize("shape", [(270000, 1), (140000, 2), (2, 140000), (1, 270000), (3, 90001)])
def test_fused_faces_degenerate_2d(shape):
    """One or two columns (both column faces on one lane / cell) and one or
    two rows (both row faces in the same slow ticks), above the cluster-path
    size so the band kernel runs, T=4."""
    bc = (((M, None), (F, 0.5)), ((F, -1.5), (M, None)))
    _run(shape, bc, 4, 9, seed=sum(shape))


@pytest.mark.parametrize("shape", [(30, 1, 40), (20, 33, 1), (1, 25, 70), (2, 2, 2)])
def test_fused_faces_degenerate_3d(shape):
    bc = (((M, None), (F, 0.5)), ((F, -1.5), (M, None)), ((M, None), (F, 2.0)))
    _run(shape, bc, 2, 7, seed=sum(shape))


@pytest.mark.parametrize("shape,fuse", [((24, 30, 70), 2), ((600, 520), 4)])
def test_fused_faces_nonlinear_source(shape, fuse):
    """Fused faces with the nonlinear source s = kappa * psi^5 (cfg5 form)."""
    from paper_1511_04292_b200.problems import nonlinear_fields

    f = nonlinear_fields(shape, seed=3)
    nd = len(shape)
    bc = (((M, None), (F, 1.0)),) + (((M, None), (M, None)),) * (nd - 1)
    rules = tuple(tuple(_rule(k, v) for k, v in pair) for pair in bc)
    w = np.array([1.4, 0.7, 0.9, 0.6])

    def make(rules):
        return G.GridProblem(spacing=(1.0,) * nd, u=np.array(f["u"], dtype=float),
                             source=np.zeros(shape), center=f["center"], lower=f["lower"],
                             upper=f["upper"], bc=rules, source_kappa=f["kappa"])

    p = make(rules)
    q = make(((G.FIXED, G.FIXED),) * nd)
    q.u[...] = p.u
    hist, _ = G.srj_solve(p, Cycle(w), 1e-300, max_iters=14, fuse=fuse)
    _, _, norms = oracle.run_bc(q, bc, w, 14, kappa=f["kappa"])
    assert np.array_equal(p.u, q.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])
