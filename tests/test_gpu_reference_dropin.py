"""The drop-in contract end to end: the reference's OWN objects through our API.

The unmodified reference package (``pip install --no-deps`` into
``baseline/_ref``) builds the problems with its own
builders (``/root/reference/pkg/src/srj/problems.py``: ``laplace2d_neumann``
:246, ``poisson2d_dirichlet`` :279, ``grad_shafranov`` :634, ``spherical_poisson``
:443 with its ``tie_origin`` post-sweep hook) and the schedule
with its own ``tables.shipped_table().lookup`` + ``schedule.quantize``.  The
same objects go to the reference's ``srj.grids.srj_solve`` (numba, CPU,
``grids.py:642-687``) and to ``paper_1511_04292_b200.srj_solve`` (GPU); the
returned fields, iteration counts and per-step histories must be identical
bit for bit.  Skipped when ``baseline/_ref`` is absent (it is git-ignored and
travels with the working tree).
"""

import copy
import os
import sys

import numpy as np
import pytest

from paper_1511_04292_b200 import grids as G

pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


@pytest.fixture(scope="module")
def ref():
    if not os.path.isdir(os.path.join(REF, "srj")):
        pytest.skip("baseline/_ref (the installed reference) is absent")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/srj_numba_cache")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import srj.grids as rg
    import srj.problems as rp
    import srj.schedule as rs
    import srj.tables as rt

    return rg, rp, rs, rt


def _cases(rp):
    rng = np.random.default_rng(11)
    lap = rp.laplace2d_neumann(48)
    lap.u[...] = rng.standard_normal(lap.u.shape)  # a nonconstant start (zero is the solution)
    return [
        ("laplace2d_neumann(48)", lap, (6, 48), 1e-9),
        ("poisson2d_dirichlet(130, 120)", rp.poisson2d_dirichlet(130, 120).problem, (4, 128), 1e-10),
        ("grad_shafranov(A, 0, 40)", rp.grad_shafranov("A", 0.0, 40), (8, 40), 1e-11),
        ("grad_shafranov(B, 0.34, 40)", rp.grad_shafranov("B", 0.34, 40), (8, 40), 1e-11),
        # post_sweep hook (tie_origin) + MIRROR theta faces; 3D with a periodic phi axis
        ("spherical_poisson(2, 24)", rp.spherical_poisson(2, 24).problem, (6, 32), 1e-10),
        ("spherical_poisson(3, 12)", rp.spherical_poisson(3, 12).problem, (4, 100), 1e-8),
        # the reference's 1-D problem (_wj1): mask + tie_origin on a line
        ("spherical_poisson(1, 96)", rp.spherical_poisson(1, 96).problem, (5, 100), 1e-10),
    ]


def _check(h_gpu, h_ref, ours, problem, name):
    assert h_gpu.iterations == h_ref.iterations, name
    assert h_gpu.converged == h_ref.converged, name
    assert np.array_equal(np.asarray(h_gpu.residual_inf), np.asarray(h_ref.residual_inf)), name
    assert np.array_equal(np.asarray(h_gpu.true_residual_inf),
                          np.asarray(h_ref.true_residual_inf)), name
    assert np.array_equal(ours.u, problem.u), name


def test_unrefreshed_ghosts_fixed_steps(ref):
    """Ghosts that violate the boundary rule at the start: the reference
    sweeps them as given and refreshes only after each sweep
    (``grids.py:557-558``); fixed step counts on grids that take the fused
    band kernel (2D) and the 3D path with periodic faces and a post-sweep hook."""
    rg, rp, rs, rt = ref
    rng = np.random.default_rng(3)
    lap = rp.laplace2d_neumann(700)
    lap.u[...] = rng.standard_normal(lap.u.shape)
    cycle = rs.quantize(rt.shipped_table().lookup(6, 700))
    ours = copy.deepcopy(lap)
    h_ref, _ = rg.srj_solve(lap, cycle, 1e-300, max_iters=37)
    h_gpu, _ = G.srj_solve(ours, cycle, 1e-300, max_iters=37)
    _check(h_gpu, h_ref, ours, lap, "laplace2d_neumann(700), 37 steps")
    sph = rp.spherical_poisson(3, 16).problem  # mirror + periodic faces, tie_origin hook
    sph.u[...] = rng.standard_normal(sph.u.shape)
    cycle = rs.quantize(rt.shipped_table().lookup(4, 100))
    ours = copy.deepcopy(sph)
    h_ref, _ = rg.srj_solve(sph, cycle, 1e-300, max_iters=23)
    h_gpu, _ = G.srj_solve(ours, cycle, 1e-300, max_iters=23)
    _check(h_gpu, h_ref, ours, sph, "spherical_poisson(3, 16), 23 steps")


def test_reference_gauss_seidel_and_sor(ref):
    """``gauss_seidel_solve`` / ``sor_solve`` (``grids.py:697-712``) on the
    reference's objects, unrefreshed ghosts included."""
    rg, rp, rs, rt = ref
    rng = np.random.default_rng(4)
    for name, solver, args in (("gauss_seidel", "gauss_seidel_solve", ()),
                               ("sor 1.6", "sor_solve", (1.6,))):
        lap = rp.laplace2d_neumann(40)
        lap.u[...] = rng.standard_normal(lap.u.shape)
        ours = copy.deepcopy(lap)
        h_ref = getattr(rg, solver)(lap, *args, 1e-300, max_iters=25)[0]
        h_gpu = getattr(G, solver)(ours, *args, 1e-300, max_iters=25)[0]
        _check(h_gpu, h_ref, ours, lap, name)


def test_reference_objects_through_the_gpu_drop_in(ref):
    rg, rp, rs, rt = ref
    for name, problem, (P, N), tol in _cases(rp):
        cycle = rs.quantize(rt.shipped_table().lookup(P, N))
        ours = copy.deepcopy(problem)
        h_ref, _ = rg.srj_solve(problem, cycle, tol, max_iters=200_000)
        h_gpu, _ = G.srj_solve(ours, cycle, tol, max_iters=200_000)
        _check(h_gpu, h_ref, ours, problem, name)


def test_reference_single_sweeps_and_jacobi(ref):
    """``weighted_jacobi_sweep`` (``grids.py:574-599``, both traversals) and
    ``jacobi_solve`` (``:690-694``) on the reference's objects."""
    rg, rp, rs, rt = ref
    rng = np.random.default_rng(8)
    gs = rp.grad_shafranov("B", 0.34, 64)
    gs.u[...] = rng.standard_normal(gs.u.shape)
    ours = copy.deepcopy(gs)
    for k, (om, trav) in enumerate(((1.7, "forward"), (250.0, "reverse"), (0.6, "forward"))):
        r_ref = rg.weighted_jacobi_sweep(gs, om, traversal=trav)
        r_gpu = G.weighted_jacobi_sweep(ours, om, traversal=trav)
        assert r_gpu == r_ref, k
        assert np.array_equal(ours.u, gs.u), k
    lap = rp.laplace2d_neumann(64)
    lap.u[...] = rng.standard_normal(lap.u.shape)
    ours = copy.deepcopy(lap)
    h_ref, _ = rg.jacobi_solve(lap, 1e-4, max_iters=3000)
    h_gpu, _ = G.jacobi_solve(ours, 1e-4, max_iters=3000)
    _check(h_gpu, h_ref, ours, lap, "jacobi_solve laplace2d_neumann(64)")
