"""The BASELINE configs' own schedules at their own sizes, against the oracle.

SURVEY Appendix A: with weights up to 3.5e6 (cfg2, P=6) or 1.56e6 (cfg4,
P=15) a single re-association shows up as a 1e-9..1e-3 relative difference
within a cycle, so short windows on small grids do not prove the long runs.
These tests run the real schedules for long stretches (the first 1,024
sweeps of cfg2 at 4096^2, a full P=15 cycle of cfg4 on 512^2, a full cycle
of cfg5 at 256^3, the first 64 sweeps of cfg3 at 512^3) and compare the GPU
field and both per-step norm histories with the oracle bit for bit
(reference ``_wj2``/``_wj3``, ``grids.py:351-408``; stopping loop
``:602-687``), plus cfg5's relative-L2 solve to 1e-8 on a reduced grid with
the identical iteration count.  The oracle runs multi-threaded (its max norms
are order-free, so threads are bitwise neutral).
"""

import os

import numpy as np
import pytest

import oracle
from helpers import problem_from
from paper_1511_04292_b200 import grids as G
from paper_1511_04292_b200.problems import config_fields, config_schedule

pytestmark = pytest.mark.gpu

THREADS = os.cpu_count() or 8


def _compare(name, shape, steps, fuse=0, cyc=None):
    f = config_fields(name, shape)
    cyc = cyc or config_schedule(name)
    w = cyc.weight_sequence
    p = problem_from(f)
    hist, _ = G.srj_solve(p, cyc, tol=1e-300, max_iters=steps, fuse=fuse)
    q = problem_from(f)
    done, _, norms = oracle.run(q, w, 0, steps, kappa=f.get("kappa"), nthreads=THREADS)
    assert done == steps == hist.iterations
    assert np.array_equal(p.u, q.u), f"{name}: field differs from the oracle"
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])
    assert np.array_equal(hist.residual_inf, norms[:, 0] / np.abs(w[np.arange(steps) % len(w)]))
    return p


def test_cfg2_full_size_first_1024_sweeps():
    """4096^2, P=6 (M=25,530, omega_1 = 3.5e6): sweeps 0..1023 incl. the
    largest weights of the cycle's first phase, T=4 band kernel."""
    _compare("cfg2", None, 1024)


def test_cfg4_p15_full_cycle_on_512():
    """The P=15 N=2048 cycle (M=9,548, omega up to 1.56e6; SURVEY Appendix A's
    most rounding-sensitive case) for one whole cycle on a 512^2 grid of the
    cfg4 recipe."""
    cyc = config_schedule("cfg4")
    assert cyc.m == 9548
    _compare("cfg4", (512, 512), cyc.m, cyc=cyc)


def test_cfg5_full_size_full_cycle():
    """Nonlinear 256^3 (psi^5 source fused in the 3D tile kernel, T=2) for one
    whole cycle of its effective-N schedule (P=8 N=150 row, M=474)."""
    cyc = config_schedule("cfg5")
    assert cyc.m == 474
    _compare("cfg5", None, cyc.m)


def test_cfg3_full_size_first_64_sweeps():
    """512^3 (1.09 GB per field), P=10: the first 64 sweeps, 3D tile kernel."""
    _compare("cfg3", None, 64)


def test_cfg5_relative_l2_solve_iteration_count():
    """cfg5's stopping rule (relative L2 1e-8 of the initial residual, checked
    every M-cycle) on a 128^3 grid of the cfg5 recipe (on 64^3 the N=150 row over-relaxes
    the psi^5 feedback and diverges in both): the same iteration
    count and check values as the oracle's solve, and the same field."""
    cyc = config_schedule("cfg5")
    f = config_fields("cfg5", (128, 128, 128))
    want = problem_from(f)
    steps, status, _, checks = oracle.solve(want, cyc.weight_sequence, 1e-8, max_iters=200 * cyc.m,
                                            rule="residual_l2", kappa=f["kappa"],
                                            nthreads=THREADS)
    assert status == 1
    p = problem_from(f)
    hist, _ = G.srj_solve(p, cyc, 1e-8, max_iters=200 * cyc.m, stop="residual_l2")
    assert hist.converged and hist.iterations == steps
    assert np.array_equal(p.u, want.u)
    np.testing.assert_allclose(hist.relative_l2[:, 1], [c[1] for c in checks], rtol=1e-12)


def test_cfg2_relative_l2_solve_iteration_count_reduced():
    """cfg2's rule (relative L2 1e-8, checked every M-cycle) with cfg2's own
    P=6 N=4096 cycle on a 512^2 grid: identical count and field."""
    cyc = config_schedule("cfg2")
    f = config_fields("cfg2", (512, 512))
    want = problem_from(f)
    steps, status, _, checks = oracle.solve(want, cyc.weight_sequence, 1e-8, max_iters=4 * cyc.m,
                                            rule="residual_l2", nthreads=THREADS)
    p = problem_from(f)
    hist, _ = G.srj_solve(p, cyc, 1e-8, max_iters=4 * cyc.m, stop="residual_l2")
    assert hist.iterations == steps and hist.converged == (status == 1)
    assert np.array_equal(p.u, want.u)
    np.testing.assert_allclose(hist.relative_l2[:, 1], [c[1] for c in checks], rtol=1e-12)


def test_cfg5_schedule_divergence_on_small_grid_same_step():
    """On 64^3 the cfg5 schedule over-relaxes the psi^5 feedback: the GPU
    solve raises DivergenceError at the same step the oracle's overflow guard
    fires (grids.py:618-625), with the same history."""
    cyc = config_schedule("cfg5")
    f = config_fields("cfg5", (64, 64, 64))
    want = problem_from(f)
    steps, status, norms, _ = oracle.solve(want, cyc.weight_sequence, 1e-8, max_iters=200 * cyc.m,
                                           rule="residual_l2", kappa=f["kappa"], nthreads=THREADS)
    assert status == 2
    p = problem_from(f)
    with pytest.raises(G.DivergenceError) as exc:
        G.srj_solve(p, cyc, 1e-8, max_iters=200 * cyc.m, stop="residual_l2")
    assert exc.value.iterations == steps
    assert np.array_equal(exc.value.history.true_residual_inf, norms[:, 1])
