"""Pin the CPU oracle against the reference's own outputs (tests/golden).

The fixtures were produced by running the reference package
(/root/reference/pkg/src/srj) with tools/make_golden.py; the oracle must
reproduce them bit for bit, which is what makes it a valid checker for the GPU
path on a machine where the reference is absent.
"""

import numpy as np
import pytest

import oracle
from conftest import fields_from, load_golden
from helpers import problem_from

FIXED_STEP_CASES = ["var2d", "var2d_mask", "var3d", "var3d_mask", "const2d_p6",
                    "const3d_p6"]


@pytest.mark.parametrize("name", FIXED_STEP_CASES)
def test_oracle_reproduces_reference_steps(name):
    g = load_golden(name)
    p = problem_from(fields_from(g))
    w = g["weights"]
    steps = int(g["steps"])
    done, status, norms = oracle.run(p, w, 0, steps)
    assert done == steps and status == 0
    assert np.array_equal(p.u, g["u_final"])
    metric = norms[:, 0] / np.abs(w[np.arange(steps) % len(w)])
    assert np.array_equal(metric, g["residual_inf"])
    assert np.array_equal(norms[:, 1], g["true_residual_inf"])


@pytest.mark.parametrize("name", ["var2d_mask", "var3d", "const2d_p6"])
def test_numpy_restatement_matches_c_oracle(name):
    g = load_golden(name)
    a = problem_from(fields_from(g))
    b = problem_from(fields_from(g))
    for w in g["weights"][:25]:
        assert oracle.step(a, w) == oracle.np_step(b, w)
    assert np.array_equal(a.u, b.u)


def test_oracle_threads_are_bitwise_neutral():
    g = load_golden("var3d_mask")
    a = problem_from(fields_from(g))
    b = problem_from(fields_from(g))
    _, _, na = oracle.run(a, g["weights"], 0, 40, nthreads=1)
    _, _, nb = oracle.run(b, g["weights"], 0, 40, nthreads=4)
    assert np.array_equal(a.u, b.u) and np.array_equal(na, nb)


def test_oracle_reference_stopping_rule():
    g = load_golden("solve2d_p2")
    p = problem_from(fields_from(g))
    steps, status, norms, _ = oracle.solve(p, g["weights"], float(g["tol"]))
    assert status == 1 and bool(g["converged"])
    assert steps == len(g["residual_inf"])
    assert np.array_equal(p.u, g["u_final"])
    metric = norms[:, 0] / np.abs(g["weights"][np.arange(steps) % len(g["weights"])])
    assert np.array_equal(metric, g["residual_inf"])


def test_oracle_divergence_guard():
    g = load_golden("diverge2d")
    p = problem_from(fields_from(g))
    steps, status, norms = oracle.run(p, g["weights"], 0, 100_000, 1e-12)
    assert status == 2
    assert steps == int(g["iterations"])
    metric = norms[:, 0] / np.abs(g["weights"][np.arange(steps) % len(g["weights"])])
    assert np.array_equal(metric, g["residual_inf"])
    assert np.array_equal(norms[:, 1], g["true_residual_inf"])


def test_oracle_five_point_known_answers():
    # test_grids.py:254-264: 5-point average 2.5; (dmax, rmax) = (1.25, 10.0)
    g = load_golden("five_point")
    for omega in (1.0, 0.5):
        p = problem_from(fields_from(g))
        dm, rm = oracle.step(p, omega)
        want = g[f"w{omega}"]
        assert (dm, rm, p.u[1, 1]) == tuple(want)
    assert tuple(g["w1.0"])[2] == 2.5
    assert tuple(g["w0.5"])[:2] == (1.25, 10.0)


def test_oracle_residual_matches_numpy():
    g = load_golden("var2d_mask")
    p = problem_from(fields_from(g))
    ss, mx = oracle.residual(p)
    r = p.residual_field()[p.mask]
    assert mx == np.max(np.abs(r))
    assert ss == pytest.approx(float(np.sum(r * r)), rel=1e-13)


def test_oracle_nonlinear_source_restatement():
    from paper_1511_04292_b200.problems import nonlinear_fields
    from paper_1511_04292_b200.schedule import quantize
    from paper_1511_04292_b200.tables import shipped_table

    f = nonlinear_fields((30, 32, 34), seed=5)
    w = quantize(shipped_table().get(8, 32)).weight_sequence
    a = problem_from(f)
    b = problem_from(f)
    for k in range(30):
        assert oracle.step(a, w[k], kappa=f["kappa"]) == oracle.np_step(b, w[k], kappa=f["kappa"])
    assert np.array_equal(a.u, b.u)
    # the nonlinear residual decreases over a cycle of the P=6 schedule
    r0 = oracle.residual(problem_from(f), kappa=f["kappa"])[0]
    c = problem_from(f)
    oracle.run(c, w, 0, len(w), kappa=f["kappa"])
    assert oracle.residual(c, kappa=f["kappa"])[0] < r0


BC_CASES = ["neumann2d", "periodic2d", "facedir3d", "gs_a", "gs_b", "gs_a_solve",
            "spherical2d", "spherical3d",
            # 1-D grids (_wj1, grids.py:331-348; tools/make_golden_1d.py)
            "line_spherical", "line_var_faces", "line_var_periodic", "line_var_fixed",
            "line_const_solve"]


@pytest.mark.parametrize("name", BC_CASES)
def test_oracle_boundary_rules_match_reference(name):
    from conftest import bc_from, post_from

    g = load_golden(name)
    p = problem_from(fields_from(g))
    steps, status, norms = oracle.run_bc(p, bc_from(g), g["weights"], int(g["steps"]),
                                         tol=float(g["tol"]), post=post_from(g))
    assert steps == len(g["residual_inf"])
    assert status == (1 if bool(g["converged"]) else 0)
    assert np.array_equal(p.u, g["u_final"])
    metric = norms[:, 0] / np.abs(g["weights"][np.arange(steps) % len(g["weights"])])
    assert np.array_equal(metric, g["residual_inf"])
    assert np.array_equal(norms[:, 1], g["true_residual_inf"])


@pytest.mark.parametrize("name,shape,k", [("cfg4", (120, 97), 6), ("cfg3", (22, 18, 30), 3)])
def test_dependency_cone_crops(name, shape, k):
    """The crop construction the full-size GPU tests rely on: after k sweeps
    the window of a cropped sub-problem equals the full grid's; the stale
    ghost ring (k+1 cells out) first reaches the window at sweep k+2."""
    from helpers import crop_window, problem_from
    from paper_1511_04292_b200.problems import config_fields, config_schedule

    f = config_fields(name, shape)
    w = config_schedule(name).weight_sequence
    nd = len(shape)
    lo, hi = [n // 2 - 4 for n in shape], [n // 2 + 4 for n in shape]
    sub, win = crop_window(f, lo, hi, k)
    for steps, same in ((k, True), (k + 1, True), (k + 2, False)):
        p, q = problem_from(f), problem_from(sub)
        oracle.run(p, w, 0, steps)
        oracle.run(q, w, 0, steps)
        a = p.u[tuple(slice(l + 1, h + 1) for l, h in zip(lo, hi))]
        b = q.u[tuple(slice(s.start + 1, s.stop + 1) for s in win)]
        assert np.array_equal(a, b) == same
    assert nd == len(win)


GS_CASES = ["gs_var2d", "sor_var2d", "gs_var3d", "sor_var3d", "gs_const2d_solve", "sor_neumann2d",
            "gs_line", "sor_line"]


@pytest.mark.parametrize("name", GS_CASES)
def test_oracle_gauss_seidel_matches_reference(name):
    """oracle_gs (lexicographic in-place sweeps) reproduces the reference
    gauss_seidel_solve / sor_solve bit for bit (fields, both histories,
    iteration count of the tolerance run)."""
    from conftest import bc_from

    g = load_golden(name)
    p = problem_from(fields_from(g))
    steps, status, norms = oracle.gs_solve(p, float(g["omega"]), int(g["steps"]),
                                           tol=float(g["tol"]), bc=bc_from(g), sor=bool(g["sor"]))
    assert steps == len(g["residual_inf"])
    assert status == (1 if bool(g["converged"]) else 0)
    assert np.array_equal(p.u, g["u_final"])
    assert np.array_equal(norms[:, 0], g["residual_inf"])
    assert np.array_equal(norms[:, 1], g["true_residual_inf"])
