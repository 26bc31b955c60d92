"""Schedule generation for untabulated (P, N), on CPU.

Pinned against the reference optimizer's own output
(``tests/golden/optimizer.npz``, ``tools/make_golden.py optimizer`` running
``srj.optimize.solve``) and against the shipped table rows.
"""

import math

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1511_04292_b200.optimize import kappa_min, optimal_schedule
from paper_1511_04292_b200.schedule import quantize, validate_cycle
from paper_1511_04292_b200.tables import shipped_table

FIXTURE = np.load(f"{GOLDEN}/optimizer.npz")
TAGS = sorted({k.rsplit("_", 1)[0] for k in FIXTURE.files})


def _case(tag):
    p, n, d, dirichlet = (int(v) for v in FIXTURE[tag + "_case"])
    return p, n, d, "dirichlet" if dirichlet else "neumann"


@pytest.mark.parametrize("tag", TAGS)
def test_matches_reference_optimizer(tag):
    """Same optimum as srj.optimize.solve (which converges in doubles to
    1e-12 for small P, hence the 1e-9 bar)."""
    p, n, d, bc = _case(tag)
    s = optimal_schedule(p, n, bc=bc, d=d)
    np.testing.assert_allclose(s.omegas, FIXTURE[tag + "_omegas"], rtol=1e-9)
    np.testing.assert_allclose(s.betas, FIXTURE[tag + "_betas"], rtol=1e-9)


def test_full_precision_table_rows_from_a_neighbour_start():
    """The shipped 16-digit ('computed') rows, re-derived from the row of the
    neighbouring N (a real continuation, not a restart at the answer)."""
    table = shipped_table()
    done = 0
    for p, n in table.keys():
        row = table.get(p, n)
        if p < 2 or p > 6 or not _full_precision(p, n):
            continue
        other = [m for (q, m) in table.keys() if q == p and m != n]
        start = table.get(p, min(other, key=lambda m: abs(math.log(m / n))))
        s = optimal_schedule(p, n, start=start)
        np.testing.assert_allclose(s.omegas, row.omegas, rtol=1e-9)
        np.testing.assert_allclose(s.betas, row.betas, rtol=1e-9)
        done += 1
    assert done >= 2


def _full_precision(p, n):
    import json
    import os

    from paper_1511_04292_b200 import tables

    path = os.path.join(os.path.dirname(tables.__file__), "data", "parameter_tables.json")
    with open(path) as fh:
        rows = json.load(fh)["rows"]
    return any(r["p"] == p and r["n"] == n and r["digits"] >= 15 for r in rows)


@pytest.mark.parametrize("p,n", [(6, 32768), (8, 1024), (10, 8192)])
def test_published_six_digit_rows(p, n):
    """Paper-table rows (six significant digits) from another row's start."""
    table = shipped_table()
    other = [m for (q, m) in table.keys() if q == p and m != n]
    start = table.get(p, max(m for m in other if m < n))
    s = optimal_schedule(p, n, start=start)
    row = table.get(p, n)
    np.testing.assert_allclose(s.omegas, row.omegas, rtol=6e-6)
    np.testing.assert_allclose(s.betas, row.betas, rtol=6e-6)


def _worst_log_gamma(s, n):
    km = kappa_min(n)
    grid = km * (2.0 / km) ** np.linspace(0.0, 1.0, 400001)
    return float(np.max(np.sum(s.betas[None, :] * np.log(np.abs(1.0 - np.outer(grid, s.omegas))),
                               axis=1)))


@pytest.mark.parametrize("p,n", [(14, 1024)])
def test_high_p_published_rows_are_not_better(p, n):
    """Some published high-P rows are not the optimum to six digits (P=13
    N=128 is ~1e-4 off and the reference optimizer's answer equals ours,
    optimizer.npz).  The objective decides: our worst-case amplification
    over [kappa_min, 2] is never above the published row's."""
    table = shipped_table()
    other = [m for (q, m) in table.keys() if q == p and m != n]
    start = table.get(p, min(other, key=lambda m: abs(math.log(m / n))))
    s = optimal_schedule(p, n, start=start)
    assert _worst_log_gamma(s, n) <= _worst_log_gamma(table.get(p, n), n) + 1e-15


def test_analytic_jacobian_matches_finite_differences():
    import mpmath

    from paper_1511_04292_b200 import optimize as O

    with mpmath.workdps(O.DIGITS):
        st = shipped_table().get(7, 1024)
        sysm = O._System(7, O.kappa_min(1300))
        x = O._initial_point(sysm, list(st.omegas), list(st.betas))
        ja, jf = sysm.jacobian(x), sysm.jacobian_fd(x, sysm.residual(x))
        worst = max(abs(ja[i, j] - jf[i, j]) / (1 + abs(jf[i, j]))
                    for i in range(ja.rows) for j in range(ja.cols))
    assert worst < 1e-15


def test_optimum_equioscillates_and_bounds_the_band():
    """The defining property: equal maxima of log Gamma at kappa_min, the P-1
    interior extrema and kappa = 2, and nothing higher anywhere in the band."""
    p, n = 7, 3000  # untabulated N
    s = optimal_schedule(p, n)
    km = kappa_min(n)

    def f(k):
        return float(np.sum(s.betas * np.log(np.abs(1.0 - s.omegas * k))))

    level = f(km)
    assert f(2.0) == pytest.approx(level, abs=1e-12)
    for i in range(p - 1):  # interior maximum between consecutive poles
        lo, hi = 1.0 / s.omegas[i], 1.0 / s.omegas[i + 1]
        ks = lo + (hi - lo) * np.linspace(1e-6, 1 - 1e-6, 20001)
        vals = np.sum(s.betas[None, :] * np.log(np.abs(1.0 - np.outer(ks, s.omegas))), axis=1)
        assert vals.max() == pytest.approx(level, abs=1e-9)
    grid = km * (2.0 / km) ** np.linspace(0.0, 1.0, 200001)
    vals = np.sum(s.betas[None, :] * np.log(np.abs(1.0 - np.outer(grid, s.omegas))), axis=1)
    assert vals.max() <= level + 1e-12
    assert level < 0.0


def test_single_level_and_cycle_pipeline():
    one = optimal_schedule(1, 500)
    assert one.omegas[0] == pytest.approx(2.0 / (2.0 + kappa_min(500)), rel=1e-15)
    s = optimal_schedule(5, 777)
    cyc = quantize(s)
    rep = validate_cycle(cyc, (kappa_min(777), 2.0))
    assert rep.passed
    assert cyc.weight_sequence.size == cyc.m


def test_argument_errors():
    with pytest.raises(ValueError):
        optimal_schedule(16, 100)
    with pytest.raises(ValueError):
        kappa_min(1)
    with pytest.raises(ValueError):
        kappa_min(100, bc="robin")
