"""Optimal SRJ schedules for untabulated (P, N) -- SURVEY.md 8(f) rank 3.

Host side (mpmath), computed once per schedule; nothing here runs on the
device.  The reference computes schedules with ``srj.optimize.solve``
(``optimize.py:803-879``); this module reaches the same optimum by a
different route.

The optimality criterion is the SRJ paper's (arXiv:1511.04292, section 3;
reference ``optimize.py:1-22``): a P-level schedule (omega_1 > ... > omega_P,
fractions beta_i summing to 1) minimises

    max over kappa in [kappa_min, 2] of  f(kappa) = sum_i beta_i log|1 - omega_i kappa|,

the log of the per-iteration amplification factor Gamma (``core.py:150-190``).
At the optimum f equioscillates: its maxima at kappa_min, at the P-1
interior extrema kappa_1..kappa_{P-1} (one between consecutive poles
1/omega_i) and at kappa = 2 are equal.  The reference eliminates the
fractions and the sensitivities in closed form (``beta_from``,
``domega_dbeta``) and continues in P; here the minimax KKT system is solved
as it stands, with the multipliers as unknowns, and continued in kappa_min
from the nearest tabulated row of the same P:

    unknowns   u_i = log omega_i (P), beta_1..beta_{P-1} (beta_P = 1 - sum),
               v_k = log kappa_k (P-1), multipliers lambda_0..lambda_P, level t
    equations  f(kappa_j) = t                          j = 0..P     (equal ripple)
               kappa_k f'(kappa_k) = 0                 k = 1..P-1   (interior extrema)
               sum_j lambda_j df(kappa_j)/d omega_i / (beta_i/omega_i) = 0   i = 1..P
               sum_j lambda_j df(kappa_j)/d beta_i = 0                       i = 1..P-1
               sum_j lambda_j = 1

(4P equations, 4P unknowns; the interior kappa_j move with the design but
f' = 0 there, so their motion drops out of the stationarity conditions).
Newton with an analytic Jacobian at 40 significant digits and a
backtracking line search that keeps the iterate interleaved.
``tests/test_optimize.py`` pins the results against the reference
optimizer's own output (``tests/golden/optimizer.npz``, made by
``tools/make_golden.py optimizer``) and the shipped full-precision rows.
"""

import math

import mpmath
import numpy as np

from .schedule import WeightSchedule

__all__ = ["OptimizeError", "kappa_min", "optimal_schedule", "solve_kkt"]

KAPPA_MAX = 2
DIGITS = 40


class OptimizeError(RuntimeError):
    """The Newton continuation did not converge."""


def kappa_min(n, d=2, bc="neumann"):
    """Smallest model-problem eigenvalue (restated from ``core.py:229-259``):
    (2/d) sin^2(pi/2n) for Neumann, 2 sin^2(pi/2n) for Dirichlet faces."""
    if not n >= 2:
        raise ValueError(f"n must be >= 2, got {n}")
    if d not in (1, 2, 3):
        raise ValueError(f"d must be 1, 2 or 3, got {d}")
    s2 = math.sin(math.pi / (2.0 * n)) ** 2
    if bc == "neumann":
        return (2.0 / d) * s2
    if bc == "dirichlet":
        return 2.0 * s2
    raise ValueError(f"unknown boundary kind {bc!r}")


# ----------------------------------------------------------------- system
class _System:
    """The KKT system at a fixed kappa_min (mpmath scalars throughout)."""

    def __init__(self, p, km):
        self.p = p
        self.km = mpmath.mpf(km)

    def unpack(self, x):
        p = self.p
        om = [mpmath.exp(x[i]) for i in range(p)]
        be = [x[p + i] for i in range(p - 1)]
        be.append(1 - mpmath.fsum(be))
        ka = [mpmath.exp(x[2 * p - 1 + k]) for k in range(p - 1)]
        lam = [x[3 * p - 2 + j] for j in range(p + 1)]
        t = x[4 * p - 1]
        return om, be, ka, lam, t

    def points(self, ka):
        return [self.km] + list(ka) + [mpmath.mpf(KAPPA_MAX)]

    @staticmethod
    def f(om, be, k):
        return mpmath.fsum(b * mpmath.log(abs(1 - w * k)) for w, b in zip(om, be))

    def residual(self, x):
        p = self.p
        om, be, ka, lam, t = self.unpack(x)
        pts = self.points(ka)
        out = [self.f(om, be, k) - t for k in pts]
        for k in ka:
            out.append(mpmath.fsum(b * w * k / (1 - w * k) for w, b in zip(om, be)))
        for i in range(p):
            w = om[i]
            out.append(mpmath.fsum(l * w * k / (1 - w * k) for l, k in zip(lam, pts)))
        for i in range(p - 1):
            out.append(mpmath.fsum(
                l * (mpmath.log(abs(1 - om[i] * k)) - mpmath.log(abs(1 - om[p - 1] * k)))
                for l, k in zip(lam, pts)))
        out.append(mpmath.fsum(lam) - 1)
        return out

    def feasible(self, x):
        p = self.p
        om, be, ka, lam, _ = self.unpack(x)
        if any(om[i] <= om[i + 1] for i in range(p - 1)):
            return False
        if any(not (0 < b < 1) for b in be) and p > 1:
            return False
        for i, k in enumerate(ka):
            if not (1 / om[i] < k < 1 / om[i + 1]):
                return False
        return self.km < (ka[0] if ka else KAPPA_MAX)

    def jacobian(self, x, f0=None):
        """Analytic Jacobian.  With D = 1 - omega_i kappa_j, R = omega_i kappa_j / D
        and L = log|D|: dL/du_i = dL/dv_j = -R, dR/du_i = dR/dv_j = R / D."""
        p = self.p
        om, be, ka, lam, _ = self.unpack(x)
        pts = self.points(ka)
        npt = p + 1
        dd = [[1 - om[i] * pts[j] for j in range(npt)] for i in range(p)]
        rr = [[om[i] * pts[j] / dd[i][j] for j in range(npt)] for i in range(p)]
        ll = [[mpmath.log(abs(dd[i][j])) for j in range(npt)] for i in range(p)]
        rd = [[rr[i][j] / dd[i][j] for j in range(npt)] for i in range(p)]
        n = 4 * p
        jac = mpmath.matrix(n, n)
        cu, cb, cv, cl, ct = 0, p, 2 * p - 1, 3 * p - 2, 4 * p - 1
        row = 0
        for j in range(npt):  # equal ripple
            for i in range(p):
                jac[row, cu + i] = -be[i] * rr[i][j]
            for m in range(p - 1):
                jac[row, cb + m] = ll[m][j] - ll[p - 1][j]
            if 0 < j < p:
                jac[row, cv + j - 1] = -mpmath.fsum(be[i] * rr[i][j] for i in range(p))
            jac[row, ct] = -1
            row += 1
        for k in range(1, p):  # interior extrema
            for i in range(p):
                jac[row, cu + i] = be[i] * rd[i][k]
            for m in range(p - 1):
                jac[row, cb + m] = rr[m][k] - rr[p - 1][k]
            jac[row, cv + k - 1] = mpmath.fsum(be[i] * rd[i][k] for i in range(p))
            row += 1
        for i in range(p):  # stationarity in omega
            jac[row, cu + i] = mpmath.fsum(lam[j] * rd[i][j] for j in range(npt))
            for k in range(1, p):
                jac[row, cv + k - 1] = lam[k] * rd[i][k]
            for j in range(npt):
                jac[row, cl + j] = rr[i][j]
            row += 1
        for i in range(p - 1):  # stationarity in beta
            jac[row, cu + i] = -mpmath.fsum(lam[j] * rr[i][j] for j in range(npt))
            jac[row, cu + p - 1] = mpmath.fsum(lam[j] * rr[p - 1][j] for j in range(npt))
            for k in range(1, p):
                jac[row, cv + k - 1] = lam[k] * (rr[p - 1][k] - rr[i][k])
            for j in range(npt):
                jac[row, cl + j] = ll[i][j] - ll[p - 1][j]
            row += 1
        for j in range(npt):  # multipliers sum to one
            jac[row, cl + j] = 1
        return jac

    def jacobian_fd(self, x, f0):
        """Finite-difference Jacobian (checks the analytic one in the tests)."""
        n = len(x)
        jac = mpmath.matrix(n, n)
        for c in range(n):
            h = mpmath.mpf(10) ** (-(DIGITS // 2)) * max(1, abs(x[c]))
            xp = list(x)
            xp[c] += h
            fp = self.residual(xp)
            for r in range(n):
                jac[r, c] = (fp[r] - f0[r]) / h
        return jac


def _norm(v):
    return max(abs(e) for e in v)


def _interior_extrema(om, be):
    """Zeros of f' in each interleaving interval (bisection on the slope)."""
    ka = []
    for i in range(len(om) - 1):
        lo, hi = 1 / om[i], 1 / om[i + 1]

        def slope(k):
            return mpmath.fsum(b * w / (1 - w * k) for w, b in zip(om, be))

        a = lo * (1 + mpmath.mpf(10) ** -30)
        b = hi * (1 - mpmath.mpf(10) ** -30)
        sa = slope(a)
        for _ in range(200):
            m = (a + b) / 2
            if sa * slope(m) <= 0:
                b = m
            else:
                a, sa = m, slope(m)
        ka.append((a + b) / 2)
    return ka


def _initial_point(sysm, om, be):
    """Newton start from a schedule: interior extrema by bisection, level from
    the equal-ripple values, multipliers by least squares on the linear
    stationarity equations."""
    p = sysm.p
    om = [mpmath.mpf(w) for w in om]
    be = [mpmath.mpf(b) for b in be]
    s = mpmath.fsum(be)
    be = [b / s for b in be]
    ka = _interior_extrema(om, be)
    pts = sysm.points(ka)
    t = mpmath.fsum(sysm.f(om, be, k) for k in pts) / len(pts)
    rows = []
    for i in range(p):
        w = om[i]
        rows.append(([w * k / (1 - w * k) for k in pts], 0))
    for i in range(p - 1):
        rows.append(([mpmath.log(abs(1 - om[i] * k)) - mpmath.log(abs(1 - om[p - 1] * k))
                      for k in pts], 0))
    rows.append(([mpmath.mpf(1)] * (p + 1), 1))
    a = mpmath.matrix([r for r, _ in rows])
    b = mpmath.matrix([v for _, v in rows])
    lam = mpmath.lu_solve(a.T * a, a.T * b)
    x = [mpmath.log(w) for w in om] + be[:-1] + [mpmath.log(k) for k in ka]
    x += [lam[j] for j in range(p + 1)] + [t]
    return x


def _newton(sysm, x, tol, max_iter=60):
    f0 = sysm.residual(x)
    r0 = _norm(f0)
    for it in range(max_iter):
        if r0 < tol:
            return x, r0, it
        jac = sysm.jacobian(x, f0)
        try:
            dx = mpmath.lu_solve(jac, mpmath.matrix([-e for e in f0]))
        except ZeroDivisionError as exc:
            raise OptimizeError("singular Jacobian") from exc
        alpha = mpmath.mpf(1)
        for _ in range(40):
            xn = [x[i] + alpha * dx[i] for i in range(len(x))]
            if sysm.feasible(xn):
                fn = sysm.residual(xn)
                rn = _norm(fn)
                if rn < r0 or rn < tol:
                    break
            alpha /= 2
        else:
            raise OptimizeError(f"line search failed at residual {float(r0):.3e}")
        x, f0, r0 = xn, fn, rn
    if r0 < tol:
        return x, r0, max_iter
    raise OptimizeError(f"no convergence: residual {float(r0):.3e} after {max_iter} steps")


def solve_kkt(p, km, start, tol=None, steps=None):
    """Optimal P-level schedule at kappa_min = km, continued from ``start``.

    ``start``: (omegas, betas) of a nearby optimal schedule (any kappa_min);
    kappa_min is moved geometrically from the start's own optimum to ``km``
    (the first Newton solve happens at the start's kappa_min estimate),
    halving the step whenever Newton fails.

    Returns (omegas, betas, info) as mpmath numbers.
    """
    with mpmath.workdps(DIGITS):
        tol = mpmath.mpf(10) ** -(DIGITS - 12) if tol is None else mpmath.mpf(tol)
        om0 = [mpmath.mpf(w) for w in start[0]]
        be0 = [mpmath.mpf(b) for b in start[1]]
        if p == 1:
            w = 2 / (2 + mpmath.mpf(km))
            return [w], [mpmath.mpf(1)], {"newton_iterations": 0, "residual": 0.0,
                                          "continuation_steps": 0}
        # kappa_min the start schedule is optimal for: the equal-ripple
        # point left of 1/omega_1, i.e. f(kappa) = f(2) with kappa < 1/omega_1
        f2 = _System.f(om0, [b / mpmath.fsum(be0) for b in be0], mpmath.mpf(KAPPA_MAX))
        ks = mpmath.findroot(
            lambda k: _System.f(om0, [b / mpmath.fsum(be0) for b in be0], k) - f2,
            (mpmath.mpf(10) ** -30, (1 / om0[0]) * (1 - mpmath.mpf(10) ** -12)),
            solver="anderson")
        ks = mpmath.mpf(ks)
        sysm = _System(p, ks)
        x = _initial_point(sysm, om0, be0)
        x, _, iters = _newton(sysm, x, tol)
        total, nsteps = iters, 0
        target = mpmath.mpf(km)
        cur = ks
        ratio = mpmath.mpf(1.5)
        while cur != target:
            up = target > cur
            nxt = min(cur * ratio, target) if up else max(cur / ratio, target)
            try:
                xt, _, iters = _newton(_System(p, nxt), list(x), tol)
            except OptimizeError:
                ratio = mpmath.sqrt(ratio)
                if ratio < 1 + mpmath.mpf(10) ** -6:
                    raise
                continue
            x, cur, total, nsteps = xt, nxt, total + iters, nsteps + 1
            if steps is not None and nsteps > steps:
                raise OptimizeError("too many continuation steps")
        sysm = _System(p, target)
        x, res, iters = _newton(sysm, x, tol)
        om, be, _, lam, _ = sysm.unpack(x)
        if any(l < 0 for l in lam):
            raise OptimizeError("negative multiplier: not the minimax optimum")
        return om, be, {"newton_iterations": total + iters, "residual": float(res),
                        "continuation_steps": nsteps}


def optimal_schedule(p, n, bc="neumann", d=2, table=None, start=None):
    """WeightSchedule minimising the maximum amplification over
    [kappa_min(n, d, bc), 2] (the reference's ``optimize.solve(p, n, bc, d)``).

    Starts from ``start`` (a WeightSchedule with the same P) or else from the
    shipped table row of the same P whose kappa_min is closest.
    """
    if not 1 <= p <= 15:
        raise ValueError(f"p must be in 1..15, got {p}")
    km = kappa_min(n, d, bc)
    if start is None:
        from .tables import shipped_table

        table = table or shipped_table()
        rows = [s for key, s in _table_rows(table) if key[0] == p]
        if not rows and p > 1:
            raise OptimizeError(f"no tabulated P={p} row to start from")
        if p > 1:
            start = min(rows, key=lambda s: abs(math.log(kappa_min(s.n) / km)))
    if p == 1:
        w = 2.0 / (2.0 + km)
        return WeightSchedule(omegas=[w], betas=[1.0], n=int(n))
    om, be, info = solve_kkt(p, km, (list(start.omegas), list(start.betas)))
    bf = np.array([float(b) for b in be])
    return WeightSchedule(omegas=[float(w) for w in om], betas=bf / bf.sum(), n=int(n))


def _table_rows(table):
    for key in table.keys():
        yield key, table.get(*key)
