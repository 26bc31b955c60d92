"""Golden vectors for 1-D grids (reference ``_wj1`` / ``_gs1``, grids.py:331-348,
:410-424), produced by running the REFERENCE here:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tools/make_golden_1d.py

Same fixture format as ``make_golden.bc_fixture`` (tests/conftest.py loaders).
"""

import numpy as np

import make_golden as M
from make_golden import G, quantize, shipped_table


def gs_fixture(name, prob, omega, steps, tol=1e-300):
    arr = {"u0": prob.u.copy(), "source": prob.source.copy(), "center": prob.center.copy(),
           "lower0": prob.lower[0].copy(), "upper0": prob.upper[0].copy()}
    for side in range(2):
        arr[f"bc0{side}"] = np.array(prob.bc[0][side].kind)
    if prob.mask is not None:
        arr["mask"] = prob.mask.copy()
    if omega is None:
        hist, _ = G.gauss_seidel_solve(prob, tol=tol, max_iters=steps)
    else:
        hist, _ = G.sor_solve(prob, omega, tol=tol, max_iters=steps)
    arr.update(omega=np.float64(1.0 if omega is None else omega), sor=np.bool_(omega is not None),
               steps=np.int64(steps), tol=np.float64(tol), u_final=prob.u,
               residual_inf=hist.residual_inf, true_residual_inf=hist.true_residual_inf,
               converged=np.bool_(hist.converged))
    M.save(name, **arr)


def main():
    from srj.problems import spherical_poisson

    table = shipped_table()
    rng = np.random.default_rng(151104292)
    w64 = quantize(table.get(6, 64).schedule).weight_sequence

    # the reference's own 1-D problem: spherically symmetric Poisson with the
    # slaved first cell (mask) and the tie_origin hook, solved to a tolerance
    sp = spherical_poisson(1, 48).problem
    M.bc_fixture("line_spherical", sp, quantize(table.get(6, 64).schedule).weight_sequence,
                 200_000, tol=1e-9, post="tie_origin")

    def rand(n, masked, bc):
        f = M.random_fields(rng, (n,), masked)
        return G.GridProblem(spacing=(1.0,), u=f["u"], source=f["source"], center=f["center"],
                             lower=f["lower"], upper=f["upper"], mask=f["mask"], bc=bc)

    M.bc_fixture("line_var_faces", rand(203, True, ((G.face_dirichlet(0.375), G.MIRROR),)),
                 w64, 160)
    M.bc_fixture("line_var_periodic", rand(130, False, ((G.PERIODIC, G.PERIODIC),)), w64, 160)
    M.bc_fixture("line_var_fixed", rand(61, False, ((G.FIXED, G.FIXED),)), w64, 160)

    # constant stencil: -u'' = f on 150 cells, Dirichlet, P=3 row, to 1e-10
    n = 150
    h = 1.0 / (n + 1)
    x = np.arange(1, n + 1) * h
    f = np.exp(-((x - 0.3) ** 2) / (2 * 0.05 ** 2)) - 0.5 * np.exp(-((x - 0.7) ** 2) / (2 * 0.1 ** 2))
    one = np.ones(n)
    const = G.GridProblem(spacing=(h,), u=np.zeros(n + 2), source=f, center=2.0 / h ** 2 * one,
                          lower=(-one / h ** 2,), upper=(-one / h ** 2,),
                          bc=((G.FIXED, G.FIXED),))
    M.bc_fixture("line_const_solve", const, quantize(table.lookup(3, 150)).weight_sequence,
                 500_000, tol=1e-10)

    gs_fixture("gs_line", rand(97, True, ((G.FIXED, G.FIXED),)), None, 50)
    gs_fixture("sor_line", rand(140, False, ((G.MIRROR, G.FIXED),)), 1.5, 50)


if __name__ == "__main__":
    main()
