"""Generate tests/golden/*.npz by running the REFERENCE implementation here.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tools/make_golden.py

Every fixture is produced by the reference's own public API
(``srj.grids.srj_solve`` / ``weighted_jacobi_sweep``, ``srj.schedule.quantize``,
``srj.tables.shipped_table``) on seeded inputs, so the oracle (``oracle/``) and
the host-side restatements in ``paper_1511_04292_b200`` can be pinned against
it on a machine where the reference is absent (the GPU box).

It also exports the shipped parameter table (the paper's published SRJ
schedules, ``pkg/src/srj/data/parameter_tables.txt``) into this project's own
JSON format at ``paper_1511_04292_b200/data/parameter_tables.json``.
"""

import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REPO)

import srj.grids as G  # noqa: E402  (reference)
from srj.core import WeightSchedule  # noqa: E402
from srj.schedule import quantize  # noqa: E402
from srj.tables import shipped_table  # noqa: E402

from paper_1511_04292_b200 import problems as P  # noqa: E402  (input generators)


def save(name, **arrays):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def ref_problem(fields):
    """Reference GridProblem from the project-neutral field dict."""
    nd = fields["source"].ndim
    return G.GridProblem(
        spacing=(1.0,) * nd,
        u=fields["u"].copy(),
        source=fields["source"].copy(),
        center=fields["center"].copy(),
        lower=tuple(a.copy() for a in fields["lower"]),
        upper=tuple(a.copy() for a in fields["upper"]),
        bc=((G.FIXED, G.FIXED),) * nd,
        mask=None if fields.get("mask") is None else fields["mask"].copy(),
    )


def pack(prefix, fields):
    out = {}
    nd = fields["source"].ndim
    out[prefix + "u0"] = fields["u"]
    out[prefix + "source"] = fields["source"]
    out[prefix + "center"] = fields["center"]
    for ax in range(nd):
        out[f"{prefix}lower{ax}"] = fields["lower"][ax]
        out[f"{prefix}upper{ax}"] = fields["upper"][ax]
    if fields.get("mask") is not None:
        out[prefix + "mask"] = fields["mask"]
    return out


def random_fields(rng, shape, masked):
    nd = len(shape)
    f = {
        "u": rng.standard_normal(tuple(s + 2 for s in shape)),
        "source": rng.standard_normal(shape),
        "center": rng.uniform(4.0, 8.0, shape),
        "lower": tuple(-rng.uniform(0.5, 1.0, shape) for _ in range(nd)),
        "upper": tuple(-rng.uniform(0.5, 1.0, shape) for _ in range(nd)),
        "mask": (rng.uniform(size=shape) > 0.25) if masked else None,
    }
    return f


def fixed_steps(name, fields, weights, steps):
    """Run the reference srj_solve for exactly `steps` elementary steps."""
    prob = ref_problem(fields)
    from srj.schedule import CycleSchedule  # noqa: F401

    class _Cycle:  # srj_solve reads only weight_sequence (grids.py:676)
        weight_sequence = np.asarray(weights, dtype=float)

    hist, _ = G.srj_solve(prob, _Cycle(), tol=1e-300, max_iters=steps)
    arrays = pack("", fields)
    arrays.update(
        weights=np.asarray(weights, dtype=float),
        steps=np.int64(steps),
        u_final=prob.u,
        residual_inf=hist.residual_inf,
        true_residual_inf=hist.true_residual_inf,
    )
    save(name, **arrays)


def bc_fixture(name, prob, weights, steps, tol=1e-300, post=None):
    """Run the reference srj_solve on a full GridProblem (any bc)."""
    nd = prob.ndim
    arr = {"u0": prob.u.copy(), "source": prob.source.copy(),
           "center": prob.center.copy()}
    for ax in range(nd):
        arr[f"lower{ax}"] = prob.lower[ax].copy()
        arr[f"upper{ax}"] = prob.upper[ax].copy()
        for side in range(2):
            rule = prob.bc[ax][side]
            arr[f"bc{ax}{side}"] = np.array(rule.kind)
            if rule.kind == "face_dirichlet":
                arr[f"bcval{ax}{side}"] = np.asarray(rule.values, dtype=float)
    if prob.mask is not None:
        arr["mask"] = prob.mask.copy()
    if post is not None:  # name of the post_sweep hook the test restates
        arr["post"] = np.array(post)

    class _Cycle:
        weight_sequence = np.asarray(weights, dtype=float)

    hist, _ = G.srj_solve(prob, _Cycle(), tol=tol, max_iters=steps)
    arr.update(weights=np.asarray(weights, dtype=float), steps=np.int64(steps),
               tol=np.float64(tol), u_final=prob.u, residual_inf=hist.residual_inf,
               true_residual_inf=hist.true_residual_inf,
               converged=np.bool_(hist.converged))
    save(name, **arr)


def optimizer_fixtures(cases=((2, 300, "neumann", 2), (3, 90, "dirichlet", 3),
                                 (4, 1000, "neumann", 2), (5, 333, "dirichlet", 2),
                                 (6, 300, "neumann", 2), (6, 4096, "neumann", 2),
                                 (8, 700, "neumann", 2), (10, 512, "neumann", 2),
                                 (12, 3000, "neumann", 2), (13, 128, "neumann", 2))):
    """Optimal schedules from the reference optimizer (optimize.solve,
    optimize.py:803-879) for tabulated and untabulated (P, N)."""
    import time

    from srj import optimize as O

    arr = {}
    for p, n, bc, d in cases:
        t0 = time.time()
        rep = O.solve(p, n, bc=bc, d=d)
        tag = f"p{p}_n{n}_{bc}_d{d}"
        arr[tag + "_omegas"] = np.asarray(rep.schedule.omegas, dtype=float)
        arr[tag + "_betas"] = np.asarray(rep.schedule.betas, dtype=float)
        arr[tag + "_case"] = np.array([p, n, d, 1 if bc == "dirichlet" else 0])
        print(tag, f"{time.time() - t0:.1f}s", flush=True)
        save("optimizer", **arr)  # incremental: keep what finished


def gs_fixtures():
    """Gauss-Seidel / SOR (grids.py:410-476, :697-716): in-place lexicographic
    sweeps, reference ghost refresh after each, fixed-step and tolerance runs."""
    from srj.problems import laplace2d_neumann

    rng = np.random.default_rng(1511)

    def run(name, prob, omega, steps, tol=1e-300):
        nd = prob.ndim
        arr = {"u0": prob.u.copy(), "source": prob.source.copy(), "center": prob.center.copy()}
        for ax in range(nd):
            arr[f"lower{ax}"] = prob.lower[ax].copy()
            arr[f"upper{ax}"] = prob.upper[ax].copy()
            for side in range(2):
                arr[f"bc{ax}{side}"] = np.array(prob.bc[ax][side].kind)
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
        save(name, **arr)

    run("gs_var2d", ref_problem(random_fields(rng, (37, 45), True)), None, 60)
    run("sor_var2d", ref_problem(random_fields(rng, (70, 33), False)), 1.6, 60)
    run("gs_var3d", ref_problem(random_fields(rng, (9, 14, 10), True)), None, 40)
    run("sor_var3d", ref_problem(random_fields(rng, (12, 11, 13), False)), 1.3, 40)
    c2 = P.poisson_fields((40, 52), n_gauss=8, seed=1, noise=False, width=(0.02, 0.1))
    run("gs_const2d_solve", ref_problem(c2), None, 20000, tol=1e-9)
    nm = laplace2d_neumann(24)
    nm.u[1:-1, 1:-1] = np.random.default_rng(3).standard_normal(nm.shape)
    nm.refresh_ghosts()
    run("sor_neumann2d", nm, 1.7, 80)


def spherical_fixtures():
    """Spherical Poisson (problems.py:443-600): mask + mirror/periodic ghosts +
    the tie_origin post_sweep hook (u[1] = u[2], u[0] = u[2])."""
    from srj.problems import spherical_poisson

    w64 = quantize(shipped_table().get(6, 64).schedule).weight_sequence
    bc_fixture("spherical2d", spherical_poisson(2, 16).problem, w64, 300, post="tie_origin")
    bc_fixture("spherical3d", spherical_poisson(3, 10).problem, w64, 300, post="tie_origin")


def main():
    table = shipped_table()
    rng = np.random.default_rng(20151113)

    # ---- table export (product data) --------------------------------------
    rows = []
    for row in table.rows():
        s = row.schedule
        rows.append({
            "p": int(s.p), "n": int(s.n), "rho": float(s.rho),
            "digits": int(row.precision_digits),
            "provenance": row.provenance,
            "omegas": [float(w) for w in s.omegas],
            "betas": [float(b) for b in s.betas],
        })
    data_path = os.path.join(REPO, "paper_1511_04292_b200", "data",
                             "parameter_tables.json")
    with open(data_path, "w") as fh:
        json.dump({"format": "srj-b200-tables/1",
                   "source": "SRJ paper tables P=2..15 (arXiv:1511.04292), "
                             "as shipped with the reference package",
                   "rows": rows}, fh, indent=0)
    print(f"wrote {data_path} ({len(rows)} rows)")

    # ---- schedules the configs use ---------------------------------------
    sched = {}
    for tag, (p, n) in {"cfg1": (2, 256), "cfg2": (6, 4096),
                        "cfg3": (10, 512), "cfg4": (15, 32768),
                        "cfg5": (8, 256), "p6n64": (6, 64),
                        "p10n550": (10, 550), "p6n256": (6, 256)}.items():
        ws = table.lookup(p, n)
        for strat in ("floor", "round", "ceil"):
            try:
                cyc = quantize(ws, strat)
            except Exception as exc:  # degenerate -> record the failure
                sched[f"{tag}_{strat}_error"] = np.array(str(exc))
                continue
            sched[f"{tag}_{strat}_q"] = cyc.q
            sched[f"{tag}_{strat}_seq"] = cyc.weight_sequence
        sched[f"{tag}_pn"] = np.array([p, n, ws.n])
    save("schedules", **sched)

    # ---- known-answer single sweeps (test_grids.py:254-264) --------------
    u = np.zeros((3, 3))
    u[0, 1], u[2, 1], u[1, 0], u[1, 2] = 1.0, 2.0, 3.0, 4.0
    one = np.ones((1, 1))
    five = {"u": u, "source": np.zeros((1, 1)), "center": 4.0 * one,
            "lower": (-one, -one), "upper": (-one, -one), "mask": None}
    res = {}
    for omega in (1.0, 0.5):
        prob = ref_problem(five)
        dm, rm = G.weighted_jacobi_sweep(prob, omega)
        res[f"w{omega}"] = np.array([dm, rm, prob.u[1, 1]])
    save("five_point", **pack("", five), **res)

    # ---- fixed-step parity cases (variable coefficients, FIXED ghosts) ----
    cyc64 = quantize(table.get(6, 64).schedule)
    w64 = cyc64.weight_sequence
    fixed_steps("var2d", random_fields(rng, (37, 45), False), w64, 160)
    fixed_steps("var2d_mask", random_fields(rng, (29, 70), True), w64, 160)
    fixed_steps("var3d", random_fields(rng, (11, 13, 17), False), w64, 120)
    fixed_steps("var3d_mask", random_fields(rng, (9, 14, 10), True), w64, 120)

    # ---- constant-coefficient Dirichlet Poisson (the BASELINE configs' form)
    # 2D: cfg1-style 8-Gaussian source on a reduced grid, P=2 N=100 row.
    c2 = P.poisson_fields((60, 60), n_gauss=8, seed=1, noise=False)
    cyc2 = quantize(table.lookup(2, 100))
    prob = ref_problem(c2)
    hist, _ = G.srj_solve(prob, cyc2, tol=1e-10)
    arr = pack("", c2)
    arr.update(weights=cyc2.weight_sequence, tol=np.float64(1e-10),
               u_final=prob.u, residual_inf=hist.residual_inf,
               true_residual_inf=hist.true_residual_inf,
               converged=np.bool_(hist.converged))
    save("solve2d_p2", **arr)

    # 2D noise + Gaussians, P=6 schedule, fixed prefix (cfg2 form, reduced N)
    c2n = P.poisson_fields((64, 64), n_gauss=8, seed=2, noise=True)
    fixed_steps("const2d_p6", c2n, quantize(table.lookup(6, 64)).weight_sequence,
                400)
    # 3D 16-Gaussian, P=10-style schedule at reduced N (cfg3 form)
    c3 = P.poisson_fields((20, 22, 24), n_gauss=16, seed=3, noise=False,
                          width=(0.02, 0.08))
    fixed_steps("const3d_p6", c3, w64, 300)

    # ---- non-FIXED boundary rules (BoundaryRule, grids.py:73-112) ---------
    from srj.problems import grad_shafranov, laplace2d_neumann

    nm = laplace2d_neumann(24)
    nm.u[1:-1, 1:-1] = np.random.default_rng(3).standard_normal(nm.shape)
    nm.refresh_ghosts()
    bc_fixture("neumann2d", nm, w64, 200)

    f = random_fields(rng, (20, 26), False)
    per = G.GridProblem(spacing=(1.0, 1.0), u=f["u"], source=f["source"],
                        center=f["center"], lower=f["lower"], upper=f["upper"],
                        bc=((G.FIXED, G.FIXED), (G.PERIODIC, G.PERIODIC)))
    bc_fixture("periodic2d", per, w64, 150)

    f = random_fields(rng, (9, 11, 12), True)
    fd = G.GridProblem(
        spacing=(1.0,) * 3, u=f["u"], source=f["source"], center=f["center"],
        lower=f["lower"], upper=f["upper"], mask=f["mask"],
        bc=((G.face_dirichlet(rng.standard_normal((11, 12))), G.MIRROR),
            (G.PERIODIC, G.PERIODIC),
            (G.face_dirichlet(0.75), G.face_dirichlet(rng.standard_normal((9, 11))))))
    bc_fixture("facedir3d", fd, w64, 120)

    spherical_fixtures()
    gs_fixtures()
    bc_fixture("gs_a", grad_shafranov("A", 0.0, 40), w64, 300)
    bc_fixture("gs_b", grad_shafranov("B", 0.0, 48), w64, 300)
    gs_row = table.lookup(14, 300)
    bc_fixture("gs_a_solve", grad_shafranov("A", 0.0, 60),
               quantize(gs_row).weight_sequence,
               200_000, tol=1e-10)

    # builder pins for the restated Grad-Shafranov / Neumann problems
    pins = {}
    for test, c, n in (("A", 0.0, 40), ("A", 0.34, 33), ("B", 0.0, 48)):
        p = grad_shafranov(test, c, n)
        tag = f"gs_{test}_{str(c).replace('.', 'p')}_{n}"
        pins[tag + "_u"] = p.u
        pins[tag + "_center"] = p.center
        pins[tag + "_lower1"] = p.lower[1]
        pins[tag + "_upper1"] = p.upper[1]
        pins[tag + "_lower0"] = p.lower[0]
        if p.mask is not None:
            pins[tag + "_mask"] = p.mask
    save("builders", **pins)

    # ---- divergence (test_grids.py:421-432 on a FIXED-ghost problem) -----
    bad = quantize(WeightSchedule(omegas=[50.0, 0.5], betas=[0.5, 0.5], n=64))
    dv = random_fields(rng, (24, 24), False)
    dv["center"] = np.full((24, 24), 4.0)
    dv["lower"] = (np.full((24, 24), -1.0),) * 2
    dv["upper"] = (np.full((24, 24), -1.0),) * 2
    prob = ref_problem(dv)
    try:
        G.srj_solve(prob, bad, tol=1e-12, max_iters=100_000)
        raise SystemExit("expected DivergenceError")
    except G.DivergenceError as err:
        arr = pack("", dv)
        arr.update(weights=bad.weight_sequence, iterations=np.int64(err.iterations),
                   residual_inf=err.history.residual_inf,
                   true_residual_inf=err.history.true_residual_inf)
        save("diverge2d", **arr)


if __name__ == "__main__":
    if sys.argv[1:] == ["spherical"]:
        spherical_fixtures()
    elif sys.argv[1:] == ["optimizer"]:
        optimizer_fixtures()
    elif sys.argv[1:] == ["gs"]:
        gs_fixtures()
    else:
        main()
