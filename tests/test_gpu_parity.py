"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden
vectors and the CPU oracle, bitwise.

Bar (BASELINE north_star): per-point relative L-inf error <= 1e-12 after a fixed
number of sweeps and the same iteration count -- met here as exact equality
(the kernels reproduce the reference's operation order).
"""

import ctypes

import numpy as np
import pytest

import oracle
from conftest import fields_from, load_golden
from helpers import Cycle, crop_window, problem_from
from paper_1511_04292_b200 import grids as G
from paper_1511_04292_b200.problems import config_fields, nonlinear_fields
from paper_1511_04292_b200.schedule import quantize
from paper_1511_04292_b200.tables import shipped_table

pytestmark = pytest.mark.gpu

FIXED_STEP_CASES = ["var2d", "var2d_mask", "var3d", "var3d_mask", "const2d_p6",
                    "const3d_p6"]


@pytest.fixture(scope="module")
def table():
    return shipped_table()


def run_steps(problem, weights, steps, fuse=0, chunk=None):
    return G.srj_solve(problem, Cycle(weights), tol=1e-300, max_iters=steps,
                       fuse=fuse, chunk=chunk)


@pytest.mark.parametrize("name", FIXED_STEP_CASES)
@pytest.mark.parametrize("fuse", [1, 2, 3, 4, 8])
def test_golden_fixed_steps_bitwise(name, fuse):
    g = load_golden(name)
    p = problem_from(fields_from(g))
    hist, interior = run_steps(p, g["weights"], int(g["steps"]), fuse=fuse, chunk=64)
    assert np.array_equal(p.u, g["u_final"])
    assert np.array_equal(hist.residual_inf, g["residual_inf"])
    assert np.array_equal(hist.true_residual_inf, g["true_residual_inf"])
    assert not hist.converged and hist.iterations == int(g["steps"])


@pytest.mark.parametrize("fuse", [1, 4])
def test_golden_reference_stopping_rule(fuse):
    g = load_golden("solve2d_p2")
    p = problem_from(fields_from(g))
    hist, _ = G.srj_solve(p, Cycle(g["weights"]), float(g["tol"]), fuse=fuse, chunk=1000)
    assert hist.converged
    assert hist.iterations == len(g["residual_inf"])
    assert np.array_equal(hist.residual_inf, g["residual_inf"])
    assert np.array_equal(hist.true_residual_inf, g["true_residual_inf"])
    assert np.array_equal(p.u, g["u_final"])


def test_golden_divergence():
    g = load_golden("diverge2d")
    p = problem_from(fields_from(g))
    with pytest.raises(G.DivergenceError) as info:
        G.srj_solve(p, Cycle(g["weights"]), 1e-12, max_iters=100_000)
    err = info.value
    assert err.iterations == int(g["iterations"])
    assert err.history.iterations == err.iterations and not err.history.converged
    assert np.array_equal(err.history.residual_inf, g["residual_inf"])


@pytest.mark.parametrize("omega", [1.0, 0.5])
def test_five_point_known_answers(omega):
    g = load_golden("five_point")
    p = problem_from(fields_from(g))
    dm, rm = G.weighted_jacobi_sweep(p, omega)
    assert (dm, rm, p.u[1, 1]) == tuple(g[f"w{omega}"])


def test_exact_solution_is_fixed_point():
    # test_grids.py:266-273 on the GPU path
    n = 10
    f = config_fields("cfg1", (n, n))
    p = problem_from(f)
    a = np.zeros((n * n, n * n))
    idx = np.arange(n * n).reshape(n, n)
    c = float(f["center"][0, 0])
    lo = float(f["lower"][0][0, 0])
    for i in range(n):
        for j in range(n):
            a[idx[i, j], idx[i, j]] = c
            for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                if 0 <= i + di < n and 0 <= j + dj < n:
                    a[idx[i, j], idx[i + di, j + dj]] = lo
    p.interior[...] = np.linalg.solve(a, f["source"].ravel()).reshape(n, n)
    before = p.interior.copy()
    dm, _ = G.weighted_jacobi_sweep(p, 0.7)
    assert dm <= 1e-14 * np.max(np.abs(before)) * c
    assert np.max(np.abs(p.interior - before)) <= 1e-14


def test_zero_problem_converges_in_one_step(table):
    f = config_fields("cfg1", (16, 16))
    f["source"] = np.zeros((16, 16))
    cyc = quantize(table.get(6, 64))
    hist, _ = G.srj_solve(problem_from(f), cyc, tol=1e-12)
    assert hist.converged and hist.iterations == 1


def test_max_iters_exhaustion(table):
    f = config_fields("cfg1", (32, 32))
    hist, _ = G.jacobi_solve(problem_from(f), 1e-300, max_iters=50)
    assert not hist.converged and hist.iterations == 50


# ---------------------------------------------------------------- vs oracle
def oracle_steps(f, w, steps, kappa=None):
    p = problem_from(f)
    done, status, norms = oracle.run(p, w, 0, steps, kappa=kappa, nthreads=8)
    return p, norms


@pytest.mark.parametrize("fuse", [1, 4, 6])
def test_cfg2_form_bitwise_vs_oracle(table, fuse):
    """cfg2 recipe (noise + 8 Gaussians, P=6 N=4096 schedule, omega_1=3.5e6) on a
    reduced 384x400 grid; 1500 steps including the largest weights."""
    f = config_fields("cfg2", (384, 400))
    w = quantize(table.lookup(6, 4096)).weight_sequence
    want, norms = oracle_steps(f, w, 1500)
    p = problem_from(f)
    hist, _ = run_steps(p, w, 1500, fuse=fuse, chunk=500)
    assert np.array_equal(p.u, want.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


def test_cfg1_full_solve_reference_rule(table):
    """cfg1 at full size (256^2, P=2 N=250 row): reference rule to 1e-10 gives the
    identical iteration count and field as the oracle."""
    f = config_fields("cfg1")
    cyc = quantize(table.lookup(2, 256))
    want = problem_from(f)
    steps, status, onorms, _ = oracle.solve(want, cyc.weight_sequence, 1e-10, nthreads=8)
    assert status == 1
    p = problem_from(f)
    hist, _ = G.srj_solve(p, cyc, 1e-10)
    assert hist.converged and hist.iterations == steps
    assert np.array_equal(p.u, want.u)


def test_cfg1_relative_l2_rule(table):
    f = config_fields("cfg1")
    cyc = quantize(table.lookup(2, 256))
    want = problem_from(f)
    steps, status, _, checks = oracle.solve(want, cyc.weight_sequence, 1e-10,
                                            rule="residual_l2", nthreads=8)
    assert status == 1
    p = problem_from(f)
    hist, _ = G.srj_solve(p, cyc, 1e-10, stop="residual_l2")
    assert hist.converged and hist.iterations == steps
    assert np.array_equal(p.u, want.u)
    got = hist.relative_l2
    assert len(got) == len(checks)
    np.testing.assert_allclose(got[:, 1], [c[1] for c in checks], rtol=1e-12)


def test_cfg3_form_3d_bitwise(table):
    f = config_fields("cfg3", (40, 36, 70))
    w = quantize(table.lookup(10, 512)).weight_sequence
    want, norms = oracle_steps(f, w, 400)
    p = problem_from(f)
    hist, _ = run_steps(p, w, 400, chunk=128)
    assert np.array_equal(p.u, want.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


@pytest.mark.parametrize("shape", [(40, 44, 36), (64, 130)])
def test_nonlinear_source_bitwise(table, shape):
    f = nonlinear_fields(shape, seed=5)
    w = quantize(table.lookup(8, 32)).weight_sequence
    want, norms = oracle_steps(f, w, 2 * len(w), kappa=f["kappa"])
    p = problem_from(f)
    hist, _ = run_steps(p, w, 2 * len(w), chunk=100)
    assert np.array_equal(p.u, want.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


def test_residual_kernel_vs_oracle(table):
    for f in (config_fields("cfg2", (130, 257)), config_fields("cfg3", (17, 19, 66))):
        p = problem_from(f)
        rng = np.random.default_rng(0)
        p.interior[...] = rng.standard_normal(p.shape)
        from paper_1511_04292_b200.grids import _device_grid

        dev = _device_grid(p)
        ss, mx = dev.residual(0)
        dev.close()
        oss, omx = oracle.residual(p)
        assert mx == omx
        assert ss == pytest.approx(oss, rel=1e-13)


def test_dense_kernel_entry_point():
    """srj_wj_dense: the kernel-level drop-in for _WJ_KERNELS[ndim]."""
    import torch

    from paper_1511_04292_b200 import _lib

    lib = _lib.load()
    for name in ("var2d_mask", "var3d", "line_var_faces"):  # _wj2, _wj3, _wj1
        g = load_golden(name)
        f = fields_from(g)
        nd = f["source"].ndim
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
        u = dev(f["u"])
        un = u.clone()
        arrs = [dev(f["source"]), dev(f["center"])]
        lo = [dev(a) for a in f["lower"]]
        hi = [dev(a) for a in f["upper"]]
        act = dev(f["mask"].astype(np.uint8)) if f["mask"] is not None else None
        norms = torch.zeros(2, dtype=torch.float64, device="cuda")
        n = (ctypes.c_int64 * 3)(*f["source"].shape, *([0] * (3 - nd)))
        lop = (ctypes.c_void_p * nd)(*[a.data_ptr() for a in lo])
        hip = (ctypes.c_void_p * nd)(*[a.data_ptr() for a in hi])
        w = float(g["weights"][3])
        rc = lib.srj_wj_dense(nd, n, u.data_ptr(), un.data_ptr(), arrs[0].data_ptr(),
                              arrs[1].data_ptr(), lop, hip,
                              act.data_ptr() if act is not None else None, w,
                              norms.data_ptr(), None)
        _lib.check(rc)
        torch.cuda.synchronize()
        p = problem_from(f)
        dm, rm = oracle.step(p, w)
        got = un.cpu().numpy()
        assert np.array_equal(got, p.u)
        if nd == 1:  # the dense 1-D kernel is _wj1's own arithmetic: signed zeros included
            assert np.array_equal(np.signbit(got), np.signbit(p.u))
        assert tuple(norms.cpu().numpy()) == (dm, rm)


def test_fusion_depth_invariance_full_size_cfg2(table):
    """Size-independent property at the full cfg2 size (4096^2): every fused depth
    gives the bitwise-identical field and norms as single sweeps."""
    f = config_fields("cfg2")
    w = quantize(table.lookup(6, 4096)).weight_sequence
    ref = problem_from(f)
    h1, _ = run_steps(ref, w, 48, fuse=1)
    for fuse in (4, 8):
        p = problem_from(f)
        h, _ = run_steps(p, w, 48, fuse=fuse)
        assert np.array_equal(p.u, ref.u)
        assert np.array_equal(h.residual_inf, h1.residual_inf)


@pytest.mark.parametrize("c", [67141636.00000001, 4.0 * 4097.0 ** 2, 6.0 * 513.0 ** 2,
                               3.0, 7.123456789, -5.5, 1e-30, 2.0 ** 60 + 12345.0])
def test_reciprocal_division_is_correctly_rounded(c):
    """The constant-stencil kernels divide by c through y = RN(1/c) plus two
    Markstein corrections; it must equal IEEE division bit for bit."""
    import torch

    from paper_1511_04292_b200 import _lib

    lib = _lib.load()
    g = torch.Generator(device="cuda").manual_seed(1234)
    n = 1 << 24
    for lo, hi in ((-60.0, 60.0), (-1000.0, 1000.0), (-1.0, 1.0)):
        mant = torch.rand(n, generator=g, device="cuda", dtype=torch.float64) + 1.0
        expo = torch.randint(int(lo), int(hi), (n,), generator=g, device="cuda")
        sign = torch.where(torch.rand(n, generator=g, device="cuda") < 0.5, -1.0, 1.0)
        a = (sign * torch.ldexp(mant, expo)).to(torch.float64)
        # adversarial mantissas near midpoints of quotients
        a[: n // 4] = torch.nextafter(a[: n // 4] * c, torch.full_like(a[: n // 4], float("inf")))
        a[:8] = torch.tensor([0.0, -0.0, float("inf"), -float("inf"), float("nan"),
                              1e-310, -1e300, 5e-324], dtype=torch.float64)
        out = torch.empty_like(a)
        ref = torch.empty_like(a)
        _lib.check(lib.srj_selftest_div(a.data_ptr(), n, c, out.data_ptr(), ref.data_ptr(), None))
        torch.cuda.synchronize()
        same = (out.view(torch.int64) == ref.view(torch.int64)) | (torch.isnan(out) & torch.isnan(ref))
        assert bool(same.all()), f"{int((~same).sum())} mismatches for c={c}"


# ------------------------------------------------- slab decomposition on 1 GPU
def _emulated_steps(f, world, fuse, w, steps, chunks=(1,)):
    """``world`` ranks on this GPU through the C exchange (srj_slab_run with
    every slab, dependency-ordered on one stream); returns (field, norms)."""
    from paper_1511_04292_b200.distributed import EmulatedRanks

    ranks = EmulatedRanks(problem_from(f), world, fuse)
    try:
        cur, done, norms = 0, 0, []
        bounds = [int(steps * c) for c in chunks]
        for end in bounds:
            cur = ranks.run_chunk(cur, w, done, end - done, fuse)
            norms.append(ranks.norms(end - done))
            done = end
        return ranks.download_owned(cur), np.concatenate(norms)
    finally:
        ranks.close()


@pytest.mark.parametrize("world,fuse", [(2, 4), (4, 3), (3, 1), (40, 4), (7, 2)])
def test_slab_decomposition_bitwise_on_one_gpu(table, world, fuse):
    """k-rank slab solve through the C exchange (edge launches, peer copies
    ordered by flag words, inner launches) == single-GPU solve bit for bit
    (cfg2 recipe); 40 ranks make slabs thinner than two halos (all edge);
    two chunks check the snapshot rotation and the flag epochs across calls."""
    f = config_fields("cfg2", (331, 270))
    w = quantize(table.lookup(6, 4096)).weight_sequence
    field, norms = _emulated_steps(f, world, fuse, w, 97, chunks=(0.37, 1.0))
    p = problem_from(f)
    hist, _ = run_steps(p, w, 97, fuse=fuse)
    assert np.array_equal(field, p.interior)
    assert np.array_equal(norms[:, 1], hist.true_residual_inf)
    assert np.array_equal(norms[:, 0] / np.abs(w[:97]), hist.residual_inf)


@pytest.mark.parametrize("fuse", [1, 2, 3])
def test_slab_decomposition_3d_on_one_gpu(table, fuse):
    f = config_fields("cfg3", (37, 30, 66))
    w = quantize(table.lookup(10, 512)).weight_sequence
    field, norms = _emulated_steps(f, 3, fuse, w, 40, chunks=(0.5, 1.0))
    p = problem_from(f)
    hist, _ = run_steps(p, w, 40, fuse=1)
    assert np.array_equal(field, p.interior)
    assert np.array_equal(norms[:, 1], hist.true_residual_inf)


def test_slab_decomposition_nonlinear_on_one_gpu(table):
    from paper_1511_04292_b200.problems import nonlinear_fields

    f = nonlinear_fields((40, 33, 29), seed=5)
    w = quantize(table.get(8, 32)).weight_sequence
    field, norms = _emulated_steps(f, 4, 2, w, 30)
    q = problem_from(f)
    _, _, onorms = oracle.run(q, w, 0, 30, kappa=f["kappa"], nthreads=8)
    assert np.array_equal(field, q.interior)
    assert np.array_equal(norms[:, 1], onorms[:, 1])


@pytest.mark.parametrize("shape,world,fuse,masked", [((300, 200), 3, 1, True),
                                                     ((260, 330), 4, 2, False),
                                                     ((40, 21, 70), 3, 1, True)])
def test_slab_decomposition_per_cell_coefficients(shape, world, fuse, masked):
    """Per-cell coefficients (+ mask) across slabs: the staged exchange around
    the per-cell kernels (2D one sweep, 2D two fused sweeps, 3D one sweep) ==
    the single-grid solve bit for bit."""
    rng = np.random.default_rng(31 + len(shape) + fuse)
    nd = len(shape)
    f = {"u": rng.standard_normal(tuple(n + 2 for n in shape)), "source": rng.standard_normal(shape),
         "center": 2.0 * nd + rng.random(shape),
         "lower": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd)),
         "upper": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd)),
         "mask": (rng.random(shape) > 0.15) if masked else None}
    w = np.concatenate([[9.0], rng.uniform(0.5, 1.0, 6)])
    field, norms = _emulated_steps(f, world, fuse, w, 41, chunks=(0.4, 1.0))
    p = problem_from(f)
    hist, _ = run_steps(p, w, 41, fuse=fuse)
    assert np.array_equal(field, p.interior)
    assert np.array_equal(norms[:, 1], hist.true_residual_inf)


def test_slab_ranks_agree_when_only_one_slab_is_masked(table):
    """A mask inside ONE rank's rows: every rank must take the per-cell kernels
    (and the same fused depth), or the slabs would fuse different numbers of
    sweeps per launch; the result is still the single-grid solve's."""
    f = config_fields("cfg2", (120, 150))
    mask = np.ones((120, 150), dtype=bool)
    mask[100:110, 30:60] = False  # rows of the last of three ranks only
    f = dict(f, mask=mask)
    w = quantize(table.lookup(6, 4096)).weight_sequence
    field, norms = _emulated_steps(f, 3, 0, w, 37, chunks=(0.5, 1.0))
    p = problem_from(f)
    hist, _ = run_steps(p, w, 37)
    assert np.array_equal(field, p.interior)
    assert np.array_equal(norms[:, 1], hist.true_residual_inf)


@pytest.mark.parametrize("stop", ["update_inf", "residual_l2"])
@pytest.mark.parametrize("world", [1, 3])
def test_emulated_rank_solve_matches_srj_solve(table, stop, world):
    """The N-rank stopping logic (solver.run_solve over EmulatedRanks: chunked
    per-step norms, replay to the exact step, per-layer L2 with an exactly
    rounded sum) == grids.srj_solve on one grid: same iteration count,
    histories, L2 check values and field, both rules."""
    from paper_1511_04292_b200.distributed import EmulatedRanks
    from paper_1511_04292_b200.grids import layer_sum_squares
    from paper_1511_04292_b200.solver import LocalComm, run_solve, source_l2

    f = config_fields("cfg1", (120, 97))
    cyc = quantize(table.get(2, 100))
    kw = dict(stop=stop, chunk=200 if stop == "update_inf" else None,
              check_every=77 if stop == "residual_l2" else None)
    tol = 1e-9 if stop == "update_inf" else 1e-7
    p = problem_from(f)
    hist, _ = G.srj_solve(p, cyc, tol, max_iters=60000, fuse=4, **kw)
    assert hist.converged
    ranks = EmulatedRanks(problem_from(f), world, 4)
    try:
        l2_ref = source_l2(ranks, LocalComm, layer_sum_squares(f["source"]))
        h, conv, div, cur = run_solve(ranks, LocalComm, cyc.weight_sequence, tol, 60000, True,
                                      stop, kw["check_every"], 4, kw["chunk"], l2_ref,
                                      int(np.prod(f["source"].shape)))
        field = ranks.download_owned(cur)
    finally:
        ranks.close()
    assert conv and not div
    assert np.array_equal(h["residual_inf"], hist.residual_inf)
    assert np.array_equal(h["true_residual_inf"], hist.true_residual_inf)
    assert np.array_equal(h["relative_l2"], hist.relative_l2)
    assert np.array_equal(field, p.interior)


def test_distributed_srj_solve_single_rank(table):
    """distributed.srj_solve without a process group (world 1): the slab path
    end to end through the public API, == grids.srj_solve."""
    from paper_1511_04292_b200 import distributed as D

    f = config_fields("cfg3", (30, 26, 40))
    cyc = quantize(table.get(6, 32))
    p = problem_from(f)
    hist, _ = G.srj_solve(p, cyc, 1e-8, max_iters=5000, stop="residual_l2", fuse=2)
    q = problem_from(f)
    h2, owned = D.srj_solve(q, cyc, 1e-8, max_iters=5000, stop="residual_l2", fuse=2, gather=True)
    assert hist.iterations == h2.iterations and h2.converged
    assert np.array_equal(hist.relative_l2, h2.relative_l2)
    assert np.array_equal(q.u, p.u)
    assert np.array_equal(owned, p.interior)


def test_slab_grid_single_rank(table):
    """SlabGrid at world size 1 (bench.py at N=1 with --slab): no neighbours,
    no edge rows, same field as the plain solver."""
    from paper_1511_04292_b200.distributed import SlabDecomposition, SlabGrid
    from paper_1511_04292_b200.problems import slab_config_fields

    shape = (300, 257)
    f = config_fields("cfg2", shape)
    w = quantize(table.lookup(6, 4096)).weight_sequence
    g = SlabGrid(slab_config_fields("cfg2", SlabDecomposition(300, 1, 0, 4), shape))
    try:
        cur = g.run(0, w, 0, 41)
        field = g.backend.download_owned(cur)
        norms = g.norms.numpy().reshape(-1, 2)
    finally:
        g.close()
    p = problem_from(f)
    hist, _ = run_steps(p, w, 41, fuse=4)
    assert np.array_equal(field, p.interior)
    assert np.array_equal(norms[:, 1], hist.true_residual_inf)


def test_residual_layers_match_oracle(table):
    """srj_plan_residual_layers: per-layer max|r| exact, sum r^2 to 1e-13
    against the oracle's residual; independent of the split."""
    from paper_1511_04292_b200.engine import DeviceGrid

    for shape in ((70, 333), (9, 40, 77)):
        f = config_fields("cfg2" if len(shape) == 2 else "cfg3", shape)
        p = problem_from(f)
        run_steps(p, quantize(table.get(6, 64)).weight_sequence, 13)
        dev = DeviceGrid(p.u, p.source, p.center, p.lower, p.upper)
        try:
            layers = dev.residual_layers(0)
        finally:
            dev.close()
        r = p.residual_field()
        axes = tuple(range(1, r.ndim))
        assert np.array_equal(layers[:, 1], np.max(np.abs(r), axis=axes))
        np.testing.assert_allclose(layers[:, 0], np.sum(r * r, axis=axes), rtol=1e-13)
        ss, mx = oracle.residual(p)
        import math

        assert math.isclose(math.fsum(layers[:, 0]), ss, rel_tol=1e-13)


# ------------------------------------------- non-FIXED boundary rules on GPU
BC_CASES = ["neumann2d", "periodic2d", "facedir3d", "gs_a", "gs_b", "spherical2d",
            "spherical3d"]


@pytest.mark.parametrize("name", BC_CASES)
def test_boundary_rules_bitwise_vs_reference(name):
    """mirror / periodic / face-Dirichlet (scalar and array) ghosts refreshed on
    the device after every sweep (and the spherical tie_origin post_sweep hook
    as a device gather) == the reference srj_solve bit for bit."""
    from conftest import post_from, rules_from

    g = load_golden(name)
    p = problem_from(fields_from(g), bc=rules_from(g), post=post_from(g))
    hist, _ = run_steps(p, g["weights"], int(g["steps"]), chunk=77)
    assert np.array_equal(p.u, g["u_final"])
    assert np.array_equal(hist.residual_inf, g["residual_inf"])
    assert np.array_equal(hist.true_residual_inf, g["true_residual_inf"])


def test_grad_shafranov_full_solve_vs_reference():
    """The paper's Grad-Shafranov test A (mirror theta ends, variable
    coefficients, P=14 N=300 row) solved to 1e-10 with the reference rule."""
    from conftest import rules_from

    g = load_golden("gs_a_solve")
    p = problem_from(fields_from(g), bc=rules_from(g))
    hist, _ = G.srj_solve(p, Cycle(g["weights"]), float(g["tol"]))
    assert hist.converged and hist.iterations == len(g["residual_inf"])
    assert np.array_equal(p.u, g["u_final"])
    assert np.array_equal(hist.residual_inf, g["residual_inf"])


def test_masked_cells_never_written():
    # test_grids.py:434-443 on the GPU path (Grad-Shafranov test B)
    from conftest import rules_from

    g = load_golden("gs_b")
    p = problem_from(fields_from(g), bc=rules_from(g))
    inert = ~p.mask
    before = p.interior[inert].copy()
    for _ in range(3):
        G.weighted_jacobi_sweep(p, 1.0)
    run_steps(p, np.ones(1), 150)
    assert np.array_equal(p.interior[inert], before)
    assert np.any(p.interior[p.mask] != 0.0)


def test_band_kernels_without_cluster_path():
    """Small fixtures normally take the DSMEM cluster kernel; re-run the parity
    suite with it disabled so the fused band kernels are checked at small
    sizes too (SRJ_SMALL is read once per process, hence the subprocess)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, SRJ_SMALL="0")
    here = os.path.dirname(os.path.abspath(__file__))
    res = subprocess.run(
        [sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x", os.path.join(here, "test_gpu_parity.py"),
         "-k", "not band_kernels_without and not reciprocal and not full_size_windows"],
        env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]


# --------------------------------------------- paper claims on the GPU path
def _neumann(n):
    from paper_1511_04292_b200.problems import laplace_neumann_fields

    f = laplace_neumann_fields(n)
    return G.GridProblem(spacing=(1.0 / n,) * 2, u=f["u"], source=f["source"],
                         center=f["center"], lower=f["lower"], upper=f["upper"],
                         bc=((G.MIRROR, G.MIRROR),) * 2)


def _smooth_init(p, seed=0):
    """Slow cosine modes (test_grids.py:47-66 fixture, restated)."""
    n = p.shape[0]
    xc = (np.arange(n) + 0.5) / n
    rng = np.random.default_rng(seed)
    u = np.zeros(p.shape)
    for k in range(4):
        for m in range(4):
            a = rng.standard_normal()
            if k == 0 and m == 0:
                continue
            u += a * np.outer(np.cos(k * np.pi * xc), np.cos(m * np.pi * xc))
    p.interior[...] = u
    p.refresh_ghosts()
    return p


def test_measured_speedup_tracks_rho(table):
    # test_grids.py:347-356: Laplace N=64 Neumann, P=6, ratio within 25% of rho
    jac, _ = G.jacobi_solve(_smooth_init(_neumann(64)), 1e-10)
    row = table.get(6, 64)
    srj, _ = G.srj_solve(_smooth_init(_neumann(64)), quantize(row), 1e-10)
    assert jac.converged and srj.converged
    assert jac.iterations / srj.iterations == pytest.approx(row.rho, rel=0.25)


def test_jacobi_iterations_scale_with_grid_area():
    # test_grids.py:358-365
    counts = {n: G.jacobi_solve(_smooth_init(_neumann(n)), 1e-10)[0].iterations
              for n in (32, 64)}
    assert 3.4 <= counts[64] / counts[32] <= 4.6


def test_residual_drops_every_cycle(table):
    # test_grids.py:390-404: every shipped P at N=64 contracts over each M-cycle
    sizes = sorted(p for p, n in table.keys() if n == 64)
    assert len(sizes) >= 10
    rng = np.random.default_rng(7)
    for p_levels in sizes:
        cyc = quantize(table.get(p_levels, 64))
        prob = _neumann(64)
        prob.interior[...] = rng.standard_normal(prob.shape)
        prob.refresh_ghosts()
        hist, _ = G.srj_solve(prob, cyc, tol=1e-300, max_iters=2 * cyc.m + 1)
        r = hist.true_residual_inf
        assert r[cyc.m] < r[0], f"P={p_levels}: first cycle did not contract"
        assert r[2 * cyc.m] < r[cyc.m], f"P={p_levels}: second cycle stalled"


def test_cycle_permutation_changes_nothing_after_full_cycles(table):
    # test_grids.py:406-419
    cyc = quantize(table.get(6, 32))
    rolled = np.roll(cyc.weight_sequence, 7)
    steps = 3 * cyc.m
    rng = np.random.default_rng(11)
    init = rng.standard_normal((32, 32))
    a, b = _neumann(32), _neumann(32)
    for p in (a, b):
        p.interior[...] = init
        p.refresh_ghosts()
    G.srj_solve(a, cyc, tol=1e-300, max_iters=steps)
    G.srj_solve(b, Cycle(rolled), tol=1e-300, max_iters=steps)
    scale = max(1.0, np.max(np.abs(a.interior)))
    assert np.max(np.abs(a.interior - b.interior)) <= 1e-8 * scale


# ------------------------------------------------------------ edge shapes
EDGE_2D = [(1, 1), (1, 7), (3, 5), (2, 64), (5, 63), (7, 65), (9, 130), (33, 1), (64, 2),
           (13, 200)]
EDGE_3D = [(1, 1, 1), (2, 3, 4), (3, 1, 70), (5, 17, 1), (9, 20, 65), (18, 3, 129)]


@pytest.mark.parametrize("shape", EDGE_2D + EDGE_3D)
@pytest.mark.parametrize("fuse", [1, 4])
def test_edge_shapes_bitwise(table, shape, fuse):
    """Tiny, ragged and sub-band grids through every kernel path (the cluster
    path by default; the band/tile kernels in the SRJ_SMALL=0 rerun)."""
    rng = np.random.default_rng(len(shape) * 100 + sum(shape))
    f = config_fields("cfg2", shape) if len(shape) == 2 else config_fields("cfg3", shape)
    f["u"] = rng.standard_normal(f["u"].shape)
    w = quantize(table.get(6, 64)).weight_sequence
    want, norms = oracle_steps(f, w, 60)
    p = problem_from(f)
    hist, _ = run_steps(p, w, 60, fuse=fuse, chunk=23)
    assert np.array_equal(p.u, want.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


@pytest.mark.parametrize("shape", [(6, 9), (4, 5, 6)])
def test_edge_shapes_variable_and_masked(shape):
    rng = np.random.default_rng(5)
    nd = len(shape)
    f = {"u": rng.standard_normal(tuple(s + 2 for s in shape)),
         "source": rng.standard_normal(shape), "center": rng.uniform(4, 8, shape),
         "lower": tuple(-rng.uniform(0.5, 1, shape) for _ in range(nd)),
         "upper": tuple(-rng.uniform(0.5, 1, shape) for _ in range(nd)),
         "mask": rng.uniform(size=shape) > 0.3}
    w = np.array([3.0, 0.5, 1.7, 0.9])
    want, norms = oracle_steps(f, w, 40)
    p = problem_from(f)
    hist, _ = run_steps(p, w, 40, chunk=9)
    assert np.array_equal(p.u, want.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


@pytest.mark.parametrize("name,steps,fuse", [("cfg4", 12, 4), ("cfg3", 6, 2)])
def test_full_size_windows_vs_cropped_oracle(name, steps, fuse):
    """BASELINE's largest single-GPU layouts (cfg4 32768^2: 1.08e9 elements
    per buffer; cfg3 512^3): k sweeps of the real schedule at full size,
    windows at the low corner (true boundary), the middle and the far corner
    (largest offsets) bitwise against the oracle on cropped sub-problems."""
    psutil = pytest.importorskip("psutil")
    need = 40e9 if name == "cfg4" else 8e9
    if psutil.virtual_memory().available < need:
        pytest.skip("not enough host memory for the full-size fields")
    from paper_1511_04292_b200.grids import FIXED, GridProblem
    from paper_1511_04292_b200.problems import config_schedule

    f = config_fields(name)
    w = config_schedule(name).weight_sequence
    shape = f["source"].shape
    nd = len(shape)
    ext = 48 if nd == 2 else 12
    wins = [([0] * nd, [ext] * nd),
            ([n // 2 - ext // 2 for n in shape], [n // 2 + ext // 2 for n in shape]),
            ([n - ext for n in shape], list(shape))]
    crops = [crop_window(f, lo, hi, steps) for lo, hi in wins]
    p = GridProblem(spacing=(1.0,) * nd, u=f["u"], source=f["source"], center=f["center"],
                    lower=f["lower"], upper=f["upper"], bc=((FIXED, FIXED),) * nd)
    run_steps(p, w, steps, fuse=fuse)
    for (lo, hi), (sub, win) in zip(wins, crops):
        q = problem_from(sub)
        oracle.run(q, w, 0, steps)
        full = p.u[tuple(slice(l + 1, h + 1) for l, h in zip(lo, hi))]
        assert np.array_equal(full, q.u[tuple(slice(s.start + 1, s.stop + 1) for s in win)]), (lo, hi)


def test_post_sweep_gather_overlapping_vs_oracle(table):
    """A post_sweep hook whose destinations are also sources (staged through
    the plan's temporary) on a masked 3D problem with mirror ghosts."""
    from paper_1511_04292_b200.grids import FIXED, MIRROR

    def chain(uu):
        uu[0] = uu[1]
        uu[1] = uu[2]
        uu[:, 0] = uu[:, 3]

    g = load_golden("var3d_mask")
    f = fields_from(g)
    bc = ((FIXED, FIXED), (MIRROR, MIRROR), (FIXED, FIXED))
    p = problem_from(f, bc=bc, post=chain)
    w = g["weights"]
    hist, _ = run_steps(p, w, 90)
    q = problem_from(f, bc=bc, post=chain)
    spec = tuple(((r.kind, None), (s.kind, None)) for r, s in bc)
    _, _, norms = oracle.run_bc(q, spec, w, 90, post=chain)
    assert np.array_equal(p.u, q.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


def test_capi_run_time_errors():
    """srj_plan_run / srj_plan_set_post_gather argument errors (status codes +
    srj_last_error), on a live plan."""
    from paper_1511_04292_b200 import _lib
    from paper_1511_04292_b200.engine import DeviceGrid

    f = config_fields("cfg2", (40, 70))
    g = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"])
    lib, plan = g.lib, g.plan
    fa, fb, fc = (ctypes.c_void_p(t.data_ptr()) for t in g.fields)
    w = np.array([1.0, 0.5])
    wp = w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    out = ctypes.c_int32(-1)
    norms = ctypes.c_void_p(g.norms.data_ptr())

    def run(src, a, b, m=2, first=0, n=1, fuse=0, nrm=norms):
        return lib.srj_plan_run(plan, src, a, b, wp, m, first, n, fuse, nrm, ctypes.byref(out),
                                g._sp)

    assert run(fa, fa, fb) == _lib.SRJ_EINVAL and b"distinct" in lib.srj_last_error()
    assert run(fa, fb, fc, m=0) == _lib.SRJ_EINVAL
    assert run(fa, fb, fc, first=-1) == _lib.SRJ_EINVAL
    assert run(fa, fb, fc, n=1, fuse=lib.srj_max_fuse() + 1) == _lib.SRJ_EINVAL
    assert run(fa, fb, fc, n=1, nrm=None) == _lib.SRJ_EINVAL
    assert run(fa, fb, fc, n=0) == _lib.SRJ_OK and out.value == 0
    g.ensure_norms(4)
    assert run(fa, fb, fc, n=4, nrm=ctypes.c_void_p(g.norms.data_ptr())) == _lib.SRJ_OK
    assert out.value in (1, 2)
    lay = g.layout
    bad = np.array([int(lay.elems)], dtype=np.int64)
    ok = np.array([5], dtype=np.int64)
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    assert lib.srj_plan_set_post_gather(plan, ptr(bad), ptr(ok), 1) == _lib.SRJ_EINVAL
    dup = np.array([5, 5], dtype=np.int64)
    assert lib.srj_plan_set_post_gather(plan, ptr(dup), ptr(dup), 2) == _lib.SRJ_EINVAL
    assert b"distinct" in lib.srj_last_error()
    assert lib.srj_plan_set_post_gather(plan, None, None, 0) == _lib.SRJ_OK
    g.close()

    # a slab plan (exchanged faces): fused depth limited by its halo, and
    # gathers need the whole grid
    s = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"], halo0=2,
                   own=(2, 38), physical=(False, False))
    s.ensure_norms(4)
    fa, fb, fc = (ctypes.c_void_p(t.data_ptr()) for t in s.fields)
    rc = s.lib.srj_plan_run(s.plan, fa, fb, fc, wp, 2, 0, 4, 3, ctypes.c_void_p(s.norms.data_ptr()),
                            ctypes.byref(out), s._sp)
    assert rc == _lib.SRJ_EINVAL and b"halo0" in s.lib.srj_last_error()
    assert s.lib.srj_plan_set_post_gather(s.plan, ptr(ok), ptr(ok + 1), 1) == _lib.SRJ_EUNSUPPORTED
    s.close()


def test_c_abi_demo_program():
    """examples/srj_c_demo.c drives the C ABI from plain C (no Python, no
    torch): plan API and dense kernel entry point vs a CPU loop, bitwise."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "examples",
                       "bin", "srj_c_demo")
    if not os.path.exists(exe):
        pytest.skip("examples/bin/srj_c_demo not built (run __graft_entry__.build())")
    res = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "OK" in res.stdout and "mismatches 0, dense mismatches 0, norms equal" in res.stdout


@pytest.mark.parametrize("masked", [False, True])
def test_per_cell_coefficients_2d_streaming_kernel(masked):
    """2D per-cell coefficients above the small-grid cluster size run the
    streaming single-sweep kernel (srj_sweep2d_var.cuh): bitwise vs oracle,
    ragged width, mask with inactive cells that must keep their value."""
    rng = np.random.default_rng(7)
    shape = (700, 611)
    f = {"u": rng.standard_normal((702, 613)), "source": rng.standard_normal(shape),
         "center": 4.0 + rng.random(shape),
         "lower": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(2)),
         "upper": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(2)),
         "mask": (rng.random(shape) > 0.1) if masked else None}
    w = np.array([1.6, 0.6, 1.1])
    want, norms = oracle_steps(f, w, 45)
    p = problem_from(f)
    hist, _ = run_steps(p, w, 45, fuse=1, chunk=20)
    assert np.array_equal(p.u, want.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


GS_CASES = ["gs_var2d", "sor_var2d", "gs_var3d", "sor_var3d", "gs_const2d_solve", "sor_neumann2d"]


@pytest.mark.parametrize("name", GS_CASES)
def test_gauss_seidel_wavefront_vs_reference(name):
    """gauss_seidel_solve / sor_solve on the GPU wavefront == the reference's
    sequential in-place sweeps bit for bit (fields incl. ghosts, both norm
    histories, iteration count of the tolerance run)."""
    from conftest import rules_from

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
    assert hist.converged == bool(g["converged"])


@pytest.mark.parametrize("shape,omega,masked", [((700, 611), 1.0, True), ((257, 1030), 1.7, False),
                                                ((40, 44, 36), 1.0, True), ((18, 7, 90), 1.4, False)])
def test_gauss_seidel_wavefront_vs_oracle(shape, omega, masked):
    """Larger grids than the fixtures: many 32-row strips (2D), strips that span
    plane boundaries and planes shorter than a strip (3D)."""
    rng = np.random.default_rng(11)
    nd = len(shape)
    f = {"u": rng.standard_normal(tuple(n + 2 for n in shape)), "source": rng.standard_normal(shape),
         "center": 2.0 * nd + rng.random(shape),
         "lower": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd)),
         "upper": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd)),
         "mask": (rng.random(shape) > 0.1) if masked else None}
    steps = 25
    q = problem_from(f)
    _, _, norms = oracle.gs_solve(q, omega, steps, sor=omega != 1.0)
    p = problem_from(f)
    if omega == 1.0:
        hist, _ = G.gauss_seidel_solve(p, 1e-300, max_iters=steps)
    else:
        hist, _ = G.sor_solve(p, omega, 1e-300, max_iters=steps)
    assert np.array_equal(p.u, q.u)
    assert np.array_equal(hist.residual_inf, norms[:, 0])
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


def test_gauss_seidel_wavefront_short_planes():
    """3-D planes of 2..5 rows: previous-plane neighbours inside the same strip
    are written a few steps before use (read late, not prefetched)."""
    rng = np.random.default_rng(12)
    for shape in ((30, 2, 50), (11, 3, 33), (9, 5, 64)):
        f = {"u": rng.standard_normal(tuple(n + 2 for n in shape)), "source": rng.standard_normal(shape),
             "center": 6.0 + rng.random(shape),
             "lower": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(3)),
             "upper": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(3)), "mask": None}
        q = problem_from(f)
        _, _, norms = oracle.gs_solve(q, 1.0, 15)
        p = problem_from(f)
        hist, _ = G.gauss_seidel_solve(p, 1e-300, max_iters=15)
        assert np.array_equal(p.u, q.u), shape
        assert np.array_equal(hist.true_residual_inf, norms[:, 1]), shape


def _gs_fields(rng, shape, constant):
    nd = len(shape)
    if constant:  # constant stencil: the deep register rings (kPF 14 in 2D, 6 in 3D)
        cen = np.full(shape, 2.0 * nd + 0.37)
        lo = tuple(np.full(shape, -0.9 - 0.01 * a) for a in range(nd))
        hi = tuple(np.full(shape, -0.8 + 0.01 * a) for a in range(nd))
    else:
        cen = 2.0 * nd + rng.random(shape)
        lo = tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd))
        hi = tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd))
    return {"u": rng.standard_normal(tuple(n + 2 for n in shape)),
            "source": rng.standard_normal(shape), "center": cen, "lower": lo, "upper": hi,
            "mask": None}


def _gs_check(f, omega, steps):
    q = problem_from(f)
    _, _, norms = oracle.gs_solve(q, omega, steps, sor=omega != 1.0)
    p = problem_from(f)
    if omega == 1.0:
        hist, _ = G.gauss_seidel_solve(p, 1e-300, max_iters=steps)
    else:
        hist, _ = G.sor_solve(p, omega, 1e-300, max_iters=steps)
    assert np.array_equal(p.u, q.u)
    assert np.array_equal(hist.true_residual_inf, norms[:, 1])


@pytest.mark.parametrize("constant", [False, True])
@pytest.mark.parametrize("nd", [2, 3])
def test_gauss_seidel_wavefront_narrow_rows(nd, constant):
    """Rows of 1..9 columns: each progress wait covers up to kPF+1 prefetched
    steps, so its requirement must stay monotone past the last column (a wait
    skipped there let lane 0 read the previous strip's row early -- random
    seeds 278 and 315 of test_gpu_random at SRJ_RANDOM_CASES=400).  Many short
    strips keep neighbouring strips close in time, where a missing wait shows.
    ``constant`` runs the constant-stencil copies, whose deeper rings look
    ahead up to 2*kPF+1 steps."""
    rng = np.random.default_rng(13 + nd + 7 * constant)
    for ncols in range(1, 10 if nd == 2 else 7):
        shape = (3000, ncols) if nd == 2 else (40, 60, ncols)
        f = _gs_fields(rng, shape, constant)
        for omega in (1.0, 1.3):
            _gs_check(f, omega, 12)


@pytest.mark.parametrize("shape", [(2000, 300), (12, 40, 50), (30, 2, 80)])
def test_gauss_seidel_deep_ring_many_strips(shape):
    """Constant stencils with many strips and short planes on the deep rings."""
    rng = np.random.default_rng(sum(shape))
    _gs_check(_gs_fields(rng, shape, True), 1.0, 9)
    _gs_check(_gs_fields(rng, shape, True), 1.6, 7)


@pytest.mark.parametrize("shape", [(192, 200, 24), (2, 19400, 16)])
def test_gauss_seidel_beyond_deep_ring_occupancy(shape):
    """(i, j) row counts above what the deep constant-stencil ring can hold
    co-resident (148 SMs x 8 warps x 32 rows = 37,888) run on the kPF=4 copy
    instead of raising (e.g. 3-D grids of 38,400 (i, j) rows)."""
    rng = np.random.default_rng(sum(shape))
    _gs_check(_gs_fields(rng, shape, True), 1.0, 3)
