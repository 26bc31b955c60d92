"""Worker of tests/test_gpu_slab_streams.py: emulated slab ranks with ONE
STREAM PER RANK on one GPU, so the edge launches, peer copies and flag-word
waits / writes of different ranks run truly asynchronously (as between the
processes of a multi-GPU run) and only the flag protocol of ``srj_slab_run``
orders them.  No kernel waits on another: the waits are stream memory
operations.  Exits 0 when every case equals the single-grid solve bit for bit.
Run in a subprocess under a timeout, so a protocol deadlock fails the test
instead of hanging the suite."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import problem_from  # noqa: E402

from paper_1511_04292_b200 import grids as G  # noqa: E402
from paper_1511_04292_b200.distributed import EmulatedRanks  # noqa: E402
from paper_1511_04292_b200.grids import layer_sum_squares  # noqa: E402
from paper_1511_04292_b200.problems import config_fields, nonlinear_fields  # noqa: E402
from paper_1511_04292_b200.schedule import quantize  # noqa: E402
from paper_1511_04292_b200.solver import LocalComm, run_solve, source_l2  # noqa: E402
from paper_1511_04292_b200.tables import shipped_table  # noqa: E402


def steps_case(name, f, world, fuse, w, steps, chunks, kappa=None):
    ranks = EmulatedRanks(problem_from(f), world, fuse, concurrent=True)
    try:
        cur, done, norms = 0, 0, []
        for c in chunks:
            end = int(steps * c)
            cur = ranks.run_chunk(cur, w, done, end - done, fuse)
            norms.append(ranks.norms(end - done))
            done = end
        field = ranks.download_owned(cur)
    finally:
        ranks.close()
    norms = np.concatenate(norms)
    p = problem_from(f)
    hist, _ = G.srj_solve(p, type("C", (), {"weight_sequence": w})(), 1e-300, max_iters=steps,
                          fuse=fuse)
    ok = (np.array_equal(field, p.interior)
          and np.array_equal(norms[:, 1], hist.true_residual_inf))
    print(f"{name}: world={world} fuse={fuse} steps={steps} -> {'ok' if ok else 'MISMATCH'}",
          flush=True)
    return ok


def solve_case(stop, world):
    table = shipped_table()
    f = config_fields("cfg1", (120, 97))
    cyc = quantize(table.get(2, 100))
    kw = dict(stop=stop, chunk=200 if stop == "update_inf" else None,
              check_every=77 if stop == "residual_l2" else None)
    tol = 1e-9 if stop == "update_inf" else 1e-7
    p = problem_from(f)
    hist, _ = G.srj_solve(p, cyc, tol, max_iters=60000, fuse=4, **kw)
    ranks = EmulatedRanks(problem_from(f), world, 4, concurrent=True)
    try:
        l2_ref = source_l2(ranks, LocalComm, layer_sum_squares(f["source"]))
        h, conv, div, cur = run_solve(ranks, LocalComm, cyc.weight_sequence, tol, 60000, True,
                                      stop, kw["check_every"], 4, kw["chunk"], l2_ref,
                                      int(np.prod(f["source"].shape)))
        field = ranks.download_owned(cur)
    finally:
        ranks.close()
    ok = (conv and not div and hist.converged
          and np.array_equal(h["residual_inf"], hist.residual_inf)
          and np.array_equal(h["relative_l2"], hist.relative_l2)
          and np.array_equal(field, p.interior))
    print(f"solve {stop}: world={world} iterations={len(h['residual_inf'])} -> "
          f"{'ok' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    table = shipped_table()
    w6 = quantize(table.lookup(6, 4096)).weight_sequence
    w10 = quantize(table.lookup(10, 512)).weight_sequence
    ok = True
    f2 = config_fields("cfg2", (331, 270))
    for world, fuse in ((2, 4), (4, 3), (8, 4), (40, 4), (3, 1)):
        ok &= steps_case("2d", f2, world, fuse, w6, 97, (0.37, 1.0))
    # slabs tall enough that inner launches overlap the neighbours' exchanges
    ok &= steps_case("2d-large", config_fields("cfg2", (2048, 1024)), 4, 4, w6, 400, (0.5, 1.0))
    f3 = config_fields("cfg3", (37, 30, 66))
    for fuse in (1, 2):
        ok &= steps_case("3d", f3, 3, fuse, w10, 40, (0.5, 1.0))
    ok &= steps_case("3d-large", config_fields("cfg3", (96, 64, 128)), 4, 2, w10, 120, (1.0,))
    # per-cell coefficients + masks: the staged exchange over the per-cell
    # kernels (2D one sweep / two fused sweeps, 3D one sweep)
    rng = np.random.default_rng(77)

    def percell(shape, masked):
        nd = len(shape)
        return {"u": rng.standard_normal(tuple(n + 2 for n in shape)),
                "source": rng.standard_normal(shape), "center": 2.0 * nd + rng.random(shape),
                "lower": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd)),
                "upper": tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd)),
                "mask": (rng.random(shape) > 0.15) if masked else None}

    wv = np.concatenate([[9.0], rng.uniform(0.5, 1.0, 6)])
    ok &= steps_case("2d-percell", percell((300, 200), True), 3, 1, wv, 41, (0.4, 1.0))
    ok &= steps_case("2d-percell-fused", percell((260, 330), False), 4, 2, wv, 40, (0.5, 1.0))
    ok &= steps_case("3d-percell", percell((40, 21, 70), True), 3, 1, wv, 23, (1.0,))
    for stop in ("update_inf", "residual_l2"):
        ok &= solve_case(stop, 3)
    print("ALL OK" if ok else "FAILED", flush=True)
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
