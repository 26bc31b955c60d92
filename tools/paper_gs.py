"""The paper's Grad-Shafranov benchmark (PAPER.md Table 'testab') on the GPU.

python tools/paper_gs.py [--n 300] [--tol 1e-12] [--cpu]
For tests A and B at C=0 (and A at C=0.34) runs srj_solve with the P=14 N=300
schedule to the reference stopping rule, reporting iterations and wall time;
--cpu also times the CPU oracle (the reference arithmetic, one thread) on the
same problem.  The paper's numbers (3.4 GHz i7, serial): A C=0 5350 it 8.55 s,
B C=0 3450 it 1.78 s, A C=0.34 49080 it 79.22 s.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1511_04292_b200 import grids as G  # noqa: E402
from paper_1511_04292_b200.problems import grad_shafranov_fields  # noqa: E402
from paper_1511_04292_b200.schedule import quantize  # noqa: E402
from paper_1511_04292_b200.tables import shipped_table  # noqa: E402

PAPER = {("A", 0.0): (5350, 8.55), ("B", 0.0): (3450, 1.78), ("A", 0.34): (49080, 79.22)}


def build(test, c, n):
    f = grad_shafranov_fields(test, c, n)
    return G.GridProblem(spacing=(9.0 / (n - 1), np.pi / n), u=f["u"], source=f["source"],
                         center=f["center"], lower=f["lower"], upper=f["upper"],
                         bc=((G.FIXED, G.FIXED), (G.MIRROR, G.MIRROR)), mask=f["mask"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=300)
    ap.add_argument("--tol", type=float, default=1e-12)
    ap.add_argument("--cpu", action="store_true")
    a = ap.parse_args()
    cyc = quantize(shipped_table().lookup(14, a.n))
    for (test, c), (pit, psec) in PAPER.items():
        p = build(test, c, a.n)
        G.srj_solve(build(test, c, a.n), cyc, a.tol, max_iters=10)  # warm
        t0 = time.perf_counter()
        hist, _ = G.srj_solve(p, cyc, a.tol, max_iters=2_000_000)
        dt = time.perf_counter() - t0
        out = {"test": test, "C": c, "n": a.n, "P": 14, "table_N": int(cyc.source_schedule.n),
               "M": int(cyc.m), "tol": a.tol, "gpu_iterations": int(hist.iterations),
               "gpu_converged": bool(hist.converged), "gpu_seconds": round(dt, 4),
               "paper_iterations": pit, "paper_seconds_i7_serial": psec}
        if a.cpu:
            import oracle

            q = build(test, c, a.n)
            bc = (("fixed", None), ("fixed", None)), (("mirror", None), ("mirror", None))
            t0 = time.perf_counter()
            steps, status, _ = oracle.run_bc(q, bc, cyc.weight_sequence, 2_000_000, tol=a.tol)
            out.update(cpu_oracle_iterations=int(steps), cpu_oracle_seconds=round(
                time.perf_counter() - t0, 3), cpu_cores=1,
                bitwise_equal=bool(np.array_equal(q.u, p.u)))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
