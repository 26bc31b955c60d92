"""Measured acceleration rho = Jacobi iterations / SRJ iterations (paper
section 4, Fig. 'rho vs P') on the GPU path, Neumann Laplace with a smooth
start, tolerance 1e-10 (the reference stopping rule).

python tools/measured_rho.py [--sizes 64,128,256] [--ps 2,4,6,8,10]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

from paper_1511_04292_b200 import grids as G  # noqa: E402
from paper_1511_04292_b200.schedule import quantize  # noqa: E402
from paper_1511_04292_b200.tables import shipped_table  # noqa: E402
from test_gpu_parity import _neumann, _smooth_init  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="64,128,256")
    ap.add_argument("--ps", default="2,4,6,8,10,12,15")
    a = ap.parse_args()
    tab = shipped_table()
    for n in [int(x) for x in a.sizes.split(",")]:
        t0 = time.perf_counter()
        jac, _ = G.jacobi_solve(_smooth_init(_neumann(n)), 1e-10, max_iters=50_000_000)
        tj = time.perf_counter() - t0
        for p in [int(x) for x in a.ps.split(",")]:
            if (p, n) not in tab:
                continue
            row = tab.get(p, n)
            t0 = time.perf_counter()
            srj, _ = G.srj_solve(_smooth_init(_neumann(n)), quantize(row), 1e-10)
            ts = time.perf_counter() - t0
            print(json.dumps({"N": n, "P": p, "rho_theory": round(float(row.rho), 3),
                              "jacobi_iterations": int(jac.iterations),
                              "srj_iterations": int(srj.iterations),
                              "rho_measured": round(jac.iterations / srj.iterations, 3),
                              "jacobi_s": round(tj, 3), "srj_s": round(ts, 3)}), flush=True)


if __name__ == "__main__":
    main()
