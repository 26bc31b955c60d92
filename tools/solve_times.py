"""Time-to-residual of the BASELINE configs on one GPU (development/report tool).

python tools/solve_times.py [--configs cfg1,cfg2,cfg3,cfg5]
Prints one JSON line per (config, stopping rule): steps, cycles, seconds
(wall, including host<->device copies of the srj_solve call), final relative L2.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1511_04292_b200 import grids as G  # noqa: E402
from paper_1511_04292_b200.problems import CONFIGS, config_fields, config_schedule  # noqa: E402
from paper_1511_04292_b200.schedule import quantize  # noqa: E402
from paper_1511_04292_b200.tables import shipped_table  # noqa: E402


def problem(f):
    nd = f["source"].ndim
    return G.GridProblem(spacing=(1.0,) * nd, u=f["u"].copy(), source=f["source"],
                         center=f["center"], lower=f["lower"], upper=f["upper"],
                         bc=((G.FIXED, G.FIXED),) * nd, source_kappa=f.get("kappa"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="cfg1,cfg2,cfg3,cfg5")
    ap.add_argument("--max-cycles", type=int, default=600)
    a = ap.parse_args()
    tab = shipped_table()
    plan = {
        "cfg1": [("update_inf", 1e-10), ("residual_l2", 1e-10)],
        "cfg2": [("residual_l2", 1e-8)],
        "cfg3": [("residual_l2", 1e-8)],
        "cfg5": [("residual_l2", 1e-8)],
    }
    for name in a.configs.split(","):
        cfg = CONFIGS[name]
        cyc = config_schedule(name, tab)
        f = config_fields(name)
        G.srj_solve(problem(f), cyc, 1e-300, max_iters=16)  # warm-up: library, kernel setup
        for rule, tol in plan[name]:
            p = problem(f)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            try:
                hist, _ = G.srj_solve(p, cyc, tol, max_iters=a.max_cycles * cyc.m, stop=rule)
                status = "converged" if hist.converged else "max_iters"
            except G.DivergenceError as e:
                hist, status = e.history, "diverged"
            dt = time.perf_counter() - t0
            r = p.residual_field()
            if f.get("kappa") is None:
                rel = float(np.sqrt(np.sum(r * r)) / np.sqrt(np.sum(f["source"] ** 2)))
            else:
                rel = None
            print(json.dumps({"config": name, "shape": list(f["source"].shape), "P": cfg["p"],
                              "table_N": int(cyc.source_schedule.n), "M": int(cyc.m),
                              "rule": rule, "tol": tol, "status": status,
                              "steps": int(hist.iterations),
                              "cycles": round(hist.iterations / cyc.m, 3), "seconds": round(dt, 3),
                              "final_rel_l2_host": rel,
                              "last_check": (hist.relative_l2[-1].tolist()
                                             if len(hist.relative_l2) else None)}), flush=True)


if __name__ == "__main__":
    main()
