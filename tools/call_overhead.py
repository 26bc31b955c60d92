"""Fixed host cost of one srj_solve call on small grids (development tool):
wall time per call and a cProfile of the slowest phase."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1511_04292_b200 as srj  # noqa: E402
from paper_1511_04292_b200.problems import config_fields, config_schedule  # noqa: E402

cyc = config_schedule("cfg1")


def make(shape):
    f = config_fields("cfg1" if len(shape) == 2 else "cfg3", shape)
    nd = len(shape)
    return lambda: srj.GridProblem(spacing=(1.0,) * nd, u=f["u"].copy(), source=f["source"],
                                   center=f["center"], lower=f["lower"], upper=f["upper"],
                                   bc=((srj.FIXED, srj.FIXED),) * nd)


for shape in [(32, 32), (256, 256), (300, 300), (64, 64, 64)]:
    mk = make(shape)
    for it in (1, 1000):
        ts = []
        for rep in range(6):
            p = mk()
            torch.cuda.synchronize()
            t = time.perf_counter()
            srj.srj_solve(p, cyc, 1e-300, max_iters=it)
            ts.append(time.perf_counter() - t)
        print(shape, "max_iters", it, "ms per call:", [round(1e3 * x, 2) for x in ts], flush=True)

mk = make((32, 32))
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    srj.srj_solve(mk(), cyc, 1e-300, max_iters=1)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
