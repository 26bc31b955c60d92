import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from helpers import Cycle, problem_from
from paper_1511_04292_b200 import grids as G
from paper_1511_04292_b200.problems import config_fields, config_schedule
f = config_fields("cfg2"); w = config_schedule("cfg2").weight_sequence
res = {}
for fuse in (1, 4):
    p = problem_from(f)
    h, _ = G.srj_solve(p, Cycle(w), tol=1e-300, max_iters=48, fuse=fuse)
    res[fuse] = (h.residual_inf, h.true_residual_inf, p.u.copy())
a, b = res[1], res[4]
print("field equal", np.array_equal(a[2], b[2]))
d = np.flatnonzero(a[0] != b[0]); r = np.flatnonzero(a[1] != b[1])
print("dmax differ at", d, "rmax differ at", r)
for i in r[:8]: print(i, a[1][i], b[1][i], b[1][i] / a[1][i])
