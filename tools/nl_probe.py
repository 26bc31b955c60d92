import sys, time, json, numpy as np, torch
sys.path.insert(0, '.')
from paper_1511_04292_b200 import grids as G
from paper_1511_04292_b200.problems import config_fields
from paper_1511_04292_b200.schedule import quantize
from paper_1511_04292_b200.tables import shipped_table
t = shipped_table()
f = config_fields("cfg5")
for (P, N) in [(8, 256), (8, 200), (8, 150), (8, 128), (6, 150), (6, 256), (10, 150), (4, 150)]:
    try: ws = t.lookup(P, N)
    except Exception as e: print(P, N, e); continue
    cyc = quantize(ws)
    p = G.GridProblem(spacing=(1.,)*3, u=f["u"].copy(), source=f["source"], center=f["center"],
                      lower=f["lower"], upper=f["upper"], bc=((G.FIXED, G.FIXED),)*3, source_kappa=f["kappa"])
    t0 = time.perf_counter()
    try:
        h, _ = G.srj_solve(p, cyc, 1e-8, max_iters=60 * cyc.m, stop="residual_l2")
        st = "converged" if h.converged else "max"
    except G.DivergenceError as e:
        h, st = e.history, "diverged"
    print(json.dumps(dict(P=P, N=int(ws.n), M=int(cyc.m), w1=float(ws.omegas[0]), status=st, steps=int(h.iterations),
          cycles=round(h.iterations / cyc.m, 2), s=round(time.perf_counter() - t0, 3),
          checks=[round(float(x), 12) for x in h.relative_l2[:6, 1]])), flush=True)
