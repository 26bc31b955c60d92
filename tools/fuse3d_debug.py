"""Debug harness for the temporally blocked 3D kernel at a given fused depth.

python tools/fuse3d_debug.py [--n 40] [--fuse 3] [--steps 6]
Runs the cfg3 recipe on an n^3 grid through srj_solve with the given fuse and
compares field + norms with the CPU oracle (development tool).
"""

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import Cycle, problem_from  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_1511_04292_b200 import grids as G  # noqa: E402
from paper_1511_04292_b200.problems import config_fields  # noqa: E402
from paper_1511_04292_b200.schedule import quantize  # noqa: E402
from paper_1511_04292_b200.tables import shipped_table  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs=3, default=[40, 40, 40])
    ap.add_argument("--fuse", type=int, default=3)
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    f = config_fields("cfg3", tuple(a.n))
    w = quantize(shipped_table().lookup(10, 512)).weight_sequence
    p = problem_from(f)
    G.srj_solve(p, Cycle(w), 1e-300, max_iters=a.steps, fuse=a.fuse, chunk=a.steps)
    q = problem_from(f)
    oracle.run(q, w, 0, a.steps)
    got, ref = p.u[1:-1, 1:-1, 1:-1], q.u[1:-1, 1:-1, 1:-1]
    diff = np.argwhere(got != ref)
    print("fuse", a.fuse, "mismatched cells:", len(diff), "of", ref.size, flush=True)
    if len(diff):
        print("first:", diff[:10].tolist())
        print("planes:", sorted(set(diff[:, 0].tolist()))[:20])
        print("rows:", sorted(set(diff[:, 1].tolist()))[:40])
        print("cols:", sorted(set(diff[:, 2].tolist()))[:70])

if __name__ == "__main__":
    main()
