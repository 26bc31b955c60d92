"""Throughput of fused sweeps with non-FIXED faces (development tool).

python tools/bc_probe.py [--n 4096] [--steps 480]
Each line: which faces are MIRROR (rows = axis-0 faces, cols = axis-1 faces),
fused depth, GLUPS -- isolates the cost of the row- and column-face paths of
the band kernel.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from probe import measure  # noqa: E402

from paper_1511_04292_b200 import grids as G  # noqa: E402
from paper_1511_04292_b200.problems import config_fields  # noqa: E402
from paper_1511_04292_b200.schedule import quantize  # noqa: E402
from paper_1511_04292_b200.tables import shipped_table  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=480)
    ap.add_argument("--jacobi", action="store_true",
                    help="weight 0.9 on every sweep (no partial-cycle growth: the SRJ cycle's "
                         "large weights can drive a partial cycle to inf/NaN, whose cells take "
                         "the IEEE-division fallback)")
    a = ap.parse_args()
    w = quantize(shipped_table().lookup(6, 4096)).weight_sequence
    if a.jacobi:
        import numpy as np

        w = np.array([0.9])
    f = config_fields("cfg2", (a.n, a.n))
    F, M = G.FIXED, G.MIRROR
    cases = {"none": ((F, F), (F, F)), "rows": ((M, M), (F, F)), "cols": ((F, F), (M, M)),
             "west": ((F, F), (M, F)), "all": ((M, M), (M, M))}
    D = G.face_dirichlet(0.5)
    cases["all-face-dirichlet"] = ((D, D), (D, D))
    for name, bc in cases.items():
        for fuse in (1, 4):
            ms, g, _ = measure(f, w, a.steps, fuse, bc=None if name == "none" else bc)
            print(json.dumps(dict(faces=name, n=a.n, fuse=fuse, ms_per_sweep=ms, glups=g)),
                  flush=True)


if __name__ == "__main__":
    main()
