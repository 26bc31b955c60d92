"""Quick throughput probe of the sweep kernels (development tool, not the bench).

python tools/probe.py [--n 4096] [--fuse 1,2,4,8] [--steps 400]
Prints GLUPS and the algorithmic-HBM fraction (24 B per point-update) for the
2D kernel at each fused depth and the 3D kernel at 512^3 / 256^3.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1511_04292_b200.engine import DeviceGrid  # noqa: E402
from paper_1511_04292_b200.problems import config_fields, config_schedule  # noqa: E402
from paper_1511_04292_b200.schedule import quantize  # noqa: E402
from paper_1511_04292_b200.tables import shipped_table  # noqa: E402

PEAK = 6555.5


def measure(f, w, steps, fuse, warm=2, bc=None):
    """GLUPS of ``steps`` sweeps of the cycle from the initial field.  Every run
    starts from buffer 0, which srj_plan_run never writes (chunk snapshot), so
    warm-up and timed runs see the same input (a run started from another
    buffer ping-pongs through buffer 0)."""
    dev = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"],
                     kappa=f.get("kappa"), bc=bc)
    cells = int(np.prod(f["source"].shape))
    for _ in range(warm):
        dev.run(0, w, 0, min(steps, 64), fuse)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    dev.run(0, w, 0, steps, fuse)
    e1.record(dev.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    glups = cells * steps / (ms * 1e-3) / 1e9
    dev.close()
    return ms / steps, glups, glups * 24 / PEAK


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--fuse", default="1,2,3,4,5,6,8")
    ap.add_argument("--steps", type=int, default=480)
    ap.add_argument("--three", default="512,256")
    ap.add_argument("--nl", type=int, default=1)
    ap.add_argument("--bc", default="", help="2D faces: mirror | face_dirichlet (all four)")
    a = ap.parse_args()
    bc = bc3 = None
    if a.bc:
        from paper_1511_04292_b200 import grids as G

        rule = G.MIRROR if a.bc == "mirror" else G.face_dirichlet(0.5)
        bc = ((rule, rule),) * 2
        bc3 = ((rule, rule),) * 3
    tab = shipped_table()
    w = quantize(tab.lookup(6, 4096)).weight_sequence
    f = config_fields("cfg2", (a.n, a.n))
    out = []
    for fuse in [int(x) for x in a.fuse.split(",") if x]:
        ms, g, frac = measure(f, w, a.steps, fuse, bc=bc)
        r = dict(kind="2d" + ("-" + a.bc if a.bc else ""), n=a.n, fuse=fuse, ms_per_sweep=ms, glups=g, frac_alg=frac)
        print(json.dumps(r), flush=True)
        out.append(r)
    for n in [int(x) for x in a.three.split(",") if x]:
        f3 = config_fields("cfg3", (n, n, n))
        w3 = quantize(tab.lookup(10, 512)).weight_sequence
        for fuse3 in (1, 2, 3):
            ms, g, frac = measure(f3, w3, 48, fuse3, bc=bc3)
            print(json.dumps(dict(kind="3d" + ("-" + a.bc if a.bc else ""), n=n, fuse=fuse3, ms_per_sweep=ms, glups=g,
                                  frac_alg=frac)), flush=True)
    if not a.nl:
        return
    f5 = config_fields("cfg5", (256, 256, 256))
    w5 = config_schedule("cfg5").weight_sequence
    for fuse5 in (1, 2, 3):
        ms, g, frac = measure(f5, w5, 48, fuse5)
        print(json.dumps(dict(kind="3d-nl", n=256, fuse=fuse5, ms_per_sweep=ms, glups=g,
                              frac_alg=frac)), flush=True)


if __name__ == "__main__":
    main()
