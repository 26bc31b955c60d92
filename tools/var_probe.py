"""Throughput of the per-cell-coefficient (reference layout) path vs its HBM
roofline: 65 B/update (2D: u, s, c, 4 coefficients, mask byte, u') and 81 B
(3D).  Development tool; prints JSON lines."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1511_04292_b200.engine import DeviceGrid  # noqa: E402

PEAK = 6555.5


def fields(shape, masked, seed=0):
    rng = np.random.default_rng(seed)
    nd = len(shape)
    c = 4.0 + rng.random(shape)
    lo = tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd))
    hi = tuple(-(0.5 + 0.5 * rng.random(shape)) for _ in range(nd))
    mask = rng.random(shape) > 0.05 if masked else None
    return (np.zeros(tuple(n + 2 for n in shape)), rng.standard_normal(shape), c, lo, hi, mask)


FUSE = [int(x) for x in os.environ.get("VAR_FUSE", "1").split(",")]
SHAPES = [tuple(int(v) for v in s.split("x")) for s in
          os.environ.get("VAR_SHAPES", "4096x4096,512x512x512").split(",")]
for shape, bpu in ((s, 65 if len(s) == 2 else 81) for s in SHAPES):
  for fuse in (FUSE if len(shape) == 2 else [1]):
    for masked in (False, True):
        u, s, c, lo, hi, mask = fields(shape, masked)
        dev = DeviceGrid(u, s, c, lo, hi, active=mask)
        w = np.array([1.3, 0.7])
        dev.run(0, w, 0, 8, fuse)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = int(os.environ.get("VAR_STEPS", "40"))
        e0.record(dev.stream)
        dev.run(0, w, 0, steps, fuse)
        e1.record(dev.stream)
        torch.cuda.synchronize()
        g = np.prod(shape) * steps / (e0.elapsed_time(e1) * 1e-3) / 1e9
        b = bpu if masked else bpu - 1
        print(json.dumps({"shape": shape, "fuse": fuse, "masked": masked, "glups": round(g, 1),
                          "bytes_per_update": b, "frac": round(g * b / PEAK, 3)}), flush=True)
        dev.close()
