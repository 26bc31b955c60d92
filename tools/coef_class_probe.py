"""Per-cell-coefficient problems with and without coefficient classes
(srj_plan_set_coef_classes; development tool, prints JSON lines).

python tools/coef_class_probe.py [--n2 4096] [--n3 256,512] [--steps 400]

Workloads (classes = SRJ_COEF_* bits per array, engine.coef_class):
  * gs-A / gs-B: the reference's Grad-Shafranov builder (problems.py:634-717)
    at n x n: center row-constant, radial coefficients constant, the two theta
    coefficients per cell; MIRROR theta faces (one sweep per launch) and, as
    "fixed", the same arrays with FIXED faces (the fused T=2 kernel);
  * sph3d: the spherical Poisson builder's coefficient structure
    (problems.py:540-556: radial profiles, theta profiles, mask of the first
    radial layer) on FIXED faces;
  * mask2d / mask3d: a constant stencil under a 5% random mask.
Each case runs with classes off (SRJ_COEF_CLASSES=0: every array read per
cell, the round-1 path) and on, on the same device buffers' inputs, and the
final fields are compared bit for bit.
"""

import argparse
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1511_04292_b200 import grids as G  # noqa: E402
from paper_1511_04292_b200.engine import DeviceGrid  # noqa: E402
from paper_1511_04292_b200.problems import config_fields, grad_shafranov_fields  # noqa: E402
from paper_1511_04292_b200.schedule import quantize  # noqa: E402
from paper_1511_04292_b200.tables import shipped_table  # noqa: E402


def sph3d_fields(n):
    """Coefficient structure of spherical_poisson(d=3) (problems.py:540-556)."""
    dr, dth, dph = 1.0 / n, math.pi / n, 2.0 * math.pi / n
    r = (np.arange(n) + 0.5) * dr
    th = (np.arange(n) + 0.5) * dth
    shape = (n, n, n)
    z = np.zeros(shape)
    cot = 1.0 / np.tan(th)
    ph = 1.0 / (np.sin(th) ** 2 * dph ** 2)
    center = (-2.0 * r ** 2 / dr ** 2)[:, None, None] - 2.0 / dth ** 2 - 2.0 * ph[None, :, None] + z
    lower = ((r * (r - dr) / dr ** 2)[:, None, None] + z,
             (1.0 / dth ** 2 - cot / (2.0 * dth))[None, :, None] + z, ph[None, :, None] + z)
    upper = ((r * (r + dr) / dr ** 2)[:, None, None] + z,
             (1.0 / dth ** 2 + cot / (2.0 * dth))[None, :, None] + z, ph[None, :, None] + z)
    rng = np.random.default_rng(3)
    mask = np.ones(shape, dtype=bool)
    mask[0] = False
    return {"u": np.zeros(tuple(m + 2 for m in shape)), "source": rng.standard_normal(shape),
            "center": center, "lower": lower, "upper": upper, "mask": mask}


def masked_fields(name, shape):
    f = dict(config_fields(name, shape))
    f["mask"] = np.random.default_rng(7).random(shape) > 0.05
    return f


def run_case(name, f, w, steps, fuse, bc, classes):
    os.environ["SRJ_COEF_CLASSES"] = "1" if classes else "0"
    dev = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"],
                     active=f.get("mask"), bc=bc)
    cls = list(dev.coef_classes)
    cells = int(np.prod(np.shape(f["source"])))
    dev.run(0, w, 0, min(steps, 16), fuse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    out = dev.run(0, w, 0, steps, fuse)
    e1.record(dev.stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    field = dev.fields[out].cpu().numpy()
    norms = dev.norms[:2 * steps].cpu().numpy()
    dev.close()
    return dict(case=name, classes=cls if classes else "off", fuse=fuse,
                ms_per_sweep=ms / steps, glups=cells * steps / (ms * 1e-3) / 1e9), field, norms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n2", type=int, default=4096)
    ap.add_argument("--n3", default="256,512")
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--cases", default="", help="regex: run only matching case names")
    a = ap.parse_args()
    w = quantize(shipped_table().lookup(6, 4096)).weight_sequence
    F, M = G.FIXED, G.MIRROR
    n = a.n2
    cases = []
    for test in ("A", "B") if n else ():
        f = grad_shafranov_fields(test, 0.0, n)
        cases.append((f"gs-{test}-mirror", f, a.steps, 0, ((F, F), (M, M))))
        cases.append((f"gs-{test}-fixed", f, a.steps, 0, None))
    if n:
        cases.append(("mask2d", masked_fields("cfg2", (n, n)), a.steps, 0, None))
    for n3 in [int(x) for x in a.n3.split(",") if x]:
        steps3 = max(16, a.steps * 256 ** 3 // (n3 ** 3) // 4)
        cases.append((f"sph3d-{n3}", sph3d_fields(n3), steps3, 0, None))
        cases.append((f"mask3d-{n3}", masked_fields("cfg3", (n3,) * 3), steps3, 0, None))
    import re

    for name, f, steps, fuse, bc in cases:
        if a.cases and not re.search(a.cases, name):
            continue
        r0, x0, n0 = run_case(name, f, w, steps, fuse, bc, False)
        r1, x1, n1 = run_case(name, f, w, steps, fuse, bc, True)
        same = bool(np.array_equal(x0.view(np.int64), x1.view(np.int64))
                    and np.array_equal(n0.view(np.int64), n1.view(np.int64)))
        r1["speedup"] = r1["glups"] / r0["glups"]
        r1["bitwise_equal_to_off"] = same
        print(json.dumps(r0), flush=True)
        print(json.dumps(r1), flush=True)


if __name__ == "__main__":
    main()
