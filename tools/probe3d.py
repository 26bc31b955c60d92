"""3D T=2 kernel probe (development tool): throughput and a bitwise fingerprint.

python tools/probe3d.py [--sizes 512,256] [--steps 240]
Runs the cfg3 (linear, 512^3) and cfg5 (nonlinear, 256^3) fields for
``steps`` sweeps of their schedules at fuse=2 and prints, per size, GLUPS,
the per-launch time and a SHA-1 of the resulting field plus the per-step
norms.  Run it once with SRJ_RS3D=0 (shared-memory tile kernel) and once
without (register-streaming kernel): the fingerprints must be identical.
"""

import argparse
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1511_04292_b200.engine import DeviceGrid  # noqa: E402
from paper_1511_04292_b200.problems import config_fields, config_schedule  # noqa: E402


def run(workload, n, steps, fuse, reps):
    f = config_fields(workload, (n, n, n))
    w = config_schedule(workload).weight_sequence
    dev = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"],
                     kappa=f.get("kappa"))
    cells = n ** 3
    dev.run(0, w, 0, min(steps, 64), fuse)
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(dev.stream)
        out = dev.run(0, w, 0, steps, fuse)
        e1.record(dev.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    norms = dev.norms[:2 * steps].cpu().numpy()
    u = np.empty(tuple(s + 2 for s in f["source"].shape))
    dev.download_field(out, u)
    h = hashlib.sha1(u.tobytes() + norms.tobytes()).hexdigest()
    dev.close()
    return {"workload": workload, "n": n, "steps": steps, "fuse": fuse,
            "glups": cells * steps / (best * 1e-3) / 1e9,
            "us_per_launch": best * 1e3 / (steps / fuse), "sha1": h,
            "finite": bool(np.isfinite(u).all()), "max_abs": float(np.abs(u).max())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="512,256")
    ap.add_argument("--steps", type=int, default=240)
    ap.add_argument("--fuse", type=int, default=2)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--workloads", default="cfg3,cfg5")
    a = ap.parse_args()
    mode = "tb" if os.environ.get("SRJ_RS3D", "1") == "0" else "rs"
    for n in [int(x) for x in a.sizes.split(",")]:
        for wl in a.workloads.split(","):
            r = run(wl, n, a.steps, a.fuse, a.reps)
            r["kernel"] = mode
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
