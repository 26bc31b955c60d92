"""Per-sweep time of the small-grid path (development tool).

python tools/small_probe.py [--n 256] [--steps 2640]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1511_04292_b200.engine import DeviceGrid  # noqa: E402
from paper_1511_04292_b200.problems import config_fields, config_schedule  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--steps", type=int, default=2640)
a = ap.parse_args()
f = config_fields("cfg1", (a.n, a.n))
w = config_schedule("cfg1").weight_sequence
g = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"])
g.run(0, w, 0, a.steps)
torch.cuda.synchronize()
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(g.stream)
g.run(0, w, 0, a.steps)
e1.record(g.stream)
torch.cuda.synchronize()
print(f"n={a.n} steps={a.steps} {e0.elapsed_time(e1) / a.steps * 1e3:.2f} us/sweep (device), "
      f"{(time.perf_counter() - t0) / a.steps * 1e6:.2f} us/sweep (wall)")
