"""Throughput of the residual kernels (development tool): the per-layer
(sum r^2, max|r|) used by the relative-L2 rule (srj_plan_residual_layers) and
the whole-grid one (srj_plan_residual), at the cfg2 and cfg3 sizes, against
16 B per cell (u and f read once)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1511_04292_b200.engine import DeviceGrid  # noqa: E402
from paper_1511_04292_b200.problems import config_fields  # noqa: E402

PEAK = 6555.5
reps = int(os.environ.get("RESID_REPS", "20"))
for wl, shape in (("cfg2", (4096, 4096)), ("cfg3", (512, 512, 512))):
    f = config_fields(wl, shape)
    dev = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"])
    cells = int(np.prod(shape))
    for name, fn in (("layers", lambda: dev.residual_layers(0)), ("whole", lambda: dev.residual(0))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(dev.stream)
        for _ in range(reps):
            fn()
        e1.record(dev.stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = cells * 16 / (ms * 1e-3) / 1e9
        print(json.dumps({"workload": wl, "kernel": name, "ms": ms, "GBps_16B_per_cell": gbs,
                          "frac": gbs / PEAK, "note": "incl. host sync + D2H for layers"}),
              flush=True)
    dev.close()
