"""Gauss-Seidel wavefront throughput (development tool): GPU sweeps vs the
sequential CPU restatement (oracle/, one core) on the cfg2 recipe."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import oracle  # noqa: E402
from helpers import problem_from  # noqa: E402
from paper_1511_04292_b200.engine import DeviceGrid  # noqa: E402
from paper_1511_04292_b200.problems import config_fields  # noqa: E402

for shape, sweeps in (((4096, 4096), 200), ((512, 512), 2000), ((128, 128, 128), 200)):
    f = config_fields("cfg2" if len(shape) == 2 else "cfg3", shape)
    dev = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"])
    dev.gs(1, 1.0, 4)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(dev.stream)
    dev.gs(1, 1.0, sweeps)
    e1.record(dev.stream)
    torch.cuda.synchronize()
    gpu = np.prod(shape) * sweeps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    dev.close()
    q = problem_from(f)
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < 3.0:
        oracle.gs_sweep(q, 1.0)
        n += 1
    cpu = np.prod(shape) * n / (time.perf_counter() - t0) / 1e9
    print(json.dumps({"shape": shape, "gpu_glups": round(gpu, 2), "cpu_1core_glups": round(cpu, 4),
                      "speedup": round(gpu / cpu, 1)}), flush=True)
