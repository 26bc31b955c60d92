"""Host cost of the multi-GPU step loop, measured on one GPU with emulated ranks.

cfg3 (512^3, P=10) split into z-slabs of 8 ranks (64 planes each), halo 2,
T=2: every fused launch of every rank is 2-3 kernel launches (edge / inner
rows), 1-2 peer copies and 4-8 flag operations (srj_slab_run).  While a long
sleep kernel keeps the GPU busy, the host enqueues K fused launches for all
ranks; host microseconds per fused launch per rank = call time / (K * ranks).
Compare with a cfg3 8-GPU fused launch (~130 us of device time): the
DESIGN.md target is < 10%.  Also reports the device time per fused step of
the emulated 8-rank run vs the 1-rank plan (the cost of the edge/inner split
on one GPU; on real GPUs the ranks run in parallel).

usage: python tools/slab_overhead.py [ranks]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_04292_b200.distributed import EmulatedRanks  # noqa: E402
from paper_1511_04292_b200.grids import FIXED, GridProblem  # noqa: E402
from paper_1511_04292_b200.problems import config_fields, config_schedule  # noqa: E402


def main():
    ranks = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    torch.cuda.set_device(0)
    f = config_fields("cfg3")
    p = GridProblem(spacing=(1.0,) * 3, u=f["u"], source=f["source"], center=f["center"],
                    lower=f["lower"], upper=f["upper"], bc=((FIXED, FIXED),) * 3)
    w = config_schedule("cfg3").weight_sequence
    em = EmulatedRanks(p, ranks, 2)
    cur = em.run_chunk(0, w, 0, 8, 2)  # warm (TMA descriptors, attributes)
    torch.cuda.synchronize()
    out = {"ranks": ranks}
    # host enqueue cost behind a long sleep kernel, in calls short enough not
    # to fill the launch queue (which would block the host on the GPU)
    per_k = {}
    for k in (1, 2, 4):
        samples = []
        for _ in range(5):
            torch.cuda._sleep(200_000_000)  # ~0.1 s at 1.9 GHz
            t0 = time.perf_counter()
            cur = em.run_chunk(cur, w, 0, 2 * k, 2)
            samples.append(time.perf_counter() - t0)
            torch.cuda.synchronize()
        per_k[k] = min(samples) / (k * ranks) * 1e6
    out["host_us_per_fused_launch_per_rank_by_K"] = per_k
    host_us = min(per_k.values())
    out["host_us_per_fused_launch_per_rank"] = host_us
    # device time per fused step: emulated ranks (serialised on one GPU)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 200
    ev0.record()
    cur = em.run_chunk(cur, w, 0, steps, 2)
    ev1.record()
    torch.cuda.synchronize()
    out["emulated_device_us_per_fused_step_all_ranks"] = ev0.elapsed_time(ev1) * 1e3 / (steps / 2)
    em.close()
    from paper_1511_04292_b200.engine import DeviceGrid

    g = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"])
    c = g.run(0, w, 0, 8, 2)
    torch.cuda.synchronize()
    ev0.record()
    c = g.run(c, w, 0, steps, 2)
    ev1.record()
    torch.cuda.synchronize()
    out["one_rank_device_us_per_fused_step"] = ev0.elapsed_time(ev1) * 1e3 / (steps / 2)
    # host cost of one plain fused launch (srj_plan_run, no exchange): the
    # floor of the per-launch host cost, one kernel launch
    samples = []
    for _ in range(5):
        torch.cuda._sleep(200_000_000)
        t0 = time.perf_counter()
        c = g.run(c, w, 0, 64, 2)
        samples.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
    out["host_us_per_plain_fused_launch"] = min(samples) / 32 * 1e6
    out["ratio_to_8gpu_launch_130us"] = host_us / 130.0
    print(json.dumps(out))


if __name__ == "__main__":
    main()
