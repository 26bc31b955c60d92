"""Per-rank device timeline of the slab path on ONE GPU (weak/strong-scaling
proxy).  The middle rank of a 3-rank decomposition runs the real
``srj_slab_run`` -- edge launches, peer copies, flag-word stream operations,
inner launch, or in direct mode one launch whose kernel stores the edge rows
into the neighbours' halos -- against two VIRTUAL neighbours: a never-run clone slab on the
same device receives the edge rows, and this rank's own flag words are preset
far in the future, so every flag wait passes at once.  What is timed is
therefore everything a rank of a multi-GPU run does per fused launch except
the NVLink transfer itself (the copies are device-local) and waiting for a
slower neighbour; compared with the same rows as one whole grid
(``srj_plan_run``) it gives the decomposition efficiency of one rank.

    python tools/slab_rank_probe.py cfg2 4096 4096 --fuse 4 --steps 2000
    python tools/slab_rank_probe.py cfg3 64 512 512 --fuse 2 --steps 400
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1511_04292_b200.distributed import (DeviceSlab, SlabDecomposition,  # noqa: E402
                                               default_halo, run_slabs)
from paper_1511_04292_b200.engine import DeviceGrid  # noqa: E402
from paper_1511_04292_b200.problems import (config_fields, config_schedule,  # noqa: E402
                                            slab_config_fields)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e-3 / reps


MODES = {"direct_store": {}, "split_streams": {"SRJ_SLAB_DIRECT": "0"},
         "one_stream": {"SRJ_SLAB_DIRECT": "0", "SRJ_SLAB_SPLIT": "0"}}


def probe(workload, own, fuse=0, steps=1000, reps=3, modes=tuple(MODES)):
    """Efficiency of one slab rank owning ``own`` rows x the other axes
    (module docstring); returns a dict for one JSON line."""
    own = tuple(int(x) for x in own)
    nd = len(own)
    w = config_schedule(workload).weight_sequence
    halo = default_halo(nd, fuse)
    cells = int(np.prod(own))

    # the same rows as one whole grid (no neighbours)
    f = config_fields(workload, own)
    g = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"], kappa=f.get("kappa"))
    t_whole = timed(lambda: g.run(0, w, 0, steps, fuse), reps)
    g.close()

    # middle rank of three, virtual neighbours
    gshape = (3 * own[0],) + own[1:]
    d = SlabDecomposition(gshape[0], 3, 1, halo)
    out = {"workload": workload, "owned": list(own), "fuse": fuse, "halo": halo, "steps": steps,
           "whole_grid_glups": round(cells * steps / t_whole / 1e9, 2)}
    for key in modes:
        env = MODES[key]
        os.environ.update(env)
        try:
            slab = DeviceSlab(slab_config_fields(workload, d, gshape))
            lo, hi = (DeviceSlab(slab_config_fields(workload, d, gshape)) for _ in range(2))
            slab.connect_local(lo, hi)
            slab.reset()
            slab.grid.flags.fill_(0x7FFFFFF0)  # every flag wait is already satisfied
            torch.cuda.synchronize()
            t = timed(lambda: run_slabs([slab], 0, w, 0, steps, fuse), reps)
            out[key + "_glups"] = round(cells * steps / t / 1e9, 2)
            out[key + "_efficiency"] = round(t_whole / t, 4)
            for s in (slab, lo, hi):
                s.close()
        finally:
            for k in env:
                os.environ.pop(k, None)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("workload")
    ap.add_argument("shape", type=int, nargs="+", help="rows owned by the rank, then the other axes")
    ap.add_argument("--fuse", type=int, default=0)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    print(json.dumps(probe(args.workload, args.shape, args.fuse, args.steps, args.reps)),
          flush=True)


if __name__ == "__main__":
    main()
