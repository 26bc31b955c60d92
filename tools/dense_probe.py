"""Throughput of the kernel-level drop-in srj_wj_dense (reference dense layout,
65 B/update 2D, 81 B 3D) vs the HBM roofline.  Development tool."""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1511_04292_b200 import _lib  # noqa: E402

PEAK = 6555.5
lib = _lib.load()
for shape, bpu in (((4096, 4096), 64), ((512, 512, 512), 80)):
    nd = len(shape)
    g = tuple(n + 2 for n in shape)
    dev = torch.device("cuda")
    u = torch.zeros(g, dtype=torch.float64, device=dev)
    un = torch.zeros(g, dtype=torch.float64, device=dev)
    s = torch.randn(shape, dtype=torch.float64, device=dev)
    c = torch.full(shape, 4.0 + nd, dtype=torch.float64, device=dev)
    lo = [torch.full(shape, -1.0, dtype=torch.float64, device=dev) for _ in range(nd)]
    hi = [torch.full(shape, -1.0, dtype=torch.float64, device=dev) for _ in range(nd)]
    norms = torch.zeros(2, dtype=torch.float64, device=dev)
    n = (ctypes.c_int64 * 3)(*(list(shape) + [0] * (3 - nd)))
    lop = (ctypes.c_void_p * nd)(*[a.data_ptr() for a in lo])
    hip = (ctypes.c_void_p * nd)(*[a.data_ptr() for a in hi])
    st = torch.cuda.current_stream()

    def step(a, b, om):
        _lib.check(lib.srj_wj_dense(nd, n, ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                    ctypes.c_void_p(s.data_ptr()), ctypes.c_void_p(c.data_ptr()), lop, hip,
                                    None, ctypes.c_double(om), ctypes.c_void_p(norms.data_ptr()),
                                    ctypes.c_void_p(st.cuda_stream)), "srj_wj_dense")

    for _ in range(3):
        step(u, un, 0.9)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for k in range(reps):
        step(u, un, 0.9) if k % 2 == 0 else step(un, u, 0.9)
    e1.record()
    torch.cuda.synchronize()
    glups = np.prod(shape) * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    print(json.dumps({"shape": shape, "glups": round(glups, 1), "bytes_per_update": bpu,
                      "frac": round(glups * bpu / PEAK, 3)}), flush=True)
