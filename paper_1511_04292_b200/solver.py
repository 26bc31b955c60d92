"""The chunked stopping-rule loop shared by the 1-GPU and the N-rank solvers.

The reference checks its rule after every elementary step (``_iterate``,
``/root/reference/pkg/src/srj/grids.py:602-629``; metric ``dmax/|omega|`` of
``srj_solve`` ``:684``; overflow guard ``:618-625``).  On the GPU the steps of a
chunk run back to back and write their per-step (dmax, rmax) into a device
buffer; the host reads it once per chunk, finds the first step where the guard
or the rule fires and, if that step is inside the chunk, replays the chunk from
its untouched start buffer to exactly that step.  So iteration counts,
histories and the returned field are the reference's.

``backend`` runs the steps (one device: ``GridBackend``; one rank of a slab
decomposition: ``distributed.DeviceSlab``); ``comm`` combines per-rank values
(``LocalComm`` for one process, ``distributed.DistComm`` over a process
group).  Every decision is taken on all-reduced values, so all ranks stop at
the same step and raise ``DivergenceError`` at the same step.

The BASELINE's relative-L2 rule (``stop="residual_l2"``, not in the
reference) uses the per-layer residual kernel (``srj_plan_residual_layers``):
each axis-0 layer's (sum r^2, max|r|) depends only on that layer's cells, and
the host takes the exactly rounded sum over layers (``math.fsum``), so the L2
value -- and hence the stopping step -- is identical on 1 and N GPUs.
"""

import math
import time

import numpy as np

__all__ = ["GridBackend", "LocalComm", "OVERFLOW_LIMIT", "l2_from_layers", "run_solve"]

OVERFLOW_LIMIT = 1e300  # grids.py:53


class LocalComm:
    """One process: the all-reduces are the identity."""

    world = 1
    rank = 0

    @staticmethod
    def max_(a):
        return a

    @staticmethod
    def sum_(a):
        return a


class GridBackend:
    """One ``DeviceGrid`` holding the whole problem."""

    def __init__(self, dev, n_layers):
        self.dev = dev
        self.n_layers = int(n_layers)
        self.layer0 = 0

    def run_chunk(self, src, weights, first, n, fuse):
        return self.dev.run(src, weights, first, n, fuse)

    def norms(self, n):
        return self.dev.norms[:2 * n].view(n, 2).cpu().numpy()

    def residual_layers(self, buf):
        return self.dev.residual_layers(buf)


def l2_from_layers(backend, comm, layers):
    """(||r||_2, max|r|) from this rank's per-layer (sum r^2, max|r|)."""
    full = np.zeros((backend.n_layers, 2))
    full[backend.layer0:backend.layer0 + len(layers)] = layers
    full = comm.sum_(full)  # each layer is owned by exactly one rank: x + 0 == x
    return math.sqrt(math.fsum(full[:, 0])), float(np.max(full[:, 1], initial=0.0))


def source_l2(backend, comm, source_layers_sq):
    """||source||_2 from per-layer sums of squares (owned layers)."""
    full = np.zeros(backend.n_layers)
    full[backend.layer0:backend.layer0 + len(source_layers_sq)] = source_layers_sq
    full = comm.sum_(full)
    return math.sqrt(math.fsum(full))


def step_seconds_estimate(cells):
    return 3e-6 + cells * 24.0 / 5e12


def run_solve(backend, comm, weights, tol, max_iters, normalise, stop, check_every, fuse, chunk,
              l2_reference, cells, src=0):
    """Returns (dict of history arrays, converged, diverged, final buffer)."""
    tol = float(tol)
    if tol <= 0.0:
        raise ValueError("tolerance must be positive")
    if max_iters < 1:
        raise ValueError("max_iters must be at least 1")
    if stop not in ("update_inf", "residual_l2"):
        raise ValueError(f"unknown stopping rule {stop!r}")
    w = np.asarray(weights, dtype=np.float64)
    m = len(w)
    absw = np.abs(w) if normalise else np.ones(m)
    start = time.perf_counter()
    diffs, resids, secs, l2s = [], [], [], []
    converged = False
    diverged = False
    cur = src
    done = 0
    if stop == "residual_l2":
        every = int(check_every or m)
        if every < 1:
            raise ValueError("check_every must be at least 1")
        if callable(l2_reference):
            l2_reference = l2_reference()
        if l2_reference == 0.0:
            l2_reference = 1.0
        span = cap = every
    elif chunk:
        span = cap = int(chunk)
    else:
        # the first chunk covers ~2 ms of work, each next one doubles up to
        # ~50 ms, so replaying the chunk in which the rule fires costs at most
        # about as much as the work so far (sized from the GLOBAL grid, so all
        # ranks take the same chunks)
        est = step_seconds_estimate(cells)
        # (small grids: ~20 ms chunks -- a host check costs ~0.1 ms there, the
        # replay of the last chunk on average half a chunk)
        cap = int(min(65536, max(64, (0.02 if est < 2e-5 else 0.05) / est)))
        span = int(min(cap, max(32, 0.002 / est)))
    while done < max_iters:
        n = min(span, max_iters - done)
        span = min(cap, 2 * span)
        if stop == "residual_l2":
            n = min(n, every - done % every)
        out = backend.run_chunk(cur, w, done, n, fuse)
        norms = comm.max_(backend.norms(n))
        t_now = time.perf_counter() - start
        t_prev = float(secs[-1][-1]) if secs else 0.0
        metric = norms[:, 0] / absw[(done + np.arange(n)) % m]
        bad = ~np.isfinite(metric) | (metric > OVERFLOW_LIMIT)
        hit = metric < tol if stop == "update_inf" else np.zeros(n, dtype=bool)
        events = np.flatnonzero(bad | hit)
        take = n if events.size == 0 else int(events[0]) + 1
        if take < n:
            out = backend.run_chunk(cur, w, done, take, fuse)  # replay to the exact step
        diffs.append(metric[:take])
        resids.append(norms[:take, 1])
        secs.append(t_prev + (t_now - t_prev) * np.arange(1, take + 1) / take)
        done += take
        cur = out
        if events.size:
            if bad[take - 1]:
                diverged = True
            else:
                converged = True
            break
        if stop == "residual_l2" and done % every == 0:
            l2, _ = l2_from_layers(backend, comm, backend.residual_layers(cur))
            rel = l2 / l2_reference
            l2s.append((done, rel))
            if rel < tol:
                converged = True
                break
    hist = {
        "residual_inf": np.concatenate(diffs) if diffs else np.zeros(0),
        "true_residual_inf": np.concatenate(resids) if resids else np.zeros(0),
        "seconds": np.concatenate(secs) if secs else np.zeros(0),
        "relative_l2": np.asarray(l2s, dtype=float).reshape(-1, 2),
    }
    return hist, converged, diverged, cur
