"""Slab (row-block) domain decomposition of the SRJ sweep across GPUs.

The reference has no parallel path (SPEC.md:305 lists distributed memory as a
non-goal); this module is the multi-GPU design of SURVEY.md section 8(e):

* The global interior is split along axis 0 (slowest, C-order) into contiguous
  blocks, one per rank (``SlabDecomposition``).
* Each rank holds its owned rows plus ``halo`` extra rows on every side that
  has a neighbour.  The local grid treats the layer beyond a halo as a fixed
  ghost; with ``halo >= fuse`` the stale values there never reach an owned
  cell within one fused launch of ``fuse`` sweeps (the dependency cone shrinks
  one row per sweep), so the owned rows are exact.
* After every fused launch each rank sends its first/last ``halo`` owned rows
  to its neighbours' halo rows (point-to-point NCCL send/recv of contiguous
  padded layers -- no packing), which restores the invariant.
* Per-step (dmax, rmax) are computed over owned rows only and combined with
  one MAX all-reduce per chunk of steps; MAX is exact, so every rank takes the
  identical stopping decision and the k-GPU field is bitwise the 1-GPU field.

The exchange/norm logic is backend-agnostic: ``SlabSolver`` drives any object
with the ``SlabBackend`` interface.  The product backend is ``DeviceSlab``
(libsrj kernels on the rank's GPU, NCCL); the CPU tests plug the oracle in
with the ``gloo`` backend to check the decomposition without GPUs.
"""

from dataclasses import dataclass

import numpy as np

__all__ = ["DeviceSlab", "SlabDecomposition", "SlabGrid", "SlabSolver"]


@dataclass(frozen=True)
class SlabDecomposition:
    """Row ranges of rank ``rank`` out of ``world`` for an ``n0``-row grid."""

    n0: int
    world: int
    rank: int
    halo: int

    def __post_init__(self):
        if self.world < 1 or not 0 <= self.rank < self.world:
            raise ValueError("bad rank/world")
        if self.n0 < self.world * max(1, self.halo):
            raise ValueError(
                f"{self.n0} rows cannot be split over {self.world} ranks with halo {self.halo}")

    @property
    def owned(self):
        """Global interior rows [r0, r1) this rank owns (balanced split)."""
        base, extra = divmod(self.n0, self.world)
        r0 = self.rank * base + min(self.rank, extra)
        return r0, r0 + base + (1 if self.rank < extra else 0)

    @property
    def h_lo(self):
        return self.halo if self.rank > 0 else 0

    @property
    def h_hi(self):
        return self.halo if self.rank < self.world - 1 else 0

    @property
    def local_rows(self):
        """Global interior rows [a, b) stored locally (owned + halos)."""
        r0, r1 = self.owned
        return r0 - self.h_lo, r1 + self.h_hi

    @property
    def own_local(self):
        """Owned rows in local interior indices."""
        r0, r1 = self.owned
        return self.h_lo, self.h_lo + (r1 - r0)

    def local_field(self, u):
        """Slice of a ghosted global field (n0+2 rows) for this rank."""
        a, b = self.local_rows
        return u[a:b + 2]

    def local_interior(self, a_global):
        a, b = self.local_rows
        return a_global[a:b]

    def row_parts(self):
        """(edges, inner): owned local interior row ranges [a, b).  ``edges``
        are the rows the neighbours need (sent after every launch), ``inner``
        the rest (None when the slab is all edge).  The overlapped solver
        relaxes the edges first, starts the exchange, then relaxes the inner
        rows while the halo rows travel."""
        lo, hi = self.own_local
        a = lo + (self.halo if self.rank > 0 else 0)
        b = hi - (self.halo if self.rank < self.world - 1 else 0)
        if a >= b:
            return [(lo, hi)], None
        edges = []
        if a > lo:
            edges.append((lo, a))
        if b < hi:
            edges.append((b, hi))
        return edges, (a, b)

    # Exchange plan in LOCAL LAYER indices of the ghosted local field
    # (layer = local interior row + 1).
    def sends(self):
        """[(peer, first_layer, count)] of owned rows sent to neighbours."""
        lo, hi = self.own_local
        out = []
        if self.rank > 0:
            out.append((self.rank - 1, lo + 1, self.halo))
        if self.rank < self.world - 1:
            out.append((self.rank + 1, hi - self.halo + 1, self.halo))
        return out

    def recvs(self):
        """[(peer, first_layer, count)] of halo rows received from neighbours."""
        lo, hi = self.own_local
        out = []
        if self.rank > 0:
            out.append((self.rank - 1, 1, self.halo))
        if self.rank < self.world - 1:
            out.append((self.rank + 1, hi + 1, self.halo))
        return out


class SlabSolver:
    """Drives a slab backend: fused launches, halo exchange, norm all-reduce.

    backend methods:
      reserve(nsteps) -- size the per-step norm buffers for a chunk
      run(src, dst, weights, first, nsteps, norms_offset, rows=None) -- nsteps
          <= fuse sweeps from buffer src into buffer dst; rows=None relaxes and
          stores every owned row, rows=(a, b) only local rows [a, b) (the
          edge / inner split); per-step norms of those rows are folded (MAX)
          into the chunk's norm buffer at norms_offset
      layers(buf, first_layer, count) -> contiguous tensor view of layers
      norms(nsteps) -> tensor [nsteps, 2] (dmax, rmax) of the last chunk
      comm() -> context manager for the exchange (a side CUDA stream on GPU)
      comm_fence() -> order the main stream after the exchange (GPU)

    ``overlap`` (default on when the world has neighbours; SRJ_SLAB_OVERLAP=0
    turns it off): every launch is split into the edge rows the neighbours
    need and the inner rows; the halo exchange runs on the comm stream
    concurrently with the inner launch.  Edge and inner rows are
    disjoint and the exchange touches only edge rows (sent) and halo rows
    (received) of the destination buffer, so the split changes no value.
    """

    def __init__(self, backend, decomp, group=None, fuse=4, overlap=None):
        import os

        if fuse > max(1, decomp.halo) and decomp.world > 1:
            raise ValueError(f"fuse depth {fuse} exceeds halo {decomp.halo}")
        self.b = backend
        self.d = decomp
        self.group = group
        self.fuse = int(fuse)
        if overlap is None:
            overlap = os.environ.get("SRJ_SLAB_OVERLAP", "1") != "0"
        self.overlap = bool(overlap) and decomp.world > 1

    def _post_exchange(self, buf):
        import torch.distributed as dist

        ops = []
        for peer, first, count in self.d.recvs():
            ops.append(dist.P2POp(dist.irecv, self.b.layers(buf, first, count), peer,
                                  group=self.group))
        for peer, first, count in self.d.sends():
            ops.append(dist.P2POp(dist.isend, self.b.layers(buf, first, count), peer,
                                  group=self.group))
        return dist.batch_isend_irecv(ops)

    def exchange(self, buf):
        if self.d.world == 1:
            return
        for req in self._post_exchange(buf):
            req.wait()

    def run(self, src, weights, first, nsteps):
        """Steps [first, first+nsteps) from buffer ``src``; returns (dst, norms).

        ``src`` is left untouched (chunk snapshot); the result lands in one of
        the two other buffers.  ``norms`` is a host array [nsteps, 2] already
        reduced over ranks.
        """
        import torch
        import torch.distributed as dist

        self.b.reserve(nsteps)
        others = [i for i in range(3) if i != src]
        cur, k, flip = src, 0, 0
        edges, inner = self.d.row_parts() if self.overlap else (None, None)
        while k < nsteps:
            t = min(self.fuse, nsteps - k)
            dst = others[flip]
            if not self.overlap:
                self.b.run(cur, dst, weights, first + k, t, k)
                self.exchange(dst)
            else:
                for rows in edges:
                    self.b.run(cur, dst, weights, first + k, t, k, rows=rows)
                with self.b.comm():
                    reqs = self._post_exchange(dst)
                if inner is not None:
                    self.b.run(cur, dst, weights, first + k, t, k, rows=inner)
                with self.b.comm():
                    for req in reqs:
                        req.wait()
                self.b.comm_fence()
            cur, flip, k = dst, 1 - flip, k + t
        norms = self.b.norms(nsteps)
        if self.d.world > 1:
            dist.all_reduce(norms, op=dist.ReduceOp.MAX, group=self.group)
        if isinstance(norms, torch.Tensor):
            norms = norms.cpu().numpy()
        return cur, np.asarray(norms).reshape(nsteps, 2)


class DeviceSlab:
    """GPU backend: this rank's rows in a ``DeviceGrid`` (libsrj kernels)."""

    def __init__(self, fields, decomp, device=None):
        from .engine import DeviceGrid

        d = decomp
        kappa = fields.get("kappa")
        sl = d.local_interior
        self.grid = DeviceGrid(
            d.local_field(fields["u"]), sl(fields["source"]), sl(fields["center"]),
            tuple(sl(a) for a in fields["lower"]), tuple(sl(a) for a in fields["upper"]),
            active=None if fields.get("mask") is None else sl(fields["mask"]),
            kappa=None if kappa is None else sl(kappa), own=d.own_local, device=device)
        self.plane = int(self.grid.layout.plane)
        self.origin = int(self.grid.layout.origin)
        self.stream = self.grid.stream
        # deepest single-launch fusion the plan runs (libsrj srj_plan_run)
        self.max_fuse = (4 if self.grid.ndim == 2 else 3) if self.grid.constant else 1
        self._part_norms = None
        self._comm = None
        edges, _ = decomp.row_parts()
        # the overlapped solver runs the edges first (a single rank has none)
        self._first_part = edges[0] if edges else None

    def reserve(self, nsteps):
        torch = self.grid.torch
        self.grid.ensure_norms(nsteps)
        if self._part_norms is None or self._part_norms.numel() < 2 * nsteps:
            self._part_norms = torch.zeros(2 * max(nsteps, 1), dtype=torch.float64,
                                           device=self.grid.device)

    def run(self, src, dst, weights, first, nsteps, norms_offset, rows=None):
        g = self.grid
        if rows is None:
            g.run_single(g.plan, src, dst, weights, first, nsteps,
                         g.norms[2 * norms_offset:])
            return
        # edge / inner launch: its own plan over the same fields; per-step
        # norms folded into the chunk buffer (the first part of a launch
        # overwrites, later ones take the MAX -- exact, order-free)
        part = self._part_norms[:2 * nsteps]
        g.run_single(g.sub_plan(*rows), src, dst, weights, first, nsteps, part)
        with g._on(), g.torch.cuda.stream(g.stream):
            view = g.norms[2 * norms_offset:2 * (norms_offset + nsteps)]
            if rows == self._first_part:
                view.copy_(part)
            else:
                g.torch.maximum(view, part, out=view)

    def comm(self):
        """Exchange context: the comm stream, ordered after the work queued
        so far on the main stream (the edge launches)."""
        import contextlib

        g = self.grid
        torch = g.torch
        if self._comm is None:
            self._comm = torch.cuda.Stream(device=g.device)
        self._comm.wait_stream(g.stream)
        stack = contextlib.ExitStack()
        stack.enter_context(g._on())
        stack.enter_context(torch.cuda.stream(self._comm))
        return stack

    def comm_fence(self):
        """The next launch reads the received halo rows: main waits comm."""
        self.grid.stream.wait_stream(self._comm)

    def layers(self, buf, first, count):
        f = self.grid.fields[buf]
        return f[first * self.plane:(first + count) * self.plane]

    def norms(self, nsteps):
        return self.grid.norms[:2 * nsteps].clone()

    @property
    def owned_cells(self):
        lo, hi = self.grid.desc.own0_begin, self.grid.desc.own0_end
        return int(hi - lo) * int(np.prod(self.grid.shape[1:]))

    def download_owned(self, buf):
        """Owned rows of buffer ``buf`` as a host array (interior columns)."""
        lay = self.grid.layout
        u = np.empty(tuple(int(x) + 2 for x in self.grid.shape))
        self.grid.download_field(buf, u)
        lo, hi = self.grid.desc.own0_begin, self.grid.desc.own0_end
        inner = (slice(1, -1),) * (u.ndim - 1)
        return u[(slice(1 + lo, 1 + hi),) + inner]


class SlabGrid:
    """Benchmark/solver facade: one rank's slab with the DeviceGrid-like API
    (``run``, ``norms``, ``stream``) used by bench.py."""

    def __init__(self, fields, rank, world, fuse=4, group=None):
        import torch

        n0 = fields["source"].shape[0]
        self.fields = fields  # the global problem (host); the e2e bench re-uploads from it
        self.decomp = SlabDecomposition(n0, world, rank, halo=max(1, fuse))
        self.backend = DeviceSlab(fields, self.decomp)
        fuse = max(1, min(fuse, self.backend.max_fuse))
        self.solver = SlabSolver(self.backend, self.decomp, group=group, fuse=fuse)
        self.stream = self.backend.stream
        self._norms = None
        self.torch = torch

    @classmethod
    def weak_rows(cls, base, rank, world, fuse=4):
        """cfg2 weak scaling: stack ``world`` copies of the per-GPU row count
        into a (rows*world) x cols grid built with the same recipe."""
        from .problems import CONFIGS, poisson_fields

        n0, n1 = base["source"].shape
        cfg = CONFIGS["cfg2"]
        fields = poisson_fields((n0 * world, n1), cfg["n_gauss"], cfg["seed"], cfg["noise"],
                                cfg["width"])
        return cls(fields, rank, world, fuse=fuse)

    @property
    def owned_cells(self):
        return self.backend.owned_cells

    def run(self, cur, weights, first, nsteps, fuse=0):
        dst, norms = self.solver.run(cur, weights, first, nsteps)
        self._norms = norms
        return dst

    @property
    def norms(self):
        return self.torch.from_numpy(np.ascontiguousarray(self._norms).reshape(-1))
