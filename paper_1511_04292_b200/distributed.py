"""Slab (row-block) domain decomposition of the SRJ sweep across GPUs.

The reference has no parallel path (``SPEC.md:305`` lists distributed memory
as a non-goal; the paper only notes that SRJ keeps Jacobi's insensitivity to
domain decomposition, ``PAPER.md:78-80``).  This module is the multi-GPU
design of SURVEY.md section 8(e), one process per GPU:

* The global interior is split along axis 0 (slowest, C order) into
  contiguous blocks, one per rank (``SlabDecomposition``).  Each rank holds its
  owned rows plus ``halo`` >= fuse extra rows on every side with a neighbour,
  as interior rows of its local plan; the dependency cone of ``fuse`` sweeps
  shrinks one row per sweep, so the owned rows of a fused launch are exact.
* ``DeviceSlab`` runs a chunk of steps with ONE C call (``srj_slab_run``): per
  fused launch, the edge rows the neighbours need are relaxed first, copied
  into the neighbours' halo rows over NVLink (peer ``cudaMemcpyAsync`` into
  CUDA-IPC-mapped memory, on a side stream) while the inner rows are relaxed;
  the ranks order each other on the device with flag words in each other's
  memory (stream memory operations), so the host only enqueues work.
* Per-step (dmax, rmax) of owned rows are combined with one MAX all-reduce per
  chunk (exact), the relative-L2 rule with a SUM all-reduce of per-layer
  residuals (each layer owned by one rank) and an exactly rounded host sum, so
  every rank takes the same stopping decision and the N-GPU field, norms and
  iteration count are bitwise those of the 1-GPU solve (``srj_solve`` below).

``EmulatedRanks`` drives N slabs on one device through the same C exchange
(all work enqueued on one stream in dependency order): the 1-GPU test and
measurement harness of the multi-rank path.
"""

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["DeviceSlab", "DistComm", "EmulatedRanks", "SlabDecomposition", "SlabGrid",
           "SlabProblem", "jacobi_solve", "srj_solve"]


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
        the rest (None when the slab is all edge) -- the split srj_slab_run
        makes (edges relaxed and sent first, inner rows meanwhile)."""
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


def default_halo(ndim, fuse=0):
    """Fused depth the slab exchanges for: the plan default (2D 4, 3D 2)."""
    return int(fuse) if fuse else (4 if ndim == 2 else 2)


class SlabProblem:
    """One rank's rows of a global problem (FIXED faces, constant or per-cell
    coefficients, linear or nonlinear source) -- built from a global problem
    every rank holds (``from_global``) or generated rank-locally
    (``problems.slab_config_fields``), so no rank needs the global field.

    ``u``: ghosted local field (local interior rows = owned + halos, plus one
    layer beyond); ``source`` / ``kappa``, ``center``, ``lower``, ``upper``:
    local interior-shaped arrays (zero-stride broadcasts for constants)."""

    def __init__(self, decomp, global_shape, u, center, lower, upper, source=None, kappa=None,
                 mask=None):
        self.decomp = decomp
        self.global_shape = tuple(int(n) for n in global_shape)
        self.u = u
        self.source = source if source is not None else np.zeros(np.shape(center))
        self.kappa = kappa
        self.center, self.lower, self.upper = center, tuple(lower), tuple(upper)
        self.mask = mask
        if self.global_shape[0] != decomp.n0:
            raise ValueError("decomposition does not match the global shape")
        a, b = decomp.local_rows
        if tuple(np.shape(center)) != (b - a,) + self.global_shape[1:]:
            raise ValueError("local arrays do not match the decomposition")

    @property
    def ndim(self):
        return len(self.global_shape)

    @classmethod
    def from_global(cls, problem, decomp):
        """Slice a GridProblem-like object (FIXED faces, no post_sweep hook)."""
        for pair in getattr(problem, "bc", ()):
            for rule in pair:
                if rule.kind != "fixed":
                    raise NotImplementedError("the slab decomposition supports FIXED faces only")
        if getattr(problem, "post_sweep", None) is not None:
            raise NotImplementedError("post_sweep hooks need the whole grid on one GPU")
        shape = problem.source.shape
        sl = decomp.local_interior
        br = lambda a: sl(np.broadcast_to(a, shape))  # noqa: E731
        kappa = getattr(problem, "source_kappa", None)
        mask = getattr(problem, "mask", None)
        return cls(decomp, shape, decomp.local_field(problem.u), br(problem.center),
                   tuple(br(a) for a in problem.lower), tuple(br(a) for a in problem.upper),
                   source=sl(problem.source), kappa=None if kappa is None else sl(kappa),
                   mask=None if mask is None else sl(mask))

    def owned_source_sq(self):
        """Per owned layer sum of squares of the source (L2 rule reference)."""
        from .grids import layer_sum_squares

        lo, hi = self.decomp.own_local
        return layer_sum_squares(np.asarray(self.source)[lo:hi])


class DistComm:
    """MAX / SUM all-reduces of host arrays over a torch.distributed group
    (NCCL: staged through the rank's GPU; gloo: on the host)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        nccl = dist.get_backend(group) == "nccl"
        self.device = (device if device is not None else torch.device(
            "cuda", torch.cuda.current_device())) if nccl else torch.device("cpu")
        self.torch = torch

    def _reduce(self, a, op):
        t = self.torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)
        self.dist.all_reduce(t, op=op, group=self.group)
        return t.cpu().numpy()

    def max_(self, a):
        return self._reduce(a, self.dist.ReduceOp.MAX)

    def sum_(self, a):
        return self._reduce(a, self.dist.ReduceOp.SUM)

    def barrier(self):
        self.dist.barrier(group=self.group)

    def all_gather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


def agree_constant(slab, comm):
    """All ranks take the constant-stencil kernels only if every rank's rows
    allow it (a mask or varying coefficients elsewhere put every rank on the
    per-cell kernels, so all ranks fuse the same number of sweeps per launch
    and the exchange stays in step)."""
    from .engine import stencil_is_constant

    mine = stencil_is_constant(slab.center, slab.lower, slab.upper, slab.mask)
    if comm.world == 1:
        return mine
    return bool(-comm.max_(np.array([-float(mine)]))[0] > 0.5)


def agree_depth(backend, comm, fuse):
    """The fused depth every rank runs: the minimum of the ranks' own depths
    (a plan's default depends on its local size and coefficient mode)."""
    mine = backend.depth(fuse)
    if comm.world == 1:
        return mine
    return int(round(-comm.max_(np.array([-float(mine)]))[0]))


class DeviceSlab:
    """One rank's slab on its GPU: a pooled ``DeviceGrid`` (three fields +
    flag words in one allocation) and the C slab exchange (``srj_slab_*``)."""

    def __init__(self, slab, device=None, allow_constant=True):
        from .engine import DeviceGrid

        d = slab.decomp
        self.decomp = d
        self.problem = slab
        self.grid = DeviceGrid(slab.u, slab.source, slab.center, slab.lower, slab.upper,
                               active=slab.mask, kappa=slab.kappa, own=d.own_local,
                               device=device, pooled=True, allow_constant=allow_constant)
        g = self.grid
        self.lib = g.lib
        self.stream = g.stream
        self.n_layers = d.n0
        self.layer0 = d.owned[0]
        self._opened = []
        bufs = (ctypes.c_void_p * 3)(*[f.data_ptr() for f in g.fields])
        self.handle = ctypes.c_void_p()
        with g._on():
            _lib.check(self.lib.srj_slab_create(
                ctypes.byref(g.desc), int(d.halo), bufs, ctypes.c_void_p(g.flags.data_ptr()),
                int(d.rank > 0), int(d.rank < d.world - 1), ctypes.byref(self.handle)),
                "srj_slab_create")
        self._peer_ptrs = None

    # ---------------------------------------------------------------- wiring
    def _peer_struct(self, bufs, flags, dst_row):
        p = _lib.SrjSlabPeer()
        for i in range(3):
            p.bufs[i] = bufs[i]
        p.flags = flags
        p.dst_row = int(dst_row)
        return p

    def connect_local(self, lower=None, upper=None):
        """Neighbours in the same process on the same device (emulated ranks)."""
        for side, nb in ((0, lower), (1, upper)):
            if nb is None:
                continue
            dst_row = nb.decomp.own_local[1] if side == 0 else 0
            p = self._peer_struct([f.data_ptr() for f in nb.grid.fields],
                                  nb.grid.flags.data_ptr(), dst_row)
            _lib.check(self.lib.srj_slab_connect(self.handle, side, ctypes.byref(p)),
                       "srj_slab_connect")

    def connect(self, comm):
        """Map the neighbours' pooled buffers through CUDA IPC (one process per
        GPU) and wire the exchange; then reset the flags on every rank."""
        g = self.grid
        h = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        with g._on():
            _lib.check(self.lib.srj_ipc_get_handle(ctypes.c_void_p(g.pool.data_ptr()), h,
                                                   ctypes.byref(off)), "srj_ipc_get_handle")
        elems = int(g.layout.elems)
        info = {"handle": h.raw, "offset": off.value, "elems": elems,
                "own_e": self.decomp.own_local[1], "rank": self.decomp.rank}
        infos = comm.all_gather_object(info)
        r = self.decomp.rank
        for side, peer in ((0, r - 1), (1, r + 1)):
            if not 0 <= peer < self.decomp.world:
                continue
            pi = infos[peer]
            ptr = ctypes.c_void_p()
            with g._on():
                _lib.check(self.lib.srj_ipc_open(pi["handle"], int(pi["offset"]),
                                                 ctypes.byref(ptr)), "srj_ipc_open")
            self._opened.append(int(ptr.value) - int(pi["offset"]))
            base = int(ptr.value)
            bufs = [base + 8 * i * pi["elems"] for i in range(3)]
            flags = base + 8 * 3 * pi["elems"]
            dst_row = pi["own_e"] if side == 0 else 0
            p = self._peer_struct(bufs, flags, dst_row)
            _lib.check(self.lib.srj_slab_connect(self.handle, side, ctypes.byref(p)),
                       "srj_slab_connect")
        self.reset()
        comm.barrier()

    def reset(self):
        g = self.grid
        with g._on():
            _lib.check(self.lib.srj_slab_reset(self.handle, g._sp), "srj_slab_reset")
        g.stream.synchronize()

    # --------------------------------------------------------------- running
    def run_chunk(self, src, weights, first, n, fuse=0):
        return run_slabs([self], src, weights, first, n, fuse)

    def depth(self, fuse=0):
        """Sweeps per fused launch this rank's plan would run for ``fuse``
        (0 = its default), capped by the halo (``srj_slab_depth``)."""
        rc = self.lib.srj_slab_depth(self.handle, int(fuse))
        if rc < 1:
            _lib.check(rc if rc < 0 else -1, "srj_slab_depth")
        return int(rc)

    def direct(self, fuse=0):
        """True when ``run_chunk`` takes the direct data path: one launch per
        fused step whose kernel stores the edge rows into the neighbours'
        halos (``srj_slab_direct``, include/srj.h)."""
        rc = self.lib.srj_slab_direct(self.handle, int(fuse))
        if rc < 0:
            _lib.check(rc, "srj_slab_direct")
        return rc == 1

    def norms(self, n):
        return self.grid.norms[:2 * n].view(n, 2).cpu().numpy()

    def residual_layers(self, buf):
        return self.grid.residual_layers(buf)

    def download_owned(self, buf):
        """Owned rows of buffer ``buf`` as a host array (interior columns)."""
        u = np.empty(tuple(int(x) + 2 for x in self.grid.shape))
        self.grid.download_field(buf, u)
        lo, hi = self.decomp.own_local
        inner = (slice(1, -1),) * (u.ndim - 1)
        return u[(slice(1 + lo, 1 + hi),) + inner]

    @property
    def owned_cells(self):
        lo, hi = self.decomp.own_local
        return int(hi - lo) * int(np.prod(self.grid.shape[1:]))

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            with self.grid._on():
                self.lib.srj_slab_destroy(self.handle)
                for base in self._opened:
                    self.lib.srj_ipc_close(ctypes.c_void_p(base))
            self.handle = None
            self._opened = []
        self.grid.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_slabs(slabs, src, weights, first, n, fuse=0):
    """One srj_slab_run over ``slabs`` (1 = this process's rank; more = ranks
    emulated on one device, enqueued on the first slab's stream)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    k = len(slabs)
    for s in slabs:
        s.grid.ensure_norms(max(n, 1))
    handles = (ctypes.c_void_p * k)(*[s.handle.value for s in slabs])
    norms = (ctypes.c_void_p * k)(*[s.grid.norms.data_ptr() for s in slabs])
    streams = (ctypes.c_void_p * k)(*[s.stream.cuda_stream for s in slabs])
    out = ctypes.c_int32(0)
    with slabs[0].grid._on():
        _lib.check(slabs[0].lib.srj_slab_run(
            handles, k, int(src), w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(w),
            int(first), int(n), int(fuse), norms, ctypes.byref(out), streams), "srj_slab_run")
    return int(out.value)


class EmulatedRanks:
    """``world`` ranks of a slab decomposition on ONE device in one process,
    exchanging through the same C path (``srj_slab_run`` with all slabs, one
    stream; ``concurrent=True``: one stream per rank, so the flag protocol
    orders truly asynchronous ranks); the backend interface of
    ``solver.run_solve`` with the rank combination done here (use
    ``solver.LocalComm``)."""

    def __init__(self, problem, world, fuse=0, device=None, concurrent=False):
        nd = problem.source.ndim
        halo = default_halo(nd, fuse)
        n0 = problem.source.shape[0]
        self.decomps = [SlabDecomposition(n0, world, r, halo) for r in range(world)]
        self.concurrent = bool(concurrent)
        from .engine import stencil_is_constant

        locals_ = [SlabProblem.from_global(problem, d) for d in self.decomps]
        const = all(stencil_is_constant(s.center, s.lower, s.upper, s.mask) for s in locals_)
        if concurrent:
            # one stream per emulated rank: launches, peer copies and flag
            # operations of different ranks race exactly as between processes
            import torch

            self.slabs = []
            for sp in locals_:
                with torch.cuda.stream(torch.cuda.Stream(device)):
                    self.slabs.append(DeviceSlab(sp, device, allow_constant=const))
        else:
            self.slabs = [DeviceSlab(sp, device, allow_constant=const) for sp in locals_]
        for r, s in enumerate(self.slabs):
            s.connect_local(self.slabs[r - 1] if r > 0 else None,
                            self.slabs[r + 1] if r + 1 < world else None)
        for s in self.slabs:
            s.reset()
        self.n_layers = n0
        self.layer0 = 0
        self.stream = self.slabs[0].stream

    def run_chunk(self, src, weights, first, n, fuse=0):
        return run_slabs(self.slabs, src, weights, first, n, fuse)

    def _sync(self):
        if self.concurrent:
            for s in self.slabs:
                s.stream.synchronize()

    def _each(self, fn):
        """fn(slab) per rank, on that rank's stream (device reads included)."""
        if not self.concurrent:
            return [fn(s) for s in self.slabs]
        import torch

        self._sync()
        out = []
        for s in self.slabs:
            with torch.cuda.stream(s.stream):
                out.append(fn(s))
        return out

    def norms(self, n):
        return np.max(self._each(lambda s: s.norms(n)), axis=0)

    def residual_layers(self, buf):
        return np.concatenate(self._each(lambda s: s.residual_layers(buf)))

    def download_owned(self, buf):
        return np.concatenate(self._each(lambda s: s.download_owned(buf)))

    def close(self):
        self._sync()
        for s in self.slabs:
            s.close()


def _comm_for(group):
    import torch.distributed as dist

    from .solver import LocalComm

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        return DistComm(group)
    return LocalComm


def _solve(problem, weights, tol, max_iters, normalise, stop, check_every, fuse, chunk,
           l2_reference, group, gather, device):
    from . import grids as G
    from .solver import l2_from_layers, run_solve, source_l2

    comm = _comm_for(group)
    if isinstance(problem, SlabProblem):
        slab = problem
        if slab.decomp.world != comm.world or slab.decomp.rank != comm.rank:
            raise ValueError("SlabProblem decomposition does not match the process group")
    else:
        nd = problem.source.ndim
        d = SlabDecomposition(problem.source.shape[0], comm.world, comm.rank,
                              default_halo(nd, fuse))
        slab = SlabProblem.from_global(problem, d)
    backend = DeviceSlab(slab, device, allow_constant=agree_constant(slab, comm))
    try:
        if comm.world > 1:
            backend.connect(comm)
        else:
            backend.reset()
        fuse = agree_depth(backend, comm, fuse)
        if stop == "residual_l2" and l2_reference is None:
            if slab.kappa is not None:
                l2_reference = lambda: l2_from_layers(  # noqa: E731 - residual of u0
                    backend, comm, backend.residual_layers(0))[0]
            else:
                l2_reference = source_l2(backend, comm, slab.owned_source_sq())
        hist, converged, diverged, cur = run_solve(
            backend, comm, weights, tol, max_iters, normalise, stop, check_every, fuse, chunk,
            l2_reference, int(np.prod(slab.global_shape)))
        owned = backend.download_owned(cur)
    finally:
        backend.close()
    out = G._history(hist, float(tol), converged)
    if gather and not isinstance(problem, SlabProblem):
        parts = comm.all_gather_object(owned) if comm.world > 1 else [owned]
        inner = (slice(1, -1),) * (problem.u.ndim - 1)
        problem.u[(slice(1, 1 + problem.source.shape[0]),) + inner] = np.concatenate(parts)
    G._raise_if_diverged(out, diverged)
    return out, owned


def srj_solve(problem, cycle, tol, max_iters=10_000_000, *, group=None, stop="update_inf",
              check_every=None, fuse=0, chunk=None, l2_reference=None, gather=False,
              device=None):
    """``grids.srj_solve`` (reference ``grids.py:642-687``) over the ranks of
    a process group, one GPU per rank.

    ``problem``: a global GridProblem (FIXED faces) that every rank holds, or
    this rank's ``SlabProblem``.  Returns (history, owned interior rows of this
    rank); ``gather=True`` also writes the whole interior into ``problem.u`` on
    every rank.  History, iteration count and field are bitwise those of the
    single-GPU ``grids.srj_solve`` under both stopping rules; a
    ``DivergenceError`` is raised on every rank at the same step."""
    return _solve(problem, cycle.weight_sequence, tol, max_iters, True, stop, check_every, fuse,
                  chunk, l2_reference, group, gather, device)


def jacobi_solve(problem, tol, max_iters=10_000_000, *, group=None, stop="update_inf",
                 check_every=None, fuse=0, chunk=None, l2_reference=None, gather=False,
                 device=None):
    """``grids.jacobi_solve`` (``grids.py:690-694``, omega = 1) over ranks."""
    return _solve(problem, np.ones(1), tol, max_iters, False, stop, check_every, fuse, chunk,
                  l2_reference, group, gather, device)


class SlabGrid:
    """Benchmark facade: this rank's slab with the DeviceGrid-like API
    (``run``, ``norms``, ``stream``) used by bench.py; per-step norms are
    MAX-reduced over the group once per ``run``."""

    def __init__(self, slab, comm=None, device=None):
        from .solver import LocalComm

        self.comm = comm or LocalComm
        self.decomp = slab.decomp
        self.problem = slab
        self.backend = DeviceSlab(slab, device, allow_constant=agree_constant(slab, self.comm))
        if self.comm.world > 1:
            self.backend.connect(self.comm)
        else:
            self.backend.reset()
        self._depths = {}
        self.stream = self.backend.stream
        self._norms = None

    @property
    def owned_cells(self):
        return self.backend.owned_cells

    def run(self, cur, weights, first, nsteps, fuse=0):
        if fuse not in self._depths:  # one all-reduce per distinct request
            self._depths[fuse] = agree_depth(self.backend, self.comm, fuse)
        dst = self.backend.run_chunk(cur, weights, first, nsteps, self._depths[fuse])
        self._norms = self.comm.max_(self.backend.norms(nsteps))
        return dst

    @property
    def norms(self):
        import torch

        return torch.from_numpy(np.ascontiguousarray(self._norms).reshape(-1))

    def close(self):
        self.backend.close()
