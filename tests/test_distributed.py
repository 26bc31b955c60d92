"""Slab decomposition host logic on CPU: world_size 2 and 3 over gloo.

The GPU kernels are replaced by the oracle (numpy restatement, bitwise equal
to the reference) behind the same SlabBackend interface, so this checks the
decomposition, halo exchange and norm all-reduce of distributed.SlabSolver:
the gathered k-rank field and per-step norms must equal the single-process
oracle bit for bit.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1511_04292_b200.distributed import SlabDecomposition, SlabSolver
from paper_1511_04292_b200.problems import config_fields, nonlinear_fields
from paper_1511_04292_b200.schedule import quantize
from paper_1511_04292_b200.tables import shipped_table


class _P:
    """Problem-like view for the oracle."""

    def __init__(self, u, source, center, lower, upper, mask=None):
        self.u, self.source, self.center = u, source, center
        self.lower, self.upper = lower, upper
        self._active = mask


class OracleSlab:
    """CPU stand-in for DeviceSlab: three dense ghosted buffers per rank."""

    def __init__(self, fields, d):
        sl = d.local_interior
        u = np.ascontiguousarray(d.local_field(fields["u"]), dtype=np.float64)
        self.bufs = [u.copy() for _ in range(3)]
        self.src = np.ascontiguousarray(sl(fields["source"]))
        self.c = np.ascontiguousarray(sl(np.broadcast_to(fields["center"], fields["source"].shape)))
        self.lo = tuple(np.ascontiguousarray(sl(np.broadcast_to(a, fields["source"].shape)))
                        for a in fields["lower"])
        self.hi = tuple(np.ascontiguousarray(sl(np.broadcast_to(a, fields["source"].shape)))
                        for a in fields["upper"])
        k = fields.get("kappa")
        self.kappa = None if k is None else np.ascontiguousarray(sl(k))
        self.own = d.own_local
        self.first_part = d.row_parts()[0][0]
        self.normbuf = torch.zeros(2)

    def reserve(self, n):
        self.normbuf = torch.zeros(2 * n, dtype=torch.float64)

    def run(self, src, dst, weights, first, nsteps, off, rows=None):
        if rows is None:
            self.bufs[dst][...] = self.bufs[src]
            work, own = self.bufs[dst], self.own
        else:  # edge / inner part: relax a copy, store only rows [a, b)
            work, own = self.bufs[src].copy(), rows
        for s in range(nsteps):
            p = _P(work, self.src, self.c, self.lo, self.hi)
            w = weights[(first + s) % len(weights)]
            dm, rm = oracle.np_step(p, w, kappa=self.kappa, own_rows=own)
            i = 2 * (off + s)
            if rows is not None and rows != self.first_part:
                dm, rm = max(dm, float(self.normbuf[i])), max(rm, float(self.normbuf[i + 1]))
            self.normbuf[i] = dm
            self.normbuf[i + 1] = rm
        if rows is not None:
            a, b = rows
            self.bufs[dst][1 + a:1 + b] = work[1 + a:1 + b]

    def comm(self):
        import contextlib

        return contextlib.nullcontext()

    def comm_fence(self):
        pass

    def layers(self, buf, first, count):
        return torch.from_numpy(self.bufs[buf][first:first + count])

    def norms(self, n):
        return self.normbuf[:2 * n].clone()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, out_q, overlap=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fields, w, steps, fuse = case()
        d = SlabDecomposition(fields["source"].shape[0], world, rank, halo=fuse)
        solver = SlabSolver(OracleSlab(fields, d), d, fuse=fuse, overlap=overlap)
        assert solver.overlap == (world > 1 and overlap is not False)
        cur, allnorms, done = 0, [], 0
        for chunk in (steps // 3, steps - steps // 3):  # two chunks, snapshot rotation
            cur, norms = solver.run(cur, w, done, chunk)
            allnorms.append(norms)
            done += chunk
        lo, hi = d.own_local
        owned = solver.b.bufs[cur][1 + lo:1 + hi].copy()
        out_q.put((rank, owned, np.concatenate(allnorms)))
    finally:
        dist.destroy_process_group()


def case_2d():
    f = config_fields("cfg2", (41, 37))
    w = quantize(shipped_table().get(6, 64)).weight_sequence
    return f, w, 60, 3


def case_3d():
    f = config_fields("cfg3", (13, 9, 11))
    w = quantize(shipped_table().get(6, 64)).weight_sequence
    return f, w, 40, 1


def case_nl():
    f = nonlinear_fields((40, 36), seed=5)
    w = quantize(shipped_table().get(8, 32)).weight_sequence
    return f, w, 50, 2


def reference(case):
    f, w, steps, _ = case()
    from helpers import problem_from

    p = problem_from(f)
    done, _, norms = oracle.run(p, w, 0, steps, kappa=f.get("kappa"))
    return p.u, norms


@pytest.mark.parametrize("overlap", [None, False])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", [case_2d, case_3d, case_nl])
def test_slab_solver_matches_single_process(world, case, overlap):
    """overlap=None: the default edge / inner split with the exchange posted
    between the two (SlabSolver.overlap); False: one launch then exchange."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    results = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u_ref, norms_ref = reference(case)
    got = np.concatenate([r[1] for r in results])
    assert np.array_equal(got, u_ref[1:-1])
    for _, _, norms in results:
        assert np.array_equal(norms, norms_ref)


def test_decomposition_ranges():
    d = [SlabDecomposition(10, 3, r, halo=2) for r in range(3)]
    assert [x.owned for x in d] == [(0, 4), (4, 7), (7, 10)]
    assert d[0].local_rows == (0, 6) and d[1].local_rows == (2, 9) and d[2].local_rows == (5, 10)
    assert d[1].sends() == [(0, 3, 2), (2, 4, 2)]
    assert d[1].recvs() == [(0, 1, 2), (2, 6, 2)]
    with pytest.raises(ValueError):
        SlabDecomposition(5, 3, 0, halo=2)
    # edge / inner split (local interior rows)
    assert d[0].row_parts() == ([(2, 4)], (0, 2))
    assert d[1].row_parts() == ([(2, 5)], None)  # thinner than two halos: all edge
    assert d[2].row_parts() == ([(2, 4)], (4, 5))
    e = [SlabDecomposition(40, 3, r, halo=3) for r in range(3)]
    assert e[0].row_parts() == ([(11, 14)], (0, 11))
    assert e[1].row_parts() == ([(3, 6), (13, 16)], (6, 13))
    assert e[2].row_parts() == ([(3, 6)], (6, 16))


def test_overlap_schedule_order(monkeypatch):
    """The overlapped launch order (SlabSolver.overlap): edge rows, exchange
    posted on the comm context, inner rows, wait + fence -- recorded on a stub
    backend (no process group needed)."""
    import contextlib

    log = []

    class Stub:
        def reserve(self, n):
            self.n = n

        def run(self, src, dst, weights, first, nsteps, off, rows=None):
            log.append(("run", rows))

        def layers(self, buf, first, count):
            return torch.zeros(1)

        def norms(self, n):
            return torch.zeros(2 * n, dtype=torch.float64)

        @contextlib.contextmanager
        def comm(self):
            log.append(("comm",))
            yield

        def comm_fence(self):
            log.append(("fence",))

    class Req:
        def wait(self):
            log.append(("wait",))

    d = SlabDecomposition(40, 3, 1, halo=3)
    solver = SlabSolver(Stub(), d, fuse=3)
    assert solver.overlap
    monkeypatch.setattr(solver, "_post_exchange", lambda buf: log.append(("post",)) or [Req()])
    monkeypatch.setattr(dist, "all_reduce", lambda *a, **k: None)
    solver.run(0, np.array([1.0]), 0, 3)
    assert log == [("run", (3, 6)), ("run", (13, 16)), ("comm",), ("post",), ("run", (6, 13)),
                   ("comm",), ("wait",), ("fence",)]
    monkeypatch.setenv("SRJ_SLAB_OVERLAP", "0")
    assert not SlabSolver(Stub(), d, fuse=3).overlap
