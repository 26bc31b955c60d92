"""Drop-in replacement for the reference's ``srj.grids`` solver entry points.

Same names, arguments, return values and exceptions as
``/root/reference/pkg/src/srj/grids.py``; the sweeps run on the GPU through
libsrj.so (``include/srj.h``).  Inputs are the reference's own objects or this
module's look-alikes: any object with the ``GridProblem`` attributes
(``u``, ``source``, ``center``, ``lower``, ``upper``, ``bc``, ``mask`` /
``_active``, ``post_sweep``) and any cycle with ``weight_sequence``.

GPU scope: 1-D, 2-D 5-point and 3-D 7-point stencils with
every reference boundary rule (FIXED, mirror and face-Dirichlet faces run
fused multi-sweep kernels; periodic faces run one sweep per launch; a device
ghost refresh follows every launch),
constant or per-cell coefficients, optional mask,
optional nonlinear source, ``post_sweep`` hooks that copy field values (e.g.
the spherical ``tie_origin``; applied on the device as a gather after every
sweep, ``post_sweep_gather``), and Gauss-Seidel / SOR as a bitwise GPU
wavefront (``srj_plan_gs``).  1-D grids (``_wj1``) run as 1 x n 2-D grids
(``_LineGrid``).  Hooks that compute values raise ``NotImplementedError`` --
there is no CPU fallback.

Entry points and the reference code they replace:

* ``weighted_jacobi_sweep`` -- ``grids.py:574-599``
* ``srj_solve``             -- ``grids.py:642-687`` (+ ``_iterate`` ``:602-629``)
* ``jacobi_solve``          -- ``grids.py:690-694``
* ``GridProblem``, ``BoundaryRule``, ``ResidualHistory``, ``DivergenceError``
  -- ``grids.py:56-321`` (host-side types, same validation messages).

Stopping rules.  ``stop="update_inf"`` (default) is the reference's: after
every elementary step the update infinity norm divided by |omega| is compared
with ``tol`` (``grids.py:684``, ``:626``) and an overflow guard raises
``DivergenceError`` (``:618-625``).  The GPU evaluates both per step from a
device norm buffer that the host reads once per chunk; when the rule fires
inside a chunk, the chunk is replayed from its start snapshot to the exact
step, so iteration counts, histories and the returned field are those of the
reference.  ``stop="residual_l2"`` is the BASELINE's relative-L2 rule
||s - A u||_2 / ||s||_2 < tol checked every ``check_every`` steps (default one
M-cycle) with the fused residual kernel; it is an addition, not in the
reference.
"""

import time
from dataclasses import dataclass, field

import numpy as np

from .engine import DeviceGrid

__all__ = [
    "OVERFLOW_LIMIT",
    "FIXED",
    "MIRROR",
    "PERIODIC",
    "BoundaryRule",
    "DivergenceError",
    "GridProblem",
    "ResidualHistory",
    "face_dirichlet",
    "gauss_seidel_solve",
    "jacobi_solve",
    "sor_solve",
    "srj_solve",
    "weighted_jacobi_sweep",
]

OVERFLOW_LIMIT = 1e300  # grids.py:53


class DivergenceError(RuntimeError):
    """Non-finite or overflowing update (``grids.py:56-70``)."""

    def __init__(self, message, iterations, history):
        super().__init__(message)
        self.iterations = iterations
        self.history = history


_KINDS = ("fixed", "mirror", "periodic", "face_dirichlet")


@dataclass(frozen=True)
class BoundaryRule:
    """Per-face ghost rule (``grids.py:73-102``)."""

    kind: str
    values: np.ndarray | None = None

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ValueError(f"unknown boundary kind {self.kind!r}")
        if self.kind == "face_dirichlet" and self.values is None:
            raise ValueError("face_dirichlet rule needs boundary values")


FIXED = BoundaryRule("fixed")
MIRROR = BoundaryRule("mirror")
PERIODIC = BoundaryRule("periodic")


def face_dirichlet(values):
    return BoundaryRule("face_dirichlet", np.asarray(values, dtype=float))


def _face(nd, axis, pos):
    sl = [slice(1, -1)] * nd
    sl[axis] = pos
    return tuple(sl)


@dataclass
class GridProblem:
    """One discretised elliptic problem (``grids.py:122-281``).

    Extension (not in the reference): ``source_kappa`` -- when given, the
    source is the nonlinear s(u) = source_kappa * u^5 re-evaluated from the
    current iterate in every sweep, and
    ``source`` is ignored by the solvers.
    """

    spacing: tuple
    u: np.ndarray
    source: np.ndarray
    center: np.ndarray
    lower: tuple
    upper: tuple
    bc: tuple
    mask: np.ndarray | None = None
    post_sweep: object = None
    description: str = ""
    source_kappa: np.ndarray | None = None
    _active: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        self.u = np.asarray(self.u, dtype=float)
        self.source = np.asarray(self.source, dtype=float)
        self.center = np.asarray(self.center, dtype=float)
        nd = self.source.ndim
        if nd < 1 or nd > 3:
            raise ValueError("only 1-, 2- and 3-dimensional grids are supported")
        self.spacing = tuple(float(h) for h in self.spacing)
        if len(self.spacing) != nd:
            raise ValueError("spacing must provide one value per axis")
        shape = self.source.shape
        if self.u.shape != tuple(s + 2 for s in shape):
            raise ValueError(
                f"field shape {self.u.shape} does not match interior {shape} plus ghosts")
        if self.center.shape != shape:
            raise ValueError("center coefficients must have the interior shape")
        self.lower = tuple(np.asarray(a, dtype=float) for a in self.lower)
        self.upper = tuple(np.asarray(a, dtype=float) for a in self.upper)
        if len(self.lower) != nd or len(self.upper) != nd:
            raise ValueError("lower/upper must provide one array per axis")
        if any(a.shape != shape for a in self.lower + self.upper):
            raise ValueError("neighbor coefficients must have the interior shape")
        self.bc = tuple(tuple(pair) for pair in self.bc)
        if len(self.bc) != nd:
            raise ValueError("bc must provide one (low, high) pair per axis")
        for lo, hi in self.bc:
            if (lo.kind == "periodic") != (hi.kind == "periodic"):
                raise ValueError("periodic axes need the rule on both faces")
        if self.mask is not None:
            self.mask = np.asarray(self.mask, dtype=bool)
            if self.mask.shape != shape:
                raise ValueError("mask must have the interior shape")
            self._active = self.mask
        else:
            self._active = np.broadcast_to(np.True_, shape)
        if self.source_kappa is not None:
            self.source_kappa = np.asarray(self.source_kappa, dtype=float)
            if self.source_kappa.shape != shape:
                raise ValueError("source_kappa must have the interior shape")
        if self.mask is None:
            bad = bool(np.any(self.center == 0.0))
        else:
            bad = not bool(np.all(self.center[self._active] != 0.0))
        if bad:
            raise ValueError("center coefficient vanishes on an active cell")
        self.refresh_ghosts()

    @property
    def ndim(self):
        return self.source.ndim

    @property
    def shape(self):
        return self.source.shape

    @property
    def interior(self):
        return self.u[(slice(1, -1),) * self.ndim]

    def refresh_ghosts(self):
        """Host ghost refresh (``grids.py:225-247``)."""
        u = self.u
        nd = self.ndim
        for ax in range(nd):
            last = u.shape[ax] - 1
            for rule, ghost, inner, wrap in ((self.bc[ax][0], 0, 1, last - 1),
                                             (self.bc[ax][1], last, last - 1, 1)):
                if rule.kind == "mirror":
                    u[_face(nd, ax, ghost)] = u[_face(nd, ax, inner)]
                elif rule.kind == "periodic":
                    u[_face(nd, ax, ghost)] = u[_face(nd, ax, wrap)]
                elif rule.kind == "face_dirichlet":
                    u[_face(nd, ax, ghost)] = 2.0 * rule.values - u[_face(nd, ax, inner)]
        if self.post_sweep is not None:
            self.post_sweep(u)

    def operator_apply(self):
        u = self.u
        nd = self.ndim
        core = (slice(1, -1),) * nd
        acc = self.center * u[core]
        for ax in range(nd):
            lo = list(core)
            hi = list(core)
            lo[ax] = slice(0, -2)
            hi[ax] = slice(2, None)
            acc = acc + self.lower[ax] * u[tuple(lo)]
            acc = acc + self.upper[ax] * u[tuple(hi)]
        return acc

    def residual_field(self):
        if self.source_kappa is not None:
            uc = self.interior
            p2 = uc * uc
            return self.source_kappa * ((p2 * p2) * uc) - self.operator_apply()
        return self.source - self.operator_apply()

    def copy(self):
        return GridProblem(
            spacing=self.spacing, u=self.u.copy(), source=self.source.copy(),
            center=self.center.copy(), lower=tuple(a.copy() for a in self.lower),
            upper=tuple(a.copy() for a in self.upper), bc=self.bc,
            mask=None if self.mask is None else self.mask.copy(),
            post_sweep=self.post_sweep, description=self.description,
            source_kappa=None if self.source_kappa is None else self.source_kappa.copy())


@dataclass
class ResidualHistory:
    """Per-step convergence record (``grids.py:284-321``).

    Extension: ``relative_l2`` holds (step, ||r||_2/||s||_2) pairs of the
    residual-L2 stopping rule's check points (empty for the reference rule).
    """

    residual_inf: np.ndarray
    true_residual_inf: np.ndarray
    seconds: np.ndarray
    tolerance: float
    converged: bool
    relative_l2: np.ndarray = field(default_factory=lambda: np.zeros((0, 2)))

    @property
    def iterations(self):
        return len(self.residual_inf)

    def to_csv(self, path, timing=True):
        rows = ["iteration,residual_inf,wall_seconds"]
        for k in range(self.iterations):
            sec = self.seconds[k] if timing else 0.0
            rows.append(f"{k + 1},{self.residual_inf[k]:.17g},{sec:.6f}")
        with open(path, "w") as fh:
            fh.write("\n".join(rows) + "\n")


# --------------------------------------------------------------------- GPU
class _LineGrid(DeviceGrid):
    """A 1-D problem (reference kernel ``_wj1``, ``grids.py:331-348``) staged as
    a 1 x n two-dimensional grid: the line is the grid's single last-axis row,
    the axis-0 neighbour coefficients are zero and the two extra ghost rows
    hold zeros, so every product they add is +0.0 and the 5-point residual
    ``s - ((((c*u + 0) + 0) + am*u[i-1]) + ap*u[i+1])`` equals ``_wj1``'s
    ``s - ((c*u + am*u[i-1]) + ap*u[i+1])`` in every nonzero value (a zero can
    differ in sign only, which no later operation of the sweep can turn into
    a different value)."""

    def download_field(self, idx, host):
        if host.ndim == 1:
            tmp = np.empty((3, host.shape[0]))
            super().download_field(idx, tmp)
            host[...] = tmp[1]
            return
        super().download_field(idx, host)


def _lift_line(problem, active, kappa, gather):
    """Arguments of a ``_LineGrid`` for a 1-D problem."""
    n = problem.source.shape[0]
    u = np.zeros((3, n + 2))
    u[1] = problem.u
    row = lambda a: None if a is None else np.asarray(a)[None, :]  # noqa: E731
    zeros = np.zeros((1, n))
    if gather is not None:
        gather = tuple(np.asarray(g, dtype=np.int64) + (n + 2) for g in gather)
    return dict(u=u, source=row(problem.source), center=row(problem.center),
                lower=(zeros, row(problem.lower[0])), upper=(zeros, row(problem.upper[0])),
                active=row(active), kappa=row(kappa), bc=((FIXED, FIXED), tuple(problem.bc[0])),
                post_gather=gather)


def _device_grid(problem):
    """Validate the GPU scope and stage the problem on the device."""
    nd = problem.source.ndim
    if nd not in (1, 2, 3):
        raise NotImplementedError("the GPU path supports 1-, 2- and 3-dimensional grids")
    for pair in problem.bc:
        for rule in pair:
            if rule.kind not in ("fixed", "mirror", "periodic", "face_dirichlet"):
                raise NotImplementedError(f"boundary kind {rule.kind!r} is not on the GPU path")
    gather = None
    if getattr(problem, "post_sweep", None) is not None:
        gather = post_sweep_gather(problem.post_sweep, problem.u.shape)
    active = getattr(problem, "_active", None)
    if active is None:
        active = getattr(problem, "mask", None)
    kappa = getattr(problem, "source_kappa", None)
    if nd == 1:
        return _LineGrid(**_lift_line(problem, active, kappa, gather))
    return DeviceGrid(problem.u, problem.source, problem.center, problem.lower,
                      problem.upper, active=active, kappa=kappa, bc=problem.bc,
                      post_gather=gather)


def post_sweep_gather(hook, shape):
    """Express a ``post_sweep`` hook (``grids.py:146-163``, called at the end
    of ``refresh_ghosts`` :246-247) as a gather ``u[dst] = u[src]`` with
    simultaneous semantics, so the device can apply it after every sweep.

    The hook is probed on copies of the ghosted field: two arrays of unique
    values (identity and a random permutation) must agree on which flat
    positions change and which position each new value came from, and a
    random-valued array must then be reproduced exactly by that gather, so a
    hook that computes (rather than copies) values is rejected.  Returns
    (dst, src) int64 flat indices; raises ``NotImplementedError`` otherwise.
    E.g. the spherical ``tie_origin`` (``problems.py:586-589``).
    """
    shape = tuple(int(n) for n in shape)
    n = int(np.prod(shape))
    if n >= 2 ** 52:
        raise NotImplementedError("field too large to probe the post_sweep hook")
    rng = np.random.default_rng(1234)
    maps = []
    for perm in (np.arange(n), rng.permutation(n)):
        a = perm.astype(np.float64).reshape(shape)
        try:
            hook(a)
        except Exception as exc:  # noqa: BLE001 - any failure means "not a gather"
            raise NotImplementedError(f"post_sweep hook could not be probed: {exc}") from exc
        flat = a.reshape(-1)
        dst = np.flatnonzero(flat != perm)
        vals = flat[dst]
        if not (np.all(vals == np.rint(vals)) and np.all((vals >= 0) & (vals < n))):
            raise NotImplementedError("post_sweep hook is not a copy of field values")
        inv = np.empty(n, dtype=np.int64)
        inv[perm] = np.arange(n)
        maps.append((dst.astype(np.int64), inv[vals.astype(np.int64)]))
    (d0, s0), (d1, s1) = maps
    if not (np.array_equal(d0, d1) and np.array_equal(s0, s1)):
        raise NotImplementedError("post_sweep hook is not a fixed gather of field values")
    x = rng.standard_normal(shape)
    want = x.copy()
    hook(want)
    got = x.copy().reshape(-1)
    got[d0] = x.reshape(-1)[s0]
    if not np.array_equal(got.reshape(shape), want):
        raise NotImplementedError("post_sweep hook is not a fixed gather of field values")
    return d0, s0


def _step_seconds_estimate(problem):
    cells = int(np.prod(problem.source.shape))
    return 3e-6 + cells * 24.0 / 5e12


def weighted_jacobi_sweep(problem, omega, traversal="forward"):
    """One weighted Jacobi step on the GPU (``grids.py:574-599``)."""
    if traversal not in ("forward", "reverse"):
        raise ValueError("traversal must be 'forward' or 'reverse'")
    dev = _device_grid(problem)
    try:
        out = dev.run(0, np.array([float(omega)]), 0, 1, fuse=1)
        norms = dev.norms[:2].cpu().numpy()
        dev.download_field(out, problem.u)  # ghosts refreshed on the device
    finally:
        dev.close()
    return float(norms[0]), float(norms[1])


def layer_sum_squares(a):
    """Per axis-0 layer sum of squares (numpy pairwise, a function of the
    layer's values only): the L2 rule's reference norm ||source||_2 is the
    exactly rounded sum of these (``solver.source_l2``)."""
    a = np.asarray(a, dtype=np.float64)
    return np.sum(np.square(a), axis=tuple(range(1, a.ndim)))


def _history(hist, tol, converged):
    return ResidualHistory(residual_inf=hist["residual_inf"],
                           true_residual_inf=hist["true_residual_inf"],
                           seconds=hist["seconds"], tolerance=tol, converged=converged,
                           relative_l2=hist["relative_l2"])


def _raise_if_diverged(hist, diverged):
    if diverged:
        hist.converged = False
        dmax = float(hist.residual_inf[-1])
        raise DivergenceError(
            f"update norm {dmax:.3e} exceeds the overflow guard after "
            f"{hist.iterations} steps", hist.iterations, hist)


def _solve(problem, weights, tol, max_iters, normalise, stop, check_every, fuse, chunk,
           l2_reference):
    from .solver import GridBackend, LocalComm, l2_from_layers, run_solve, source_l2

    tol = float(tol)
    if tol <= 0.0:
        raise ValueError("tolerance must be positive")
    if max_iters < 1:
        raise ValueError("max_iters must be at least 1")
    if stop not in ("update_inf", "residual_l2"):
        raise ValueError(f"unknown stopping rule {stop!r}")
    dev = _device_grid(problem)
    try:
        source = np.atleast_2d(problem.source)  # a 1-D line is one axis-0 layer
        backend = GridBackend(dev, source.shape[0])
        if stop == "residual_l2" and l2_reference is None:
            if getattr(problem, "source_kappa", None) is not None:
                l2_reference = lambda: l2_from_layers(  # noqa: E731 - residual of u0
                    backend, LocalComm, dev.residual_layers(0))[0]
            else:
                l2_reference = source_l2(backend, LocalComm, layer_sum_squares(source))
        hist, converged, diverged, cur = run_solve(
            backend, LocalComm, weights, tol, max_iters, normalise, stop, check_every, fuse,
            chunk, l2_reference, int(np.prod(problem.source.shape)))
        dev.download_field(cur, problem.u)  # ghosts refreshed on the device
    finally:
        dev.close()
    out = _history(hist, tol, converged)
    _raise_if_diverged(out, diverged)
    return out, problem.interior


def srj_solve(problem, cycle, tol, max_iters=10_000_000, *, stop="update_inf",
              check_every=None, fuse=0, chunk=None, l2_reference=None):
    """Relax with the cycle's weight sequence (``grids.py:642-687``) on the GPU.

    Keyword-only extensions: ``stop`` ("update_inf" = reference rule,
    "residual_l2" = BASELINE rule), ``check_every`` (L2 rule cadence, default
    one M-cycle), ``fuse`` (sweeps per launch, 0 = automatic), ``chunk``
    (steps per host check of the reference rule), ``l2_reference`` (norm the
    L2 residual is divided by; default ||source||_2).
    """
    return _solve(problem, cycle.weight_sequence, tol, max_iters, True, stop,
                  check_every, fuse, chunk, l2_reference)


def jacobi_solve(problem, tol, max_iters=10_000_000, *, stop="update_inf",
                 check_every=None, fuse=0, chunk=None, l2_reference=None):
    """Plain Jacobi, omega = 1 (``grids.py:690-694``)."""
    return _solve(problem, np.ones(1), tol, max_iters, False, stop, check_every,
                  fuse, chunk, l2_reference)


def gauss_seidel_solve(problem, tol, max_iters=10_000_000):
    """Gauss-Seidel in lexicographic order (``grids.py:697-702``), bitwise the
    reference's in-place ``_gs2``/``_gs3`` sweeps, on a GPU wavefront
    (``srj_plan_gs``).  Same returns, stopping rule (``dmax < tol`` after every
    sweep) and ``DivergenceError`` as the reference."""
    return _gs_solve(problem, 1.0, tol, max_iters, sor=False)


def sor_solve(problem, omega, tol, max_iters=10_000_000):
    """Successive over-relaxation (``grids.py:705-716``): Gauss-Seidel with
    relaxation factor ``omega``; the stopping metric is ``dmax / omega``."""
    if not 0.0 < omega < 2.0:
        raise ValueError("SOR relaxation factor must lie in (0, 2)")
    return _gs_solve(problem, float(omega), tol, max_iters, sor=True)


def _gs_solve(problem, omega, tol, max_iters, sor):
    tol = float(tol)
    if tol <= 0.0:
        raise ValueError("tolerance must be positive")
    if max_iters < 1:
        raise ValueError("max_iters must be at least 1")
    if getattr(problem, "source_kappa", None) is not None:
        raise NotImplementedError("Gauss-Seidel has no nonlinear source")
    dev = _device_grid(problem)
    start = time.perf_counter()
    diffs, resids, secs = [], [], []
    converged = False
    diverged_at = None
    cur, work = 0, 1  # cur: snapshot at a chunk start; work: swept in place
    done = 0
    # chunks as in _solve, sized for the slower in-place wavefront sweeps
    est = 8.0 * _step_seconds_estimate(problem)
    cap = int(min(65536, max(16, 0.05 / est)))
    span = int(min(cap, max(8, 0.002 / est)))
    try:
        while done < max_iters:
            n = min(span, max_iters - done)
            span = min(cap, 2 * span)
            dev.copy_field(cur, work)
            dev.gs(work, omega, n)
            norms = dev.norms[:2 * n].view(n, 2).cpu().numpy()
            t_now = time.perf_counter() - start
            t_prev = float(secs[-1][-1]) if secs else 0.0
            metric = norms[:, 0] / omega if sor else norms[:, 0]
            bad = ~np.isfinite(metric) | (metric > OVERFLOW_LIMIT)
            events = np.flatnonzero(bad | (metric < tol))
            take = n if events.size == 0 else int(events[0]) + 1
            if take < n:  # replay from the snapshot to the exact sweep
                dev.copy_field(cur, work)
                dev.gs(work, omega, take)
            diffs.append(metric[:take])
            resids.append(norms[:take, 1])
            secs.append(t_prev + (t_now - t_prev) * np.arange(1, take + 1) / take)
            done += take
            cur, work = work, cur
            if events.size:
                if bad[take - 1]:
                    diverged_at = take - 1
                else:
                    converged = True
                break
        dev.download_field(cur, problem.u)  # ghosts refreshed on the device
    finally:
        dev.close()
    hist = ResidualHistory(
        residual_inf=np.concatenate(diffs) if diffs else np.zeros(0),
        true_residual_inf=np.concatenate(resids) if resids else np.zeros(0),
        seconds=np.concatenate(secs) if secs else np.zeros(0),
        tolerance=tol, converged=converged)
    if diverged_at is not None:
        hist.converged = False
        dmax = float(hist.residual_inf[-1])
        raise DivergenceError(
            f"update norm {dmax:.3e} exceeds the overflow guard after "
            f"{hist.iterations} steps", hist.iterations, hist)
    return hist, problem.interior
