"""SRJ weight schedules and integer M-cycles (host side, computed once per solve).

Host-side restatement of the reference's schedule inputs so the GPU path is
usable where the reference package is absent:

* ``WeightSchedule`` -- ``srj/core.py:59-127`` (validated (omega, beta, N) value)
* ``quantize``       -- ``srj/schedule.py:100-144`` (q_i = round_fn(beta_i/beta_1), q_1 = 1)
* ``layout``         -- ``srj/schedule.py:147-180`` (slot round((j + i/P) M/q_i),
                        forward probing with wraparound)
* ``CycleSchedule``  -- ``srj/schedule.py:33-83`` (q, weight_sequence, m)
* ``validate_cycle`` -- ``srj/schedule.py:183-217``
* ``effective_n``    -- only the Dirichlet/d-dimensional mapping of
                        ``srj/core.py:261-307`` used to pick a table row.

The GPU consumes ``CycleSchedule.weight_sequence`` verbatim; nothing here is on
the device.  ``tests/golden/schedules.npz`` pins ``quantize``/``layout``
bit-for-bit against the reference.
"""

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "CycleSchedule",
    "DegenerateCycleError",
    "StabilityReport",
    "WeightSchedule",
    "effective_n",
    "layout",
    "quantize",
    "validate_cycle",
]


def _frozen_vector(values, what):
    v = np.array(values, dtype=np.float64, copy=True)
    if v.ndim != 1 or v.size == 0:
        raise ValueError(f"{what} must be a non-empty 1-D vector")
    v.setflags(write=False)
    return v


@dataclass(frozen=True)
class WeightSchedule:
    """Relaxation weights omega_1 > ... > omega_P with fractions beta_i.

    Same invariants and error behaviour as ``srj/core.py:98-122``.
    """

    omegas: np.ndarray
    betas: np.ndarray
    n: int
    rho: float = None

    def __post_init__(self):
        om = _frozen_vector(self.omegas, "omegas")
        be = _frozen_vector(self.betas, "betas")
        object.__setattr__(self, "omegas", om)
        object.__setattr__(self, "betas", be)
        if om.shape != be.shape:
            raise ValueError("omegas and betas must have equal length")
        if not bool(np.all(om[1:] < om[:-1])):
            raise ValueError("omegas must be strictly decreasing")
        last = om[-1]
        if om.size == 1:
            if not 0.0 < last <= 1.0:
                raise ValueError(f"a single weight must lie in (0, 1], got {last}")
        else:
            if not 0.0 < last < 1.0:
                raise ValueError(f"omega_P must lie in (0, 1), got {last}")
            if om[0] <= 1.0:
                raise ValueError(f"omega_1 must exceed 1 for P >= 2, got {om[0]}")
        if bool(np.any(be <= 0.0)) or bool(np.any(be > 1.0)):
            raise ValueError("betas must lie in (0, 1]")
        if om.size >= 2 and bool(np.any(be >= 1.0)):
            raise ValueError("betas must lie in (0, 1)")
        off = be.sum() - 1.0
        if abs(off) > 1e-12:
            raise ValueError(f"betas must sum to 1, off by {off:.3e}")
        if not (isinstance(self.n, (int, np.integer)) and self.n >= 2):
            raise ValueError(f"n must be an integer >= 2, got {self.n}")
        rho = float(np.dot(om, be))
        if self.rho is None:
            object.__setattr__(self, "rho", rho)
        elif abs(self.rho - rho) > 1e-10 * abs(rho):
            raise ValueError(f"rho {self.rho} inconsistent with sum(omega*beta) {rho}")

    @property
    def p(self):
        return int(self.omegas.size)


class DegenerateCycleError(ValueError):
    """A repetition count came out zero (srj/schedule.py:29-30)."""


@dataclass(frozen=True)
class CycleSchedule:
    """Integer counts q and the M weights in execution order."""

    q: np.ndarray
    weight_sequence: np.ndarray
    source_schedule: WeightSchedule
    m: int = field(init=False)

    def __post_init__(self):
        q = np.array(self.q, dtype=int, copy=True)
        seq = np.array(self.weight_sequence, dtype=np.float64, copy=True)
        for a in (q, seq):
            a.setflags(write=False)
        object.__setattr__(self, "q", q)
        object.__setattr__(self, "weight_sequence", seq)
        object.__setattr__(self, "m", int(q.sum()))
        if q.ndim != 1 or q.size != self.source_schedule.p:
            raise ValueError("q must hold one count per weight")
        if q[0] != 1:
            raise ValueError("q_1 must be 1; counts are scaled to the rarest weight")
        if bool(np.any(q < 1)):
            raise DegenerateCycleError("every weight needs at least one step")
        if seq.shape != (self.m,):
            raise ValueError(f"weight sequence must have M={self.m} entries")
        expect = np.sort(np.repeat(self.source_schedule.omegas, q))
        if not np.array_equal(np.sort(seq), expect):
            raise ValueError("weight sequence is not a permutation of the counted weights")

    @property
    def p(self):
        return int(self.q.size)


_ROUNDING = {
    "floor": math.floor,
    "round": lambda x: math.floor(x + 0.5),
    "ceil": math.ceil,
}


def quantize(schedule, strategy="floor"):
    """Integer counts from fractions: q_i = fn(beta_i / beta_1), q_1 = 1."""
    if strategy not in _ROUNDING:
        raise ValueError(f"unknown strategy {strategy!r}")
    fn = _ROUNDING[strategy]
    ratios = schedule.betas / schedule.betas[0]
    counts = [1]
    counts.extend(fn(x) for x in ratios[1:])
    if min(counts) < 1:
        raise DegenerateCycleError("a fraction smaller than beta_1 quantized to zero")
    return CycleSchedule(q=np.asarray(counts, dtype=int),
                         weight_sequence=layout(counts, schedule.omegas),
                         source_schedule=schedule)


def layout(q, omegas):
    """Spread class i's q_i copies over M slots with phase i/P."""
    counts = [int(x) for x in q]
    if len(counts) != len(omegas):
        raise ValueError("q and omegas must align")
    m = sum(counts)
    nclass = len(counts)
    seq = np.full(m, np.nan)
    taken = np.zeros(m, dtype=bool)
    for cls, (qi, w) in enumerate(zip(counts, omegas)):
        spacing = m / qi
        phase = cls / nclass
        for j in range(qi):
            slot = int(math.floor((j + phase) * spacing + 0.5)) % m
            while taken[slot]:
                slot = (slot + 1) % m
            taken[slot] = True
            seq[slot] = w
    return seq


@dataclass(frozen=True)
class StabilityReport:
    max_amplification: float
    kappa_at_max: float
    passed: bool


def validate_cycle(cycle, kappa_range, grid_points=10000):
    """max over kappa of prod |1 - omega_i kappa|^q_i on a uniform band grid."""
    kmin, kmax = kappa_range
    grid = np.linspace(kmin, kmax, grid_points)
    with np.errstate(divide="ignore"):
        logs = np.log(np.abs(1.0 - np.outer(grid, cycle.source_schedule.omegas)))
    logs = logs @ cycle.q.astype(float)
    at = int(np.argmax(logs))
    top = float(logs[at])
    amp = math.inf if top > 709 else math.exp(top)
    return StabilityReport(max_amplification=amp, kappa_at_max=float(grid[at]),
                           passed=amp < 1.0)


def effective_n(sizes, d=None, bc="neumann"):
    """2-D Neumann table size with the same kappa_min (``srj/core.py:261-307``).

    Neumann:   n_eff = pi / (2 asin(sqrt(2/d) sin(pi/(2 n_max))))
    Dirichlet: n_eff = pi / (2 asin(sqrt((2/d) sum_i sin(pi/(2 n_i))^2)))
    """
    s = np.atleast_1d(np.asarray(sizes, dtype=float))
    if bool(np.any(s < 2)):
        raise ValueError("all sizes must be >= 2")
    d = int(s.size if d is None else d)
    if d not in (1, 2, 3):
        raise ValueError(f"d must be 1, 2 or 3, got {d}")
    if bc == "neumann":
        if d == 2:
            return float(s.max())
        arg = math.sqrt(2.0 / d) * math.sin(math.pi / (2.0 * s.max()))
    elif bc == "dirichlet":
        arg = math.sqrt((2.0 / d) * float(np.sum(np.sin(math.pi / (2.0 * s)) ** 2)))
    else:
        raise ValueError(f"unknown boundary kind {bc!r}")
    return math.pi / (2.0 * math.asin(arg))
