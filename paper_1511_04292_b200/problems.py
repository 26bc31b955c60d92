"""Seeded synthetic inputs for the BASELINE configurations.

Conventions (recorded in DESIGN.md, "Inputs"):

* unit square / cube, vertex-centred interior nodes x_i = i*h, i = 1..N,
  h = 1/(N+1) per axis; the ghost layer is the boundary node (FIXED ghosts),
  as ``srj/problems.py:279-330`` (poisson2d_dirichlet) does;
* operator in the reference's sign convention (``grids.py:249-262``):
  center = sum_ax 2/h_ax^2, lower = upper = -1/h_ax^2, source = -f for
  Laplace(u) = f;
* ``numpy.random.default_rng(seed)``; per Gaussian the draws are centre
  (d draws of U(0.1, 0.9)), width, amplitude; i.i.d. U(-1, 1) noise is drawn
  after all Gaussians;
* Gaussian a * exp(-|x-c|^2 / (2 w^2)), evaluated separably as the product of
  per-axis exponentials (inputs only have to be identical for the oracle and the
  GPU, which both consume the same arrays).

Coefficients are returned as zero-stride broadcast views (``np.broadcast_to``)
so a 32768^2 problem costs no coefficient memory; the GPU boundary detects the
constant stencil and uses the scalar kernels.
"""

import math

import numpy as np

__all__ = ["CONFIGS", "gaussian_sum", "poisson_fields", "nonlinear_fields",
           "config_fields", "config_schedule", "slab_config_fields"]

# BASELINE.json configs -> (shape, P, table-N, source recipe)
CONFIGS = {
    "cfg1": dict(shape=(256, 256), p=2, n_table=256, n_gauss=8, noise=False,
                 width=(0.02, 0.1), seed=1),
    "cfg2": dict(shape=(4096, 4096), p=6, n_table=4096, n_gauss=8, noise=True,
                 width=(0.02, 0.1), seed=2),
    "cfg3": dict(shape=(512, 512, 512), p=10, n_table=512, n_gauss=16,
                 noise=False, width=(0.02, 0.08), seed=3),
    "cfg4": dict(shape=(32768, 32768), p=15, n_table=32768, n_gauss=32,
                 noise=True, width=(0.02, 0.1), seed=4),
    # cfg5 uses the paper's effective-N route (srj/core.py:261-307, PAPER.md
    # section 5.1): the 256^3 Dirichlet grid matches the 2-D Neumann table at
    # N_eff = 181.7 -> the P=8 N=150 row.  The N=256 row diverges here: its
    # transient amplification is fed back through the psi^5 source
    # (profiles/round1_nl_schedules.log).
    "cfg5": dict(shape=(256, 256, 256), p=8, n_table="effective", nonlinear=True,
                 seed=5),
}


def config_schedule(name, table=None, optimal=False):
    """The CycleSchedule a BASELINE config runs (floor quantization).

    Default: the shipped table's ``lookup`` row (the reference's rule, e.g.
    cfg4 -> the P=15 N=2048 row, the largest stored).  ``optimal=True``:
    the optimal schedule for the config's exact N from ``optimize`` (the
    reference's ``optimize.solve``), e.g. P=15 at
    N=32768 for cfg4.
    """
    from .schedule import effective_n, quantize
    from .tables import shipped_table

    cfg = CONFIGS[name]
    table = table or shipped_table()
    n = cfg["n_table"]
    if n == "effective":
        shape = cfg["shape"]
        n = effective_n([s + 1 for s in shape], len(shape), "dirichlet")
    if optimal:
        from .optimize import optimal_schedule

        return quantize(optimal_schedule(cfg["p"], int(n), table=table))
    return quantize(table.lookup(cfg["p"], int(n)))


def _axes(shape, rows=None):
    """Node coordinates per axis; ``rows=(a, b)`` keeps axis-0 rows [a, b)."""
    axes = [np.arange(1, n + 1, dtype=np.float64) / (n + 1) for n in shape]
    if rows is not None:
        axes[0] = axes[0][rows[0]:rows[1]]
    return axes


def gaussian_sum(shape, rng, n_gauss, width, amp=(-1.0, 1.0), peak=None, rows=None):
    """Sum of seeded Gaussians on the vertex-centred interior grid (only
    axis-0 rows [a, b) when ``rows`` is given: same draws, same values)."""
    nd = len(shape)
    axes = _axes(shape, rows)
    out = np.zeros(tuple(len(x) for x in axes))
    for _ in range(n_gauss):
        centre = rng.uniform(0.1, 0.9, nd)
        w = rng.uniform(*width)
        a = rng.uniform(*(peak if peak is not None else amp))
        inv = 1.0 / (2.0 * w * w)
        factors = [np.exp(-np.square(x - c) * inv) for x, c in zip(axes, centre)]
        g = factors[0]
        for f in factors[1:]:
            g = np.multiply.outer(g, f)
        out += a * g
    return out


def _stencil(shape):
    h = [1.0 / (n + 1) for n in shape]
    inv = [1.0 / (x * x) for x in h]
    center = 0.0
    for v in inv:
        center += 2.0 * v
    return (np.broadcast_to(np.float64(center), shape),
            tuple(np.broadcast_to(np.float64(-v), shape) for v in inv),
            tuple(np.broadcast_to(np.float64(-v), shape) for v in inv))


def poisson_fields(shape, n_gauss=8, seed=1, noise=False, width=(0.02, 0.1)):
    """Dirichlet Poisson Laplace(u)=f, u=0 on the boundary, u0=0.

    Returns a dict with the reference GridProblem's fields (``u`` ghosted,
    ``source`` = -f, ``center``, ``lower``, ``upper``, ``mask`` = None).
    """
    shape = tuple(int(n) for n in shape)
    rng = np.random.default_rng(seed)
    f = gaussian_sum(shape, rng, n_gauss, width)
    if noise:
        f += rng.uniform(-1.0, 1.0, shape)
    center, lower, upper = _stencil(shape)
    return {
        "u": np.zeros(tuple(n + 2 for n in shape)),
        "source": -f,
        "center": center,
        "lower": lower,
        "upper": upper,
        "mask": None,
    }


def nonlinear_fields(shape, seed=5, n_gauss=4):
    """cfg5: -Laplace(psi) = 2 pi rho psi^5, psi = 1 on the boundary, psi0 = 1.

    ``kappa`` = 2*pi*rho is the per-cell factor of the fused source
    s(psi) = kappa * psi^5.
    """
    shape = tuple(int(n) for n in shape)
    rng = np.random.default_rng(seed)
    rho = gaussian_sum(shape, rng, n_gauss, width=(0.05, 0.15),
                       peak=(0.01, 0.1))
    center, lower, upper = _stencil(shape)
    return {
        "u": np.ones(tuple(n + 2 for n in shape)),
        "source": np.zeros(shape),
        "kappa": (2.0 * math.pi) * rho,
        "center": center,
        "lower": lower,
        "upper": upper,
        "mask": None,
    }


def laplace_neumann_fields(n):
    """Cell-centred n x n Laplace problem with mirrored ghosts on all faces.

    Restates ``srj/problems.py:246-276`` (laplace2d_neumann): h = 1/n, centre
    4/h^2, neighbours -1/h^2, zero source; pair with MIRROR rules.
    """
    h = 1.0 / n
    shape = (n, n)
    off = -1.0 / h ** 2
    return {"u": np.zeros((n + 2, n + 2)), "source": np.zeros(shape),
            "center": np.full(shape, 4.0 / h ** 2), "lower": (np.full(shape, off),) * 2,
            "upper": (np.full(shape, off),) * 2, "mask": None}


GS_THETA = (0.3037, 2.8903)  # test-B arc ends on r = 1 (srj/problems.py:42-43)


def grad_shafranov_fields(test, c, n):
    """The paper's Grad-Shafranov benchmark (section 5.3) as fields.

    Restates ``srj/problems.py:634-717``: Delta* psi + C^2 psi = 0 on
    r in [1, 10] (n equispaced nodes incl. both ends, whose rows hold the
    Dirichlet data) x theta in [0, pi] (n cells, cell centred, MIRROR ends).
    Rows: center = -2/dr^2 - 2/(r^2 dth^2) + C^2; radial neighbours 1/dr^2;
    theta neighbours (1/dth^2 -+ cot(theta)/(2 dth)) / r^2.  Test A: psi =
    sin^2(theta)/r on r = 1 and r = 10.  Test B: sin^2 arc on r = 1 between
    GS_THETA, zero elsewhere, relaxation restricted to the masked region
    (shape curve minus the disk of radius 1 at (x, y) = (4, 1.6)).
    Returns the field dict plus ``bc`` kinds ((fixed, fixed), (mirror, mirror)).
    """
    if test not in ("A", "B"):
        raise ValueError("test must be 'A' or 'B'")
    if n < 16:
        raise ValueError("n must be at least 16")
    dr = 9.0 / (n - 1)
    dth = math.pi / n
    r = 1.0 + np.arange(n) * dr
    theta = 0.0 + (np.arange(n) + 0.5) * dth
    ri = r[1:-1]
    r2 = (ri ** 2)[:, None]
    shape = (n - 2, n)
    cot = 1.0 / np.tan(theta)
    center = -2.0 / dr ** 2 - 2.0 / (r2 * dth ** 2) + c ** 2 + np.zeros(shape)
    rad = np.full(shape, 1.0 / dr ** 2)
    th_lo = (1.0 / dth ** 2 + cot[None, :] / (2.0 * dth)) / r2 + np.zeros(shape)
    th_hi = (1.0 / dth ** 2 - cot[None, :] / (2.0 * dth)) / r2 + np.zeros(shape)
    u = np.zeros((n, n + 2))
    mask = None
    if test == "A":
        u[0, 1:-1] = np.sin(theta) ** 2 / r[0]
        u[-1, 1:-1] = np.sin(theta) ** 2 / r[-1]
    else:
        t1, t2 = GS_THETA
        arc = (theta >= t1) & (theta <= t2)
        u[0, 1:-1] = np.where(arc, np.sin((theta - t1) / (t2 - t1) * math.pi) ** 2, 0.0)
        rr, tt = ri[:, None], theta[None, :]
        bound = (4.5 * np.sin(tt) ** 2 + 2.5 * np.sin(2.0 * tt) ** 2) * (
            1.0 - 0.4 * np.cos(3.0 * tt) + 0.3 * np.cos(5.0 * tt) + 0.05 * np.sin(25.0 * tt))
        x, y = rr * np.sin(tt), rr * np.cos(tt)
        mask = (rr < bound) & ~((x - 4.0) ** 2 + (y - 1.6) ** 2 < 1.0)
    return {"u": u, "source": np.zeros(shape), "center": center, "lower": (rad, th_lo),
            "upper": (rad.copy(), th_hi), "mask": mask,
            "bc": (("fixed", "fixed"), ("mirror", "mirror"))}


def _noise_rows(rng, shape, rows):
    """Rows [a, b) of ``rng.uniform(-1, 1, shape)`` without drawing the rest:
    every double is one 64-bit PCG64 output, so the generator is advanced past
    the a * (cells per row) draws of the rows before (rank-local inputs,
    tested against the global draw)."""
    per_row = int(np.prod(shape[1:]))
    bitgen = rng.bit_generator
    bitgen.advance(rows[0] * per_row)
    return rng.uniform(-1.0, 1.0, (rows[1] - rows[0],) + tuple(shape[1:]))


def slab_config_fields(name, decomp, shape=None):
    """Rank-local inputs of a BASELINE config for a ``SlabDecomposition``:
    the rows [a, b) = ``decomp.local_rows`` (owned + halos) of what
    ``config_fields`` builds, computed without the global arrays (Gaussians
    evaluated on the local rows, noise drawn with a PCG64 ``advance``), so a
    32768^2 grid costs each rank only its slab.  Returns a
    ``distributed.SlabProblem``."""
    from .distributed import SlabProblem

    cfg = CONFIGS[name]
    shape = tuple(int(n) for n in (shape or cfg["shape"]))
    a, b = decomp.local_rows
    local = (b - a,) + shape[1:]
    rng = np.random.default_rng(cfg["seed"])
    center, lower, upper = _stencil(shape)
    bc = lambda x: np.broadcast_to(x.reshape(-1)[:1].reshape(()), local)  # noqa: E731
    center, lower, upper = bc(center), tuple(bc(x) for x in lower), tuple(bc(x) for x in upper)
    # ghosted local field: rows [a-1, b+1) of the global ghosted field
    ug = tuple(n + 2 for n in local)
    if cfg.get("nonlinear"):
        rho = gaussian_sum(shape, rng, 4, width=(0.05, 0.15), peak=(0.01, 0.1), rows=(a, b))
        return SlabProblem(decomp, shape, np.ones(ug), center, lower, upper,
                           source=np.zeros(local), kappa=(2.0 * math.pi) * rho)
    f = gaussian_sum(shape, rng, cfg["n_gauss"], cfg["width"], rows=(a, b))
    if cfg["noise"]:
        f += _noise_rows(rng, shape, (a, b))
    return SlabProblem(decomp, shape, np.zeros(ug), center, lower, upper, source=-f)


def config_fields(name, shape=None):
    """Fields for a named BASELINE config, optionally at a reduced shape."""
    cfg = CONFIGS[name]
    shape = tuple(shape or cfg["shape"])
    if cfg.get("nonlinear"):
        return nonlinear_fields(shape, seed=cfg["seed"])
    return poisson_fields(shape, cfg["n_gauss"], cfg["seed"], cfg["noise"],
                          cfg["width"])
