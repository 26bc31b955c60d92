"""B200-native (sm_100a) SRJ weighted-Jacobi sweep path of arXiv:1511.04292.

Drop-in for the reference package's hot path ``srj.grids``: the solver entry
points keep the reference's names, arguments, results and exceptions, and run
on hand-written CUDA kernels in ``libsrj.so`` (C ABI: ``include/srj.h``).
"""

from .grids import (  # noqa: F401
    FIXED,
    MIRROR,
    OVERFLOW_LIMIT,
    PERIODIC,
    BoundaryRule,
    DivergenceError,
    GridProblem,
    ResidualHistory,
    face_dirichlet,
    gauss_seidel_solve,
    jacobi_solve,
    post_sweep_gather,
    sor_solve,
    srj_solve,
    weighted_jacobi_sweep,
)
from .optimize import optimal_schedule  # noqa: F401
from .schedule import CycleSchedule, WeightSchedule, quantize  # noqa: F401
from .tables import shipped_table  # noqa: F401
