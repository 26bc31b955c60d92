"""CPU parity oracle for the SRJ sweep path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this package.  The product package
(``paper_1511_04292_b200``) never imports it and has no CPU fallback.

Pinned against the reference (``/root/reference/pkg/src/srj``) through the
golden vectors in ``tests/golden`` that ``tools/make_golden.py`` produced by
running the reference's own ``srj_solve`` / ``weighted_jacobi_sweep`` here.
"""

from .oracle import (  # noqa: F401
    OVERFLOW_LIMIT,
    gs_solve,
    gs_sweep,
    load,
    np_step,
    refresh_ghosts,
    residual,
    run,
    run_bc,
    solve,
    step,
)
