"""Builders shared by the CPU and GPU tests."""

import numpy as np

from paper_1511_04292_b200.grids import FIXED, GridProblem


def problem_from(fields, kappa=None, bc=None):
    nd = fields["source"].ndim
    if bc is not None:
        from paper_1511_04292_b200.grids import GridProblem as GP

        return GP(spacing=(1.0,) * nd, u=np.array(fields["u"], dtype=float, copy=True),
                  source=np.array(fields["source"], dtype=float, copy=True),
                  center=np.asarray(fields["center"], dtype=float),
                  lower=tuple(np.asarray(a, dtype=float) for a in fields["lower"]),
                  upper=tuple(np.asarray(a, dtype=float) for a in fields["upper"]),
                  bc=bc, mask=fields.get("mask"))
    return GridProblem(
        spacing=(1.0,) * nd,
        u=np.array(fields["u"], dtype=float, copy=True),
        source=np.array(fields["source"], dtype=float, copy=True),
        center=np.asarray(fields["center"], dtype=float),
        lower=tuple(np.asarray(a, dtype=float) for a in fields["lower"]),
        upper=tuple(np.asarray(a, dtype=float) for a in fields["upper"]),
        bc=((FIXED, FIXED),) * nd,
        mask=fields.get("mask"),
        source_kappa=kappa if kappa is not None else fields.get("kappa"),
    )


class Cycle:
    """Minimal cycle object: srj_solve reads only ``weight_sequence``."""

    def __init__(self, weights):
        self.weight_sequence = np.asarray(weights, dtype=float)
