"""Builders shared by the CPU and GPU tests."""

import numpy as np

from paper_1511_04292_b200.grids import FIXED, GridProblem


def problem_from(fields, kappa=None, bc=None, post=None):
    nd = fields["source"].ndim
    if bc is not None:
        from paper_1511_04292_b200.grids import GridProblem as GP

        return GP(spacing=(1.0,) * nd, u=np.array(fields["u"], dtype=float, copy=True),
                  source=np.array(fields["source"], dtype=float, copy=True),
                  center=np.asarray(fields["center"], dtype=float),
                  lower=tuple(np.asarray(a, dtype=float) for a in fields["lower"]),
                  upper=tuple(np.asarray(a, dtype=float) for a in fields["upper"]),
                  bc=bc, mask=fields.get("mask"), post_sweep=post)
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


def crop_window(f, lo, hi, k):
    """Sub-problem whose interior covers [lo-k, hi+k) (clipped to the grid),
    ghost ring taken from the initial field.  After k sweeps a cell depends
    only on cells within distance k, so the window [lo, hi) of the crop's
    result equals the full grid's (dependency cone)."""
    shape = f["source"].shape
    a = [max(0, l - k) for l in lo]
    b = [min(n, h + k) for h, n in zip(hi, shape)]
    si = tuple(slice(x, y) for x, y in zip(a, b))
    sg = tuple(slice(x, y + 2) for x, y in zip(a, b))
    sub = {"u": np.array(f["u"][sg]), "source": np.array(f["source"][si]),
           "center": f["center"][si], "lower": tuple(x[si] for x in f["lower"]),
           "upper": tuple(x[si] for x in f["upper"]), "mask": None}
    win = tuple(slice(l - x, h - x) for l, h, x in zip(lo, hi, a))
    return sub, win

