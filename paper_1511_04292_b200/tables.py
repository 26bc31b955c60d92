"""Published SRJ parameter tables (P = 2..15) and the effective-N lookup.

Host-side restatement of ``srj/tables.py``: ``lookup`` returns the row with the
largest N <= target for a given P (``tables.py:170-207``), ``get`` is an exact
match (``tables.py:132-143``).  Rows come from
``data/parameter_tables.json``, exported from the reference's shipped table by
``tools/make_golden.py`` (the paper's published schedules, betas already
renormalised on load as ``tables.py:296-298`` does).
"""

import json
import os

from .schedule import WeightSchedule

__all__ = ["NoSuchRowError", "ParameterTable", "shipped_table"]

_DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data",
                     "parameter_tables.json")


class NoSuchRowError(LookupError):
    """No stored row satisfies the request (``tables.py:52-53``)."""


class ParameterTable:
    """(P, N) -> WeightSchedule map with the reference's lookup rule."""

    def __init__(self, schedules=()):
        self._by_key = {}
        for s in schedules:
            self._by_key[(s.p, s.n)] = s

    def __len__(self):
        return len(self._by_key)

    def __contains__(self, key):
        return tuple(key) in self._by_key

    def keys(self):
        return sorted(self._by_key)

    def get(self, p, n):
        try:
            return self._by_key[(p, n)]
        except KeyError:
            raise NoSuchRowError(f"no stored row for P={p}, N={n}") from None

    def lookup(self, p, n_target):
        sizes = [n for (q, n) in self._by_key if q == p]
        if not sizes:
            raise NoSuchRowError(f"no rows stored for P={p}")
        fitting = [n for n in sizes if n <= n_target]
        if not fitting:
            raise NoSuchRowError(
                f"P={p}: smallest stored N is {min(sizes)}, above target {n_target}")
        return self._by_key[(p, max(fitting))]


_CACHE = None


def shipped_table():
    """Fresh ParameterTable holding the published rows."""
    global _CACHE
    if _CACHE is None:
        with open(_DATA) as fh:
            doc = json.load(fh)
        _CACHE = [WeightSchedule(r["omegas"], r["betas"], int(r["n"]))
                  for r in doc["rows"]]
    return ParameterTable(_CACHE)
