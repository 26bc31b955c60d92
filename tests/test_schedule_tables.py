"""Host-side schedule inputs vs the reference (golden) and its published values.

References: srj/schedule.py:100-180 (quantize/layout), srj/tables.py:132-207
(get/lookup), tests test_schedule.py:33-49 and test_tables.py:35-71.
"""

import numpy as np
import pytest

from conftest import load_golden
from paper_1511_04292_b200.schedule import (
    CycleSchedule,
    DegenerateCycleError,
    WeightSchedule,
    layout,
    quantize,
)
from paper_1511_04292_b200.tables import NoSuchRowError, shipped_table

TAGS = {"cfg1": (2, 256), "cfg2": (6, 4096), "cfg3": (10, 512),
        "cfg4": (15, 32768), "cfg5": (8, 256), "p6n64": (6, 64),
        "p10n550": (10, 550), "p6n256": (6, 256)}


@pytest.fixture(scope="module")
def table():
    return shipped_table()


@pytest.mark.parametrize("tag", sorted(TAGS))
@pytest.mark.parametrize("strategy", ["floor", "round", "ceil"])
def test_schedules_bitwise_equal_reference(table, tag, strategy):
    g = load_golden("schedules")
    p, n = TAGS[tag]
    ws = table.lookup(p, n)
    assert ws.n == int(g[f"{tag}_pn"][2])
    if f"{tag}_{strategy}_error" in g:
        with pytest.raises(DegenerateCycleError):
            quantize(ws, strategy)
        return
    cyc = quantize(ws, strategy)
    assert np.array_equal(cyc.q, g[f"{tag}_{strategy}_q"])
    assert np.array_equal(cyc.weight_sequence, g[f"{tag}_{strategy}_seq"])


def test_table_has_published_rows(table):
    assert len(table) == 315
    assert {p for p, _ in table.keys()} == set(range(2, 16))


def test_lookup_rule(table):
    ws = table.lookup(10, 585)
    assert ws.n == 550 and ws.rho == pytest.approx(125.85, abs=0.01)
    with pytest.raises(NoSuchRowError):
        table.lookup(15, 32)
    with pytest.raises(NoSuchRowError):
        table.get(3, 1)


def test_published_counts(table):
    # test_schedule.py:33-36 / PAPER.md:1171
    cyc = quantize(table.get(10, 550))
    assert list(cyc.q) == [1, 1, 3, 9, 21, 49, 116, 268, 587, 1014]
    assert cyc.m == 2069


def test_layout_example():
    seq = layout([1, 3], [10.0, 0.5])
    assert sorted(seq) == [0.5, 0.5, 0.5, 10.0]
    assert seq[0] == 10.0


def test_cycle_invariants(table):
    ws = table.get(6, 64)
    with pytest.raises(ValueError, match="q_1"):
        CycleSchedule(q=[2, 1, 1, 1, 1, 1], weight_sequence=np.ones(7), source_schedule=ws)
    with pytest.raises(ValueError, match="permutation"):
        cyc = quantize(ws)
        CycleSchedule(q=cyc.q, weight_sequence=np.ones(cyc.m), source_schedule=ws)


def test_weight_schedule_validation():
    with pytest.raises(ValueError, match="decreasing"):
        WeightSchedule([1.0, 2.0], [0.5, 0.5], 10)
    with pytest.raises(ValueError, match="sum to 1"):
        WeightSchedule([5.0, 0.5], [0.5, 0.6], 10)


def test_effective_n_matches_reference_examples():
    from paper_1511_04292_b200.problems import config_schedule
    from paper_1511_04292_b200.schedule import effective_n

    # test_core.py:227-230 / core.py docstring: 585 x 280 Dirichlet -> 252.56
    assert round(effective_n((585, 280), bc="dirichlet"), 2) == 252.56
    assert abs(effective_n((257, 257, 257), 3, "dirichlet") - 181.73) < 0.01
    assert config_schedule("cfg5").source_schedule.n == 150
    assert config_schedule("cfg2").m == 25530


@pytest.mark.parametrize("test,c,n", [("A", 0.0, 40), ("A", 0.34, 33), ("B", 0.0, 48)])
def test_grad_shafranov_builder_matches_reference(test, c, n):
    """The restated paper benchmark problem equals srj.problems.grad_shafranov."""
    from paper_1511_04292_b200.problems import grad_shafranov_fields

    g = load_golden("builders")
    tag = f"gs_{test}_{str(c).replace('.', 'p')}_{n}"
    f = grad_shafranov_fields(test, c, n)
    assert np.array_equal(f["u"], g[tag + "_u"])
    assert np.array_equal(f["center"], g[tag + "_center"])
    assert np.array_equal(f["lower"][0], g[tag + "_lower0"])
    assert np.array_equal(f["lower"][1], g[tag + "_lower1"])
    assert np.array_equal(f["upper"][1], g[tag + "_upper1"])
    if test == "B":
        assert np.array_equal(f["mask"], g[tag + "_mask"])
