"""Eq. 12, 13, 21, 22 (paper_2007_00745_b200/analysis.py) pinned to the paper's
Table I and Table II (tests/golden/paper_tables.json)."""
import json
import math
import os

import pytest

from paper_2007_00745_b200 import analysis as A

T = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_tables.json")))


def test_table1_amdahl():
    # r_s from the p = infinity entry (356.22764 = 1 / r_s); the finite rows follow
    r_p = 1.0 - 1.0 / T["table1"]["inf"]
    for n, want in zip(T["table1"]["N"], T["table1"]["speedup"]):
        assert abs(A.amdahl_speedup(r_p, n) - want) < 1e-3, n
    assert abs(A.amdahl_speedup(r_p, math.inf) - T["table1"]["inf"]) < 1e-6
    assert A.amdahl_speedup(r_p, 1) == pytest.approx(1.0)
    assert A.amdahl_speedup(0.0, 32) == 1.0


def test_table2b_percentage_difference():
    t2a, t2b = T["table2a"], T["table2b"]
    for scheme in ("naive", "fcfs", "alternating"):
        for i, n in enumerate(t2a["N"]):
            d = A.percentage_difference(t2a["theoretical"][i], t2a[scheme][i])
            assert abs(d - t2b[scheme][i]) < 5e-3, (scheme, n, d)


def test_equation_properties():
    assert A.parallel_fraction(5.0, 10.0) == 0.5
    assert A.parallel_fraction(10.0, 10.0) == 1.0
    assert A.actual_speedup(10.0, 5.0) == 2.0
    assert A.percentage_difference(3.0, 3.0) == 0.0
    assert A.percentage_difference(2.0, 3.0) == A.percentage_difference(3.0, 2.0)
    prev = 0
    for p in (1, 2, 4, 8, 16, 32, 1024):
        s = A.amdahl_speedup(0.99, p)
        assert s > prev and s < 100.0
        prev = s
    assert A.load_balance_bound([1, 1, 1, 1]) == 4.0
    assert A.load_balance_bound([3, 1]) == pytest.approx(4 / 3)
    with pytest.raises(ValueError):
        A.parallel_fraction(2.0, 1.0)
    with pytest.raises(ValueError):
        A.amdahl_speedup(1.0, math.inf)
