"""Row-partition schemes (§III, Eq. 14-20): oracle plans pinned to the
worked examples, coverage invariants, and the product's mandel_plan_rows (host
logic in the C-ABI library, no GPU needed) compared with the oracle's plans."""
import json
import os

import numpy as np
import pytest

from oracle import partition as P

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
EX = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))


def test_naive_examples():
    for e in EX["naive"]:
        if "rank" in e:
            rows = P.naive_rows(e["H"], e["N"], e["rank"])
            assert rows[0] == e["first"] and rows[-1] == e["last"]
            assert rows == list(range(e["first"], e["last"] + 1))
        else:
            for r, (a, b) in enumerate(e["ranges"]):
                assert P.naive_rows(e["H"], e["N"], r) == list(range(a, b + 1))


def test_alternating_examples():
    for e in EX["alternating"]:
        assert P.alternating_rows(e["H"], e["N"], e["rank"]) == e["rows"]


def test_rows_per_task_and_messages():
    for e in EX["rows_per_task"]:
        assert P.rows_per_task(e["H"], e["N"]) == e["value"]
    for e in EX["message_count"]:
        assert P.message_count(e["scheme"], e["H"], e["N"]) == e["value"]


@pytest.mark.parametrize("fn", [P.naive_rows, P.alternating_rows])
def test_static_plans_are_permutations(fn):
    rng = np.random.default_rng(7)
    for _ in range(200):
        N = int(rng.integers(1, 40))
        H = int(rng.integers(N, 500))
        allrows = []
        for r in range(N):
            allrows += fn(H, N, r)
        assert sorted(allrows) == list(range(H)), (H, N)
        # equal shares within the regular part (Eq. 16)
        q = P.rows_per_task(H, N)
        sizes = [len(fn(H, N, r)) for r in range(N)]
        if fn is P.naive_rows:
            assert sizes[:-1] == [q] * (N - 1) and sizes[-1] == q + H % N
        else:
            assert sizes[1:] == [q] * (N - 1) and sizes[0] == q + H % N


def test_fcfs_chunks_cover():
    for H, c in [(8000, 16), (10, 3), (7, 16), (33, 1)]:
        ch = P.fcfs_chunks(H, c)
        assert sum(ch, []) == list(range(H))
        assert len(ch) == -(-H // c)


def test_invalid_plans():
    with pytest.raises(ValueError):
        P.naive_rows(3, 4, 0)
    with pytest.raises(ValueError):
        P.alternating_rows(10, 0, 0)


# ---------------------------------------------------------------------------
# The product's host-side planner (C-ABI mandel_plan_rows) against the oracle
# ---------------------------------------------------------------------------
def test_library_plan_matches_oracle(mandel):
    rng = np.random.default_rng(11)
    cases = [(8000, 4), (10, 4), (8, 4), (7, 1), (7, 7), (32768, 8), (16384, 3)]
    cases += [(int(rng.integers(n, 300)), n) for n in rng.integers(1, 33, size=60)]
    for H, N in cases:
        for r in range(N):
            assert mandel.mandel_plan_rows(mandel.MANDEL_BLOCK, H, N, r).tolist() == \
                P.naive_rows(H, N, r), (H, N, r)
            assert mandel.mandel_plan_rows(mandel.MANDEL_CYCLIC, H, N, r).tolist() == \
                P.alternating_rows(H, N, r), (H, N, r)


def test_library_plan_errors(mandel):
    with pytest.raises(mandel.MandelError) as e:
        mandel.mandel_plan_rows(mandel.MANDEL_BLOCK, 3, 4, 0)
    assert e.value.code == mandel.MANDEL_EINVAL
    with pytest.raises(mandel.MandelError):
        mandel.mandel_plan_rows(mandel.MANDEL_FCFS, 100, 2, 0)  # dynamic: no static plan
    with pytest.raises(mandel.MandelError):
        mandel.mandel_plan_rows(mandel.MANDEL_CYCLIC, 100, 2, 2)
    with pytest.raises(mandel.MandelError):
        mandel.mandel_plan_rows(mandel.MANDEL_FCFS_MASTER, 100, 4, 1)
