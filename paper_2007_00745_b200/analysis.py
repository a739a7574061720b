"""The paper's analysis equations (host-side, no GPU), used by the scaling report.

    Eq. 12  r_p = t_p / t_s                         (parallel fraction)
    Eq. 13  S_p = 1 / (r_s + r_p / p)               (Amdahl; Table I)
    Eq. 21  A_N = T_1 / T_N                         (actual speed-up)
    Eq. 22  D   = |T - A| / ((T + A) / 2) * 100     (percentage difference)

plus the load-balance bound a static partition imposes: with per-rank work w_r
(pixel-iterations), the speed-up over one rank is bounded by sum(w) / max(w)
(the paper's "top and bottom ... less time than the middle").
Pinned by tests/test_analysis.py against Table I and Table II(b).
"""
from __future__ import annotations

import math


def parallel_fraction(t_p: float, t_s: float) -> float:
    """Eq. 12: the share of the serial run's time spent generating the set."""
    if not (t_s > 0 and 0 < t_p <= t_s):
        raise ValueError("need 0 < t_p <= t_s")
    return t_p / t_s


def amdahl_speedup(r_p: float, p: float) -> float:
    """Eq. 13 with r_s = 1 - r_p; p may be math.inf (then 1/r_s)."""
    if not 0.0 <= r_p <= 1.0:
        raise ValueError("r_p must be in [0, 1]")
    r_s = 1.0 - r_p
    if math.isinf(p):
        if r_s == 0:
            raise ValueError("unbounded speed-up for r_s = 0")
        return 1.0 / r_s
    if p < 1:
        raise ValueError("p must be >= 1")
    return 1.0 / (r_s + r_p / p)


def actual_speedup(t_single: float, t_multi: float) -> float:
    """Eq. 21: total time by a single task over total time by N tasks."""
    if t_single <= 0 or t_multi <= 0:
        raise ValueError("times must be positive")
    return t_single / t_multi


def percentage_difference(theoretical: float, actual: float) -> float:
    """Eq. 22."""
    if theoretical <= 0 or actual <= 0:
        raise ValueError("speed-ups must be positive")
    return abs(theoretical - actual) / ((theoretical + actual) / 2.0) * 100.0


def efficiency(speedup: float, n: int) -> float:
    """Parallel efficiency A_N / N."""
    return speedup / n


def load_balance_bound(rank_work) -> float:
    """Upper bound of the speed-up of a partition with per-rank work ``rank_work``
    (each rank at the same rate, no communication): sum / max."""
    w = [float(v) for v in rank_work]
    if not w or max(w) <= 0:
        raise ValueError("need positive work")
    return sum(w) / max(w)
