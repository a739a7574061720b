"""The invariant DESIGN.md R18's batched escape test rests on, checked on the CPU.

The EAGER kernel tests |z|^2 only every B updates against a threshold T just below
R^2 and replays a batch exactly when T is reached.  That is correct iff every orbit
that escaped (first |z|^2 > R^2) inside a batch still has |z|^2 >= T at the batch's
end, i.e. during the B - 1 updates after its escape.  This test iterates the
recurrence in the oracle's operation order (Eq. 1, no contraction; numpy rounds each
op) past each pixel's escape and measures the smallest |z|^2 / R^2 seen in those
updates, on the full plane and on the windows where an escaped orbit grows slowest
(just left of c = -2, around +-2i, the cusp c = 1/4), for the B the library allows
per dtype (fp64 16, fp32 8), and checks it against T / R^2 from R18's definition:
fp64 T = the double whose high word is hi(R^2) - 0x100, fp32 T = bits(R^2) - 2^21.
"""
import numpy as np
import pytest


def _threshold(r2, dtype):
    if dtype == "fp64":
        hi = (np.array([r2], np.float64).view(np.uint64)[0] >> np.uint64(32)) - np.uint64(0x100)
        return float(np.array([hi << np.uint64(32)], np.uint64).view(np.float64)[0])
    b = np.array([r2], np.float32).view(np.uint32)[0] - np.uint32(1 << 21)
    return float(np.array([b], np.uint32).view(np.float32)[0])


def _min_post_escape_ratio(xmin, xmax, ymin, ymax, W, H, iter_max, R, dtype, B):
    T = np.float64 if dtype == "fp64" else np.float32
    lo_x, hi_x, lo_y, hi_y, rad = (T(v) for v in (xmin, xmax, ymin, ymax, R))
    dx, dy = (hi_x - lo_x) / T(W), (hi_y - lo_y) / T(H)
    r2 = rad * rad
    cr = np.broadcast_to((lo_x + np.arange(W).astype(T) * dx)[None, :], (H, W)).ravel().copy()
    ci = np.broadcast_to((hi_y - np.arange(H).astype(T) * dy)[:, None], (H, W)).ravel().copy()
    x = np.zeros_like(cr)
    y = np.zeros_like(cr)
    x2 = np.zeros_like(cr)
    y2 = np.zeros_like(cr)
    since = np.full(cr.size, -1, np.int64)  # updates since the escape (-1: not escaped)
    worst = np.inf
    escaped_any = 0
    with np.errstate(over="ignore", invalid="ignore"):
        for n in range(1, iter_max + B):
            act = since < B - 1  # still inside the window that matters
            if not act.any():
                break
            idx = np.nonzero(act)[0]
            a, b, a2, b2 = x[idx], y[idx], x2[idx], y2[idx]
            ny = (a + a) * b + ci[idx]
            nx = (a2 - b2) + cr[idx]
            nx2, ny2 = nx * nx, ny * ny
            s = nx2 + ny2
            x[idx], y[idx], x2[idx], y2[idx] = nx, ny, nx2, ny2
            sc = since[idx]
            post = sc >= 0
            sc[post] += 1
            if post.any():
                ratio = (s[post] / r2).astype(np.float64)
                ratio = np.where(np.isnan(ratio), np.inf, ratio)  # NaN/inf count as hits (R18)
                worst = min(worst, float(ratio.min()))
            new = (~post) & (s > r2) & (n <= iter_max)
            sc[new] = 0
            escaped_any += int(new.sum())
            stop = (~post) & (~new) & (n >= iter_max)
            sc[stop] = B  # never escaped within the budget: out of the window
            since[idx] = sc
    return worst, escaped_any


CASES = [
    # (xmin, xmax, ymin, ymax, W, H, iterMax, R)
    (-2.5, 1.5, -2.0, 2.0, 800, 800, 200, 2.0),                    # C1
    (-2.0 - 4e-15, -2.0 + 4e-15, -3e-15, 3e-15, 181, 61, 4000, 2.0),  # left of c = -2 (fp64 ulps)
    (-2.05, -1.95, -1e-3, 1e-3, 400, 40, 3000, 2.0),
    (-1e-3, 1e-3, 2.0 - 1e-3, 2.0 + 1e-3, 200, 200, 2000, 2.0),     # around 2i
    (0.2499, 0.2501, -1e-4, 1e-4, 200, 100, 5000, 2.0),             # the cusp c = 1/4
    (-2.5, 1.5, -2.0, 2.0, 400, 400, 300, 20.0),                    # R = 20 (the paper's ER 400)
]
CASES32 = [
    (-2.5, 1.5, -2.0, 2.0, 800, 800, 200, 2.0),
    (-2.000002, -1.999998, -1e-6, 1e-6, 97, 33, 4000, 2.0),         # left of c = -2 (fp32 ulps)
    (-2.05, -1.95, -1e-3, 1e-3, 400, 40, 3000, 2.0),
    (-1e-3, 1e-3, 2.0 - 1e-3, 2.0 + 1e-3, 200, 200, 2000, 2.0),
]


@pytest.mark.parametrize("case", CASES)
def test_fp64_escaped_orbits_stay_above_threshold(case):
    worst, n = _min_post_escape_ratio(*case, "fp64", B=16)
    r2 = case[-1] ** 2
    assert n > 0
    assert worst >= _threshold(r2, "fp64") / r2, (worst, case)


@pytest.mark.parametrize("case", CASES32)
def test_fp32_escaped_orbits_stay_above_threshold(case):
    worst, n = _min_post_escape_ratio(*case, "fp32", B=8)
    r2 = float(np.float32(case[-1]) * np.float32(case[-1]))
    assert n > 0
    assert worst >= _threshold(r2, "fp32") / r2, (worst, case)


def test_thresholds_follow_r18():
    # T sits just below R^2: fp64 within 2^-12 (relative), fp32 within 2^-2
    for R in (2.0, 2.5, 20.0, 1000.0):
        r2 = R * R
        t64 = _threshold(r2, "fp64")
        assert 1 - 2.0 ** -11 <= t64 / r2 < 1.0
        r2f = float(np.float32(R) * np.float32(R))
        t32 = _threshold(r2f, "fp32")
        assert 1 - 2.0 ** -1 <= t32 / r2f < 1.0
