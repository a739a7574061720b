"""Pins of the CPU oracle to things other than itself (runs without a GPU).

Each test fixes the oracle against what the paper and mathematics determine:
hand-iterated orbits, closed-form membership, exact rational brute force,
pixel-exact pin points, symmetry, decimation and iterMax invariants, and an
independent numpy implementation (tests/np_reference.py).
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import workloads as wl
from np_reference import np_map

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------
# Eq. 1 / Eq. 2 on single points
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_hand_iterated_escapes(oracle, dtype):
    for p in _golden("escape_pins.json")["hand_iterated"]:
        got = oracle.escape(p["c"][0], p["c"][1], p["iter_max"], p["R"], dtype)
        assert got == p["count"], (p, got)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_closed_form_members_never_escape(oracle, dtype):
    g = _golden("escape_pins.json")["never_escape"]
    for cr, ci in g["points"]:
        assert oracle.escape(cr, ci, g["iter_max"], g["R"], dtype) == g["iter_max"], (cr, ci)


def test_strict_compare_and_count_base(oracle):
    # c = -2: |z|^2 == 4 exactly on every update from the 2nd on; '>=' would give 1.
    assert oracle.escape(-2.0, 0.0, 57, 2.0) == 57
    # c = 2i: |z1|^2 == 4 is not an escape; z2 = -4+2i is (count 2, not 1).
    assert oracle.escape(0.0, 2.0, 57, 2.0) == 2
    # any |c| > R escapes at the first check
    for c in [(2.0001, 0.0), (0.0, -2.5), (-1.5, 1.5), (1e300, 0.0)]:
        assert oracle.escape(c[0], c[1], 1000, 2.0) == 1


def test_itermax_bounds_counts(oracle):
    # c = 0.5 escapes at 5: any iterMax <= 5 returns iterMax, larger ones return 5
    for m in range(1, 12):
        assert oracle.escape(0.5, 0.0, m, 2.0) == min(m, 5)


# --------------------------------------------------------------------------
# Exact rational brute force on dyadic 8x8 grids
# --------------------------------------------------------------------------
def _exact_count(cr: Fraction, ci: Fraction, iter_max: int, R2: Fraction, depth: int = 14):
    """Escape count from exact rational arithmetic, or None if undecided.

    Escaping orbits are followed exactly; bounded ones are decided by exact
    periodicity (a repeated z), the real segment [-2, 1/4], the main cardioid
    or the period-2 disc (closed-form membership of the Mandelbrot set)."""
    x = y = Fraction(0)
    seen = {(x, y)}
    for n in range(1, min(iter_max, depth) + 1):
        x, y = x * x - y * y + cr, 2 * x * y + ci
        if x * x + y * y > R2:
            return n
        if (x, y) in seen:
            return iter_max  # exactly periodic and never exceeded R^2
        seen.add((x, y))
    if n == iter_max:
        return iter_max
    if ci == 0 and Fraction(-2) <= cr <= Fraction(1, 4) and R2 >= 4:
        return iter_max
    q = (cr - Fraction(1, 4)) ** 2 + ci * ci
    if q * (q + (cr - Fraction(1, 4))) <= ci * ci / 4 and R2 >= 4:
        return iter_max  # main cardioid
    if (cr + 1) ** 2 + ci * ci <= Fraction(1, 16) and R2 >= 4:
        return iter_max  # period-2 disc
    return None


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
@pytest.mark.parametrize("window", [(-2.5, 1.5, -2.0, 2.0), (-2.5, 1.5, -1.0, 3.0)])
def test_exact_rational_8x8(oracle, dtype, window):
    cfg = wl.Config("g8", *window, 8, 8, 200, 2.0, dtype)
    got = oracle.render(cfg)
    xmin, xmax, ymin, ymax = (Fraction(v) for v in window)
    dx, dy = (xmax - xmin) / 8, (ymax - ymin) / 8
    for i in range(8):
        for j in range(8):
            # Cx[j] = xmin + j dx, Cy[i] = ymax - i dy (top-left corner sampling, row 0 = ymax)
            want = _exact_count(xmin + j * dx, ymax - i * dy, 200, Fraction(4))
            assert want is not None, (i, j)
            assert got[i, j] == want, (i, j, got[i, j], want)


def test_exact_grid_is_not_trivial(oracle):
    # the full-plane 8x8 grid mixes escapers (1..5) and members (200)
    got = oracle.render(wl.Config("g8", -2.5, 1.5, -2.0, 2.0, 8, 8, 200, 2.0, "fp64"))
    vals = set(np.unique(got).tolist())
    assert {1, 2, 3, 5, 200} <= vals


# --------------------------------------------------------------------------
# Step a3: the Cx / Cy arrays (SPEC.md:64-66 adapted)
# --------------------------------------------------------------------------
def test_axis_examples(oracle):
    ex = _golden("spec_examples.json")["axis"]
    cx, _ = oracle.axes(ex[0]["lo"], ex[0]["hi"], -1.0, 1.0, ex[0]["count"], 1, 2.0)
    assert cx.tolist() == ex[0]["values"]
    cx, _ = oracle.axes(ex[1]["lo"], ex[1]["hi"], -1.0, 1.0, ex[1]["count"], 1, 2.0)
    assert cx.tolist() == ex[1]["values"]
    cx, _ = oracle.axes(ex[2]["lo"], ex[2]["hi"], -1.0, 1.0, ex[2]["count"], 1, 2.0)
    assert cx[0] == ex[2]["first"] and abs(cx[-1] - ex[2]["last_approx"]) < 1e-12
    # Cy descends from ymax: row 0 is the top edge
    _, cy = oracle.axes(-2.0, 2.0, -2.0, 2.0, 4, 4, 2.0)
    assert cy.tolist() == [2.0, 1.0, 0.0, -1.0]
    _, cy = oracle.axes(-2.0, 2.0, -2.0, 2.0, 4, 4, 2.0, "fp32")
    assert cy.tolist() == [2.0, 1.0, 0.0, -1.0]


def test_derive_fp32_rounds_bounds_first(oracle):
    # 0.1 is not a float: fp32 mapping starts from float(0.1), not from 0.1
    xa, yb, dx, dy, r2 = oracle.derive(0.1, 0.9, -0.3, 0.7, 10, 10, 2.0, "fp32")
    assert xa == float(np.float32(0.1)) and yb == float(np.float32(0.7))
    assert r2 == 4.0
    assert dx == float((np.float32(0.9) - np.float32(0.1)) / np.float32(10))


PIN_POINTS_C1 = [  # (i, j, c) on C1's grid: c = (-2.5 + j*0.005, 2 - i*0.005) lands exactly
    (400, 500, (0.0, 0.0)), (400, 300, (-1.0, 0.0)), (400, 100, (-2.0, 0.0)),
    (200, 500, (0.0, 1.0)), (600, 500, (0.0, -1.0)), (400, 700, (1.0, 0.0)),
    (400, 600, (0.5, 0.0)), (400, 550, (0.25, 0.0)), (400, 350, (-0.75, 0.0)),
    (0, 0, (-2.5, 2.0)),
]
PIN_COUNT = {(0.0, 0.0): None, (-1.0, 0.0): None, (-2.0, 0.0): None, (0.0, 1.0): None,
             (0.0, -1.0): None, (1.0, 0.0): 3, (0.5, 0.0): 5, (0.25, 0.0): None,
             (-0.75, 0.0): None, (-2.5, 2.0): 1}  # None -> never escapes -> iterMax


PIN_GRIDS = {  # C3's fp32 dx = fl32(0.0005) is inexact, so fp32 pins use a dyadic grid
    "P1024f32": wl.Config("P1024f32", *wl.FULL_PLANE, 1024, 1024, 300, 2.0, "fp32"),
}


@pytest.mark.parametrize("name,scale", [("C1", 1), ("C2", 10), ("C5", 40.96),
                                        ("P1024f32", 1.28)])
def test_pin_points_on_configured_grids(oracle, name, scale):
    cfg = wl.CONFIGS.get(name) or PIN_GRIDS[name]
    ii, jj, want = [], [], []
    for i, j, c in PIN_POINTS_C1:
        I, J = round(i * scale), round(j * scale)
        if abs(I - i * scale) > 1e-9 or abs(J - j * scale) > 1e-9:
            continue
        ii.append(I)
        jj.append(J)
        want.append(PIN_COUNT[c] if PIN_COUNT[c] is not None else cfg.iter_max)
        cx = oracle.axes(cfg.xmin, cfg.xmax, cfg.ymin, cfg.ymax, cfg.W, 1, cfg.R, cfg.dtype)[0] \
            if cfg.W <= 8000 else None
        if cx is not None:
            assert cx[J] == c[0], (name, J, cx[J], c)
    assert len(ii) >= 3
    got = oracle.render_pixels(cfg, ii, jj)
    assert got.tolist() == want, (name, got.tolist(), want)


def test_asymmetric_window_orientation(oracle):
    # window [-2.5,1.5] x [0,4]: row 7, col 4 is c = -0.5 + 0.5i (cardioid, never
    # escapes) if row 0 is ymax; it would be -0.5 + 3.5i (escapes at 1) if row 0 were ymin.
    cfg = wl.Config("o", -2.5, 1.5, 0.0, 4.0, 8, 8, 200, 2.0, "fp64")
    m = oracle.render(cfg)
    assert m[7, 4] == 200 and m[0, 4] == 1


# --------------------------------------------------------------------------
# Invariants over whole maps
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_mirror_rows_identical(oracle, dtype):
    cfg = wl.C1.with_(dtype=dtype)
    m = oracle.render(cfg)
    _, cy = oracle.axes(*cfg.args()[:4], cfg.W, cfg.H, cfg.R, dtype)
    pairs = [(i, cfg.H - i) for i in range(1, cfg.H) if cy[i] == -cy[cfg.H - i]]
    assert len(pairs) > 100
    for i, k in pairs:
        assert np.array_equal(m[i], m[k]), (i, k)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_power_of_two_decimation(oracle, dtype):
    # On [-2.5,1.5]x[-2,2] with W = H = 2^k every c is an exact dyadic, so the
    # 2^k map sampled every 2^s pixels is the 2^(k-s) map, bit for bit.
    big = oracle.render(wl.Config("d", *wl.FULL_PLANE, 256, 256, 300, 2.0, dtype))
    for s in (1, 2, 3):
        small = oracle.render(wl.Config("d", *wl.FULL_PLANE, 256 >> s, 256 >> s, 300, 2.0, dtype))
        assert np.array_equal(big[::1 << s, ::1 << s], small)


def test_itermax_monotone(oracle):
    lo = oracle.render(wl.C1)
    hi = oracle.render(wl.C1.with_(iter_max=1000))
    assert np.array_equal(lo, np.minimum(hi, 200))


def test_range_and_c1_sum(oracle):
    m = oracle.render(wl.C1)
    assert m.min() >= 1 and m.max() <= 200
    # interior fraction of the full plane is ~9.5%; the map is non-trivial
    frac = float((m == 200).mean())
    assert 0.08 < frac < 0.11


# --------------------------------------------------------------------------
# Independent re-implementation (numpy), element by element
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_numpy_reference_c1(oracle, dtype):
    cfg = wl.C1.with_(dtype=dtype)
    assert np.array_equal(oracle.render(cfg), np_map(*cfg.args(), dtype))


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_numpy_reference_random_small(oracle, dtype):
    for cfg in wl.random_small_configs(50, 0, dtype):
        assert np.array_equal(oracle.render(cfg), np_map(*cfg.args(), dtype)), cfg


def test_numpy_reference_zoom_rows(oracle):
    # a few rows of C4's zoom window at a reduced width (exercises tiny dx)
    cfg = wl.C4.with_(W=512, H=512, iter_max=3000)
    rows = [0, 100, 255, 511]
    want = np_map(*cfg.args(), "fp64", rows=rows)
    for k, r in enumerate(rows):
        got = oracle.render_rows(*cfg.args(), "fp64", r, r + 1)[0]
        assert np.array_equal(got, want[k]), r


def test_fp32_differs_from_fp64(oracle):
    # the fp32 variant is a different map (own oracle), not fp64 rounded at the end
    a = oracle.render(wl.C1)
    b = oracle.render(wl.C1.with_(dtype="fp32"))
    assert 0 < int((a != b).sum()) < 5000


# --------------------------------------------------------------------------
# The FMA dtype (R17): its own oracle, pinned independently
# --------------------------------------------------------------------------
def _fma(a: float, b: float, c: float) -> float:
    """Correctly rounded fused multiply-add from exact rationals (CPython's
    Fraction -> float conversion rounds to nearest, ties to even)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _py_fma_escape(cr, ci, iter_max, r2):
    x = y = y2 = 0.0
    n = 0
    while n < iter_max:
        ny = _fma(x + x, y, ci)
        nx = _fma(x, x, -y2) + cr
        x, y = nx, ny
        y2 = y * y
        n += 1
        if _fma(x, x, y2) > r2:
            break
    return n


def test_fma_oracle_pins(oracle):
    for p in _golden("escape_pins.json")["hand_iterated"]:
        assert oracle.escape(p["c"][0], p["c"][1], p["iter_max"], p["R"], "fp64fma") == p["count"]
    g = _golden("escape_pins.json")["never_escape"]
    for cr, ci in g["points"]:
        assert oracle.escape(cr, ci, g["iter_max"], g["R"], "fp64fma") == g["iter_max"]


def test_fma_oracle_vs_exact_rounding_reference(oracle):
    for cfg in wl.random_small_configs(12, 100, "fp64fma"):
        cfg = cfg.with_(W=min(cfg.W, 12), H=min(cfg.H, 12))
        got = oracle.render(cfg)
        cx, cy = oracle.axes(*cfg.args()[:4], cfg.W, cfg.H, cfg.R, "fp64")
        for i in range(cfg.H):
            for j in range(cfg.W):
                assert got[i, j] == _py_fma_escape(float(cx[j]), float(cy[i]), cfg.iter_max,
                                                   cfg.R * cfg.R), (cfg, i, j)


def test_fma_map_is_its_own(oracle):
    # identical on C1, but a different map where rounding matters (C4's zoom window)
    assert np.array_equal(oracle.render(wl.C1), oracle.render(wl.C1.with_(dtype="fp64fma")))
    z = wl.C4.with_(W=512, H=512, iter_max=3000)
    d = int((oracle.render(z) != oracle.render(z.with_(dtype="fp64fma"))).sum())
    assert 0 < d < 512 * 512 // 20


# --------------------------------------------------------------------------
# The threaded row driver (render_rows_mt) -- the checker of every full-size parity
# test and of the CPU baseline.  It holds no arithmetic of its own; this pins that
# its row bookkeeping (chunk claims, output placement) returns exactly render_rows'
# rows, in the order asked, for any thread count and chunk size.
# --------------------------------------------------------------------------
@pytest.mark.parametrize("threads", [1, 3, 16])
@pytest.mark.parametrize("chunk", [1, 16])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_render_rows_mt_matches_render_rows(oracle, threads, chunk, dtype):
    cfg = wl.C1.with_(W=203, H=157, iter_max=400, dtype=dtype)
    whole = oracle.render(cfg)
    rng = np.random.default_rng(threads * 100 + chunk)
    row_sets = {
        "all": np.arange(cfg.H),
        "shuffled": rng.permutation(cfg.H),
        "strided": np.arange(5, cfg.H, 7),
        "repeated": np.array([3, 3, 156, 0, 77, 3]),
        "one": np.array([cfg.H - 1]),
    }
    for label, rows in row_sets.items():
        got, used = oracle.render_rows_mt(cfg, rows, threads=threads, chunk=chunk)
        assert used == threads
        assert got.shape == (len(rows), cfg.W) and got.dtype == np.uint32
        for k, r in enumerate(rows):
            want = oracle.render_rows(*cfg.args(), dtype, int(r), int(r) + 1)[0]
            assert np.array_equal(got[k], want), (label, k, int(r))
        assert np.array_equal(got, whole[rows]), label


def test_render_rows_mt_empty_and_errors(oracle):
    cfg = wl.C1.with_(W=50, H=40)
    got, _ = oracle.render_rows_mt(cfg, np.array([], dtype=np.int64), threads=4)
    assert got.shape == (0, 50)
    with pytest.raises(ValueError):  # a row outside [0, H) is rejected, not silently computed
        oracle.render_rows_mt(cfg, np.array([0, 40]), threads=2)
