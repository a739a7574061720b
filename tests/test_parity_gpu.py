"""Parity of the CUDA path (through the C ABI) with the CPU oracle, on a B200.

Integer outputs: the bar is bit-exact equality, element by element (DESIGN.md
"Parity").  Small maps are compared whole; the full-size configurations, in the
launch configuration bench.py times, are compared on seeded sampled rows the
oracle computes one by one, plus properties that hold at any size (range,
coverage, exact mirror rows, power-of-two decimation against a whole oracle map,
Σcounts against the map).
"""
import numpy as np
import pytest

import workloads as wl

pytestmark = pytest.mark.gpu

SCHEMES = ["block", "cyclic", "fcfs"]


def _torch():
    import torch
    assert torch.cuda.is_available(), "gpu test without a CUDA device"
    return torch


def _render_dev(mandel, cfg, scheme="block", ngpus=1, **kw):
    torch = _torch()
    out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device="cuda:0")
    # every other call leaves stream0 unset: the library's own (blocking) stream must then
    # still be ordered after torch's zero-fill on the default stream
    if kw.pop("pass_stream", True) and (cfg.W + cfg.H) % 2 == 0:
        kw["stream0"] = torch.cuda.current_stream().cuda_stream
    st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, ngpus, out_dev0=out,
                                 logical_ranks=ngpus > 1, **kw)
    return out, st


def _host(t):
    return t.cpu().numpy().view(np.uint32)


def _assert_same(got, want, label):
    if not np.array_equal(got, want):
        bad = np.argwhere(got != want)
        i, j = bad[0]
        raise AssertionError(f"{label}: {len(bad)} pixels differ; first at (i={i}, j={j}): "
                             f"gpu={got[i, j]} oracle={want[i, j]}")


# ---------------------------------------------------------------------------
# whole maps: C1 and reduced shapes, every scheme, logical rank counts, kernels
# ---------------------------------------------------------------------------
KERNELS = ["refill", "refill1", "refill2", "refill3", "refill4", "lazy1", "lazy2", "adaptive1", "adaptive2",
           "batch4x1", "batch4x2", "batch4x4", "batch8x1", "batch8x2", "batch8x3", "batch8x4",
           "batch16x1", "batch16x2", "batch16x4", "adaptb4x1", "adaptb8x2"]


def _batched(mandel, kernel):
    return len(mandel.KERNELS[kernel]) > 2 and mandel.KERNELS[kernel][2] > 1


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("dtype", ["fp64", "fp32", "fp64fma"])
@pytest.mark.parametrize("scheme", SCHEMES)
@pytest.mark.parametrize("ngpus", [1, 2, 3, 5, 8])
def test_c1_all_schemes(mandel, oracle, dtype, scheme, ngpus, kernel):
    cfg = wl.C1.with_(dtype=dtype)
    if dtype == "fp32" and kernel.startswith("batch16"):
        with pytest.raises(mandel.MandelError):  # fp32 allows check_every <= 8 (R18)
            _render_dev(mandel, cfg, scheme, 1, kernel=kernel)
        return
    want = oracle.render(cfg)
    out, st = _render_dev(mandel, cfg, scheme, ngpus, kernel=kernel,
                          refill_lanes=[0, 1, 5, 32][ngpus % 4])
    _assert_same(_host(out), want, f"C1/{dtype}/{scheme}/N={ngpus}")
    assert st["sum_iters"] == int(want.sum(dtype=np.uint64))
    assert st["pixels"] == cfg.pixels
    assert st["kernel_launches"] == ngpus
    assert st["kernel_scheme"] == scheme  # the row order the kernels ran is the one requested
    assert 300 < st["sm_clock_mhz"] < 2500, st["sm_clock_mhz"]  # measured in-kernel
    if scheme == "fcfs":
        # Eq. 19 analog: ceil(H/16) successful claims, counted by the device's claim atomics
        # (also at N = 1: one claimant still claims every chunk from the counter)
        assert st["chunks_claimed"] == -(-cfg.H // 16)
        assert sum(st["rank_rows"]) == cfg.H
    else:
        assert st["transfers"] == ngpus - 1  # Eq. 18 / Eq. 20: T_m = N - 1
        assert st["rank_rows"] == [len(x) for x in (
            mandel.mandel_plan_rows(scheme, cfg.H, ngpus, r) for r in range(ngpus))]


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
@pytest.mark.parametrize("scheme", ["block", "cyclic"])
def test_static_kernel_variant(mandel, oracle, dtype, scheme):
    cfg = wl.C1.with_(dtype=dtype, W=813, H=611)
    out, st = _render_dev(mandel, cfg, scheme, 3, kernel=mandel.MANDEL_KERNEL_STATIC)
    _assert_same(_host(out), oracle.render(cfg), f"static/{dtype}/{scheme}")


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("dtype", ["fp64", "fp32", "fp64fma"])
def test_random_small_configs(mandel, oracle, dtype, kernel):
    if dtype == "fp32" and kernel.startswith("batch16"):
        kernel = "batch8x" + kernel[-1]
    for k, cfg in enumerate(wl.random_small_configs(50, 0, dtype)):
        want = oracle.render(cfg)
        scheme = SCHEMES[k % 3]
        ngpus = [1, 2, 3, 4, 5, 8][k % 6]
        if scheme != "fcfs" and cfg.H < ngpus:
            ngpus = 1
        ce = 1 if (_batched(mandel, kernel) and cfg.R < 2.0) else 0  # R18 needs R >= 2
        out, st = _render_dev(mandel, cfg, scheme, ngpus, tile_px=[0, 1, 7, 32, 33][k % 5],
                              chunk_rows=[0, 1, 3][k % 3], kernel=kernel,
                              refill_lanes=[0, 1, 3, 16, 32][k % 5], check_every=ce,
                              tile_rows=[0, 1, 2, 4, 8, 16, 32][k % 7])
        _assert_same(_host(out), want, f"{cfg.name}/{dtype}/{scheme}/N={ngpus}")
        assert st["sum_iters"] == int(want.sum(dtype=np.uint64))


EDGE = [
    wl.Config("1x1", -2.5, 1.5, -2.0, 2.0, 1, 1, 50, 2.0, "fp64"),
    wl.Config("1xH", -0.8, -0.7, -0.2, 0.2, 1, 97, 300, 2.0, "fp64"),
    wl.Config("Wx1", -2.5, 1.5, 0.0, 0.01, 1025, 1, 300, 2.0, "fp64"),
    wl.Config("ragged", -2.2, 0.8, -1.3, 1.1, 257, 33, 500, 2.0, "fp64"),
    wl.Config("it1", -2.5, 1.5, -2.0, 2.0, 64, 64, 1, 2.0, "fp64"),
    wl.Config("it2", -2.5, 1.5, -2.0, 2.0, 64, 64, 2, 2.0, "fp32"),
    # iterMax just off the LAZY block length (16) and the batch lengths: counts capped
    # inside a block, escapes in the same block as the cap
    wl.Config("it17", -2.2, 0.8, -1.3, 1.3, 96, 70, 17, 2.0, "fp64"),
    wl.Config("it33_f32", -2.2, 0.8, -1.3, 1.3, 96, 70, 33, 2.0, "fp32"),
    wl.Config("it15_fma", -0.76, -0.73, 0.09, 0.12, 80, 60, 15, 2.0, "fp64fma"),
    wl.Config("far", -1e300, 1e300, -1e300, 1e300, 40, 40, 100, 2.0, "fp64"),
    wl.Config("R20", -2.5, 1.5, -2.0, 2.0, 120, 90, 2000, 20.0, "fp64"),
    wl.Config("Rsmall", -1.0, 0.5, -0.7, 0.7, 100, 100, 400, 0.75, "fp32"),
    wl.Config("tiny", -0.7436439, -0.7436438, 0.1318259, 0.131826, 64, 64, 3000, 2.0, "fp64"),
]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("cfg", EDGE, ids=[c.name for c in EDGE])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_edge_cases(mandel, oracle, cfg, scheme, kernel):
    if _batched(mandel, kernel) and (cfg.R < 2.0 or (cfg.dtype == "fp32" and kernel.startswith("batch16"))):
        # the batched check is only valid for R >= 2, and fp32 for <= 8 updates (R18):
        # requesting it otherwise is an error
        with pytest.raises(mandel.MandelError):
            _render_dev(mandel, cfg, scheme, 1, kernel=kernel)
        return
    want = oracle.render(cfg)
    for ngpus in (1, 4):
        if scheme != "fcfs" and cfg.H < ngpus:
            continue
        out, st = _render_dev(mandel, cfg, scheme, ngpus, kernel=kernel)
        got = _host(out)
        _assert_same(got, want, f"{cfg.name}/{scheme}/N={ngpus}")
        assert got.min() >= 1 and got.max() <= cfg.iter_max
        assert st["pixels"] == cfg.pixels


# The batched escape check (R18) on the orbits that stress its argument:
# escapes by a hair (|z|^2 just above R^2, the real axis just left of c = -2 where
# the escaped orbit grows slowest), orbits that touch |z|^2 = R^2 without escaping
# (c = -2), escapes that overflow to inf/NaN inside a batch (huge R), and R = 2
# exactly vs just below 2 (where the library must fall back to the per-update test).
BATCH_CASES = [
    wl.Config("left_of_-2", -2.0 - 2e-15, -2.0 + 2e-15, -1e-300, 1e-300, 97, 5, 5000, 2.0, "fp64"),
    wl.Config("left_of_-2_f32", -2.0000010, -1.9999990, -1e-30, 1e-30, 97, 5, 5000, 2.0, "fp32"),
    wl.Config("near_-2_row", -2.05, -1.95, -1e-9, 1e-9, 256, 8, 20000, 2.0, "fp64"),
    wl.Config("hugeR", -2.5, 1.5, -2.0, 2.0, 96, 80, 60, 1e150, "fp64"),
    wl.Config("hugeR_f32", -2.5, 1.5, -2.0, 2.0, 96, 80, 60, 1e18, "fp32"),
    wl.Config("R20_seahorse", -0.76, -0.73, 0.09, 0.12, 200, 150, 4000, 20.0, "fp64"),
    wl.Config("R2_fma", -0.76, -0.73, 0.09, 0.12, 200, 150, 4000, 2.0, "fp64fma"),
]


@pytest.mark.parametrize("kernel", ["refill", "batch4x1", "batch4x2", "batch8x2", "batch8x4",
                                    "batch16x1", "batch16x2", "adaptb8x2", "adaptb4x1"])
@pytest.mark.parametrize("cfg", BATCH_CASES, ids=[c.name for c in BATCH_CASES])
def test_batched_check_adversarial(mandel, oracle, cfg, kernel):
    if cfg.dtype == "fp32" and kernel.startswith("batch16"):
        kernel = "batch8x" + kernel[-1]
    want = oracle.render(cfg)
    for scheme, ngpus in (("fcfs", 1), ("cyclic", 3)):
        out, st = _render_dev(mandel, cfg, scheme, ngpus, kernel=kernel, tile_px=[0, 16][ngpus % 2])
        _assert_same(_host(out), want, f"{cfg.name}/{kernel}/{scheme}")
        assert st["sum_iters"] == int(want.sum(dtype=np.uint64))
        if kernel != "refill":
            assert st["kernel_batch"] == mandel.KERNELS[kernel][2]


@pytest.mark.parametrize("tile_rows", [1, 2, 4, 8, 16, 64])
@pytest.mark.parametrize("kernel", ["refill", "refill1", "lazy2", "adaptive2", "batch8x2", "adaptb8x2"])
@pytest.mark.parametrize("scheme", ["block", "cyclic", "fcfs"])
def test_tile_rows(mandel, oracle, tile_rows, kernel, scheme):
    # 2-D tiles: tile_rows row slots streamed in 8-column blocks; ragged in both directions
    cfg = wl.C1.with_(W=203, H=77, iter_max=600)
    want = oracle.render(cfg)
    for ngpus, tile_px, chunk in ((1, 0, 0), (3, 100, 0), (2, 37, 4), (5, 512, 3)):
        out, st = _render_dev(mandel, cfg, scheme, ngpus, kernel=kernel, tile_rows=tile_rows,
                              tile_px=tile_px, chunk_rows=chunk)
        _assert_same(_host(out), want, f"tile_rows={tile_rows}/{kernel}/{scheme}/N={ngpus}")
        assert st["sum_iters"] == int(want.sum(dtype=np.uint64)) and st["pixels"] == cfg.pixels
        if scheme != "fcfs":
            assert st["rank_rows"] == [len(x) for x in (
                mandel.mandel_plan_rows(scheme, cfg.H, ngpus, r) for r in range(ngpus))]
        else:
            assert sum(st["rank_rows"]) == cfg.H


def test_tile_rows_invalid(mandel):
    cfg = wl.C1.with_(W=64, H=64)
    for bad in (3, 6, 128):
        with pytest.raises(mandel.MandelError):
            _render_dev(mandel, cfg, "block", 1, tile_rows=bad)


@pytest.mark.parametrize("kernel", ["batch4x2", "batch8x2", "batch8x3", "batch8x4", "batch4x4"])
def test_fp32_packed_loop(mandel, oracle, kernel):
    # NEXT-4b: the fp32 batched loop on FADD2/FMUL2 slot pairs is bit-identical to the
    # scalar loop and the oracle (odd ILP packs all but the last slot)
    for k, cfg in enumerate(wl.random_small_configs(20, 7, "fp32")):
        if cfg.R < 2.0:
            cfg = cfg.with_(R=2.0)
        want = oracle.render(cfg)
        for no_pack in (False, True):
            out, st = _render_dev(mandel, cfg, ["fcfs", "block", "cyclic"][k % 3], 1 + k % 3,
                                  kernel=kernel, no_pack=no_pack, tile_rows=[1, 8][k % 2])
            _assert_same(_host(out), want, f"{cfg.name}/{kernel}/no_pack={no_pack}")
            assert st["kernel_packed"] == (0 if no_pack else 1)
    cfg = wl.C1.with_(dtype="fp32", iter_max=3000)
    out, _ = _render_dev(mandel, cfg, "fcfs", 1, kernel=kernel)
    _assert_same(_host(out), oracle.render(cfg), f"C1 fp32 packed {kernel}")


@pytest.mark.parametrize("R,batch", [(2.0, 8), (1.9999999999999998, 1), (1.5, 1), (20.0, 8)])
def test_batched_check_default_and_fallback(mandel, oracle, R, batch):
    # the default EAGER loop (an explicit ilp skips the per-view choice, which may pick LAZY):
    # batched when R >= 2, the per-update test otherwise (same map either way)
    cfg = wl.C1.with_(W=300, H=200, R=R)
    out, st = _render_dev(mandel, cfg, "fcfs", 1, ilp=2)
    _assert_same(_host(out), oracle.render(cfg), f"default R={R}")
    assert st["kernel"] == "eager" and st["kernel_batch"] == batch
    if batch == 1:
        with pytest.raises(mandel.MandelError):
            _render_dev(mandel, cfg, "fcfs", 1, check_every=4)


@pytest.mark.parametrize("ngpus", [2, 3, 5, 8])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_fcfs_master_worker(mandel, oracle, ngpus, dtype):
    # the paper's FCFS: the master computes no rows, workers claim rows
    cfg = wl.C1.with_(dtype=dtype, W=517, H=301)
    out, st = _render_dev(mandel, cfg, "fcfs_master", ngpus)
    _assert_same(_host(out), oracle.render(cfg), f"fcfs_master/N={ngpus}")
    assert st["rank_rows"][0] == 0 and st["rank_pixels"][0] == 0
    assert sum(st["rank_rows"]) == cfg.H
    assert st["chunks_claimed"] == cfg.H          # one claim per row
    assert st["transfers"] == cfg.H               # every row is sent to the master (Eq. 19: 2 H)
    if ngpus == 2:
        assert st["rank_rows"][1] == cfg.H        # one worker does everything


def test_fcfs_more_ranks_than_rows(mandel, oracle):
    cfg = wl.Config("fewrows", -2.5, 1.5, -2.0, 2.0, 300, 3, 200, 2.0, "fp64")
    out, st = _render_dev(mandel, cfg, "fcfs", 8, chunk_rows=1)
    _assert_same(_host(out), oracle.render(cfg), "fcfs N>H")
    assert st["chunks_claimed"] == 3


@pytest.mark.parametrize("chunk", [1, 5, 16, 0])
def test_single_rank_fcfs_claims_are_counted(mandel, oracle, chunk):
    """At N = 1 FCFS really claims: the device counts ceil(H/chunk) successful claims
    (the count used to be synthesised while the block order ran).  The
    pipelined host hand-off renders row bands instead and says so (kernel_scheme block,
    no claims)."""
    cfg = wl.C1.with_(W=257, H=203, iter_max=500)
    want = oracle.render(cfg)
    out, st = _render_dev(mandel, cfg, "fcfs", 1, chunk_rows=chunk)
    _assert_same(_host(out), want, f"fcfs N=1 chunk={chunk}")
    c = chunk or 16
    assert st["chunks_claimed"] == -(-cfg.H // c)
    assert st["kernel_scheme"] == "fcfs" and st["rank_rows"] == [cfg.H]
    got, st = mandel.render(*cfg.args(), "fp64", "fcfs", 1, bands=4, chunk_rows=chunk)
    _assert_same(got, want, "banded")
    assert st["kernel_scheme"] == "block" and st["chunks_claimed"] == 0 and st["kernel_launches"] == 4


def test_host_output_entry_point(mandel, oracle):
    cfg = wl.C1.with_(W=640, H=480)
    out = np.zeros(cfg.pixels, dtype=np.uint32)
    mandel.mandel_render(*cfg.args(), "fp64", "cyclic", 1, out)
    _assert_same(out.reshape(cfg.H, cfg.W), oracle.render(cfg), "mandel_render host out")
    got, st = mandel.render(*cfg.args(), "fp32", "fcfs", 1)
    _assert_same(got, oracle.render(cfg.with_(dtype="fp32")), "render fp32")
    assert st["d2h_ms"] > 0


@pytest.mark.parametrize("H", [200, 201, 233, 96])
def test_pipelined_band_state_alignment(mandel, oracle, H):
    # band states are packed back to back: odd chunk-map lengths must not misalign the
    # next band's 64-bit counters (H = 200: 13 FCFS chunks)
    cfg = wl.C1.with_(W=150, H=H, iter_max=300)
    want = oracle.render(cfg)
    for scheme in SCHEMES:
        got, st = mandel.render(*cfg.args(), "fp64", scheme, 1, bands=7)
        _assert_same(got, want, f"H={H}/{scheme}")


@pytest.mark.parametrize("taper", [0, 30, 70, 100])
@pytest.mark.parametrize("bands", [2, 5, 12, 32])
def test_pipelined_band_taper(mandel, oracle, taper, bands):
    # tapered outside-in bands (thin middle bands, some empty at 32 bands) still cover
    # every row exactly once
    cfg = wl.C1.with_(W=211, H=307 if bands < 32 else 70, iter_max=500)
    want = oracle.render(cfg)
    for rep in range(2):  # the second render uses the view's cached compute time
        got, st = mandel.render(*cfg.args(), "fp64", "fcfs", 1, bands=bands, band_taper=taper)
        _assert_same(got, want, f"bands={bands}/taper={taper}/rep={rep}")
        assert st["sum_iters"] == int(want.sum(dtype=np.uint64)) and st["pixels"] == cfg.pixels


@pytest.mark.parametrize("bands", [0, 1, 2, 3, 7, 32])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_pipelined_host_output(mandel, oracle, bands, scheme):
    # one GPU + host destination: row bands copied to the host while later bands compute
    cfg = wl.C1.with_(W=333, H=251, iter_max=700)
    want = oracle.render(cfg)
    got, st = mandel.render(*cfg.args(), "fp64", scheme, 1, bands=bands)
    _assert_same(got, want, f"bands={bands}/{scheme}")
    assert st["sum_iters"] == int(want.sum(dtype=np.uint64)) and st["pixels"] == cfg.pixels
    assert st["kernel_launches"] == (1 if bands == 1 else (bands or 8))


def test_repeat_is_deterministic(mandel):
    cfg = wl.C1.with_(iter_max=1000)
    a, _ = _render_dev(mandel, cfg, "fcfs", 1)
    for scheme, n in (("fcfs", 3), ("block", 1), ("cyclic", 4), ("fcfs", 1)):
        b, _ = _render_dev(mandel, cfg, scheme, n)
        assert bool((a == b).all()), (scheme, n)


# ---------------------------------------------------------------------------
# full-size configurations, in bench.py's launch configuration (1 GPU, FCFS)
# ---------------------------------------------------------------------------
def _sampled_rows_check(oracle, cfg, out, nrows, seed):
    rows = wl.sample_rows(cfg.H, nrows, seed, include=(0, 1, cfg.H // 2 - 1))
    got = _host(out[rows.tolist()])
    want, _ = oracle.render_rows_mt(cfg, rows)
    _assert_same(got, want, f"{cfg.name} sampled rows")


def _properties(oracle, cfg, out, st):
    torch = _torch()
    assert int(out.min()) >= 1 and int(out.max()) <= cfg.iter_max  # coverage of a 0-prefill
    total = int(out.to(torch.int64).sum())
    assert st["sum_iters"] == total
    assert st["pixels"] == cfg.pixels


def _whole_map_check(oracle, cfg, out, band_rows):
    """Every pixel of the device map ``out`` against the oracle, in row bands (bounded
    host memory): the oracle renders each band on all host threads (render_rows_mt, pinned
    to render_rows in test_oracle_pins) while the next band is still on the device.
    Reports the mismatch count over the whole map and the first mismatching pixel."""
    bad, first = 0, None
    for r0 in range(0, cfg.H, band_rows):
        r1 = min(cfg.H, r0 + band_rows)
        got = _host(out[r0:r1])
        want, _ = oracle.render_rows_mt(cfg, np.arange(r0, r1))
        diff = got != want
        nb = int(diff.sum())
        if nb:
            if first is None:
                i, j = np.argwhere(diff)[0]
                first = (r0 + int(i), int(j), int(got[i, j]), int(want[i, j]))
            bad += nb
    assert bad == 0, (f"{cfg.name}: {bad} of {cfg.pixels} pixels differ; first at (i, j) = "
                      f"({first[0]}, {first[1]}): gpu={first[2]} oracle={first[3]}")


# The north_star's parity target: bit-exact uint32 maps on all five configs, every pixel
# (Eq. 2 defines I_{i,j} for each pixel).  C1 is whole in the tests above;
# C2-C5 here, rendered in bench.py's launch configuration (1 GPU, FCFS, default kernel:
# the per-view EAGER/LAZY choice), plus the other kernel where the oracle is cheap.
WHOLE = [("C2", "refill"), ("C2", "lazy2"), ("C3", "refill"), ("C4", "refill"), ("C4", "batch8x2"),
         ("C5", "refill")]


@pytest.mark.slow
@pytest.mark.parametrize("name,kernel", WHOLE, ids=[f"{n}-{k}" for n, k in WHOLE])
def test_full_size_whole_map(mandel, oracle, name, kernel):
    torch = _torch()
    cfg = wl.CONFIGS[name]
    out, st = _render_dev(mandel, cfg, "fcfs", 1, kernel=kernel)
    _properties(oracle, cfg, out, st)
    if kernel == "refill":
        # the per-view choice the bench runs: LAZY on C4's zoom, batched EAGER elsewhere
        assert st["kernel"] == ("lazy" if name == "C4" else "eager"), st["kernel"]
    _whole_map_check(oracle, cfg, out, band_rows=2048 if cfg.W <= 16384 else 1024)
    del out
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("kernel", ["refill", "lazy2", "refill2", "batch4x2"])
@pytest.mark.parametrize("name,nrows", [("C2", 48), ("C3", 48), ("C4", 16)])
def test_full_size_sampled(mandel, oracle, name, nrows, kernel):
    cfg = wl.CONFIGS[name]
    out, st = _render_dev(mandel, cfg, "fcfs", 1, kernel=kernel)
    _properties(oracle, cfg, out, st)
    _sampled_rows_check(oracle, cfg, out, nrows, seed=sum(map(ord, name)))
    if name in ("C2", "C3"):
        # exact mirror rows (rows i and H-i with bitwise-opposite Cy are identical)
        _, cy = oracle.axes(*cfg.args()[:4], 1, cfg.H, cfg.R, cfg.dtype)
        pairs = [(i, cfg.H - i) for i in range(1, cfg.H) if cy[i] == -cy[cfg.H - i]]
        assert len(pairs) > 100
        a = out[[p[0] for p in pairs]]
        b = out[[p[1] for p in pairs]]
        assert bool((a == b).all())


@pytest.mark.slow
@pytest.mark.parametrize("kernel", ["refill", "lazy2"])
def test_zoom_fma_sampled(mandel, oracle, kernel):
    # the FMA dtype where it differs from fp64 (C4's zoom), full size, sampled rows
    cfg = wl.C4.with_(dtype="fp64fma")
    out, st = _render_dev(mandel, cfg, "fcfs", 1, kernel=kernel)
    _properties(oracle, cfg, out, st)
    _sampled_rows_check(oracle, cfg, out, 12, seed=17)


@pytest.mark.slow
def test_c5_decimation_and_rows(mandel, oracle):
    torch = _torch()
    cfg = wl.C5
    out, st = _render_dev(mandel, cfg, "fcfs", 1)
    _properties(oracle, cfg, out, st)
    # c is an exact dyadic on 32768^2 over [-2.5,1.5]x[-2,2]: every 32nd pixel is the 1024^2 map
    small = wl.Config("C5/32", *wl.FULL_PLANE, 1024, 1024, cfg.iter_max, cfg.R, "fp64")
    want, _ = oracle.render_rows_mt(small, np.arange(1024))
    _assert_same(_host(out[::32, ::32].contiguous()), want, "C5[::32, ::32]")
    _sampled_rows_check(oracle, cfg, out, 12, seed=5)
    del out
    torch.cuda.empty_cache()


@pytest.mark.slow
@pytest.mark.parametrize("scheme", SCHEMES)
def test_c2_schemes_agree(mandel, scheme):
    ref, _ = _render_dev(mandel, wl.C2, "fcfs", 1)
    out, st = _render_dev(mandel, wl.C2, scheme, 8)
    assert bool((ref == out).all())
    assert st["pixels"] == wl.C2.pixels


@pytest.mark.parametrize("max_sms", [1, 3, 16])
@pytest.mark.parametrize("scheme", SCHEMES + ["fcfs_master"])
def test_max_sms_slices(mandel, oracle, max_sms, scheme):
    # ranks as fixed GPU slices (one CTA per SM, the paper-table tool's tasks)
    cfg = wl.C1.with_(W=257, H=131, iter_max=700)
    want = oracle.render(cfg)
    for ngpus in (2, 5):
        out, st = _render_dev(mandel, cfg, scheme, ngpus, max_sms=max_sms,
                              kernel=["refill", "lazy2"][ngpus % 2])
        _assert_same(_host(out), want, f"max_sms={max_sms}/{scheme}/N={ngpus}")
        assert st["sum_iters"] == int(want.sum(dtype=np.uint64))


def test_concurrent_call_is_ebusy(mandel, oracle):
    # calls are not reentrant (include/mandel.h): a second call while one runs -> EBUSY
    import threading
    big = wl.C2.with_(iter_max=20000)           # ~50 ms of device time per render
    small = wl.C1.with_(W=64, H=48, iter_max=100)
    codes, started = [], threading.Event()

    def long_render():
        out = np.zeros(big.pixels, dtype=np.uint32)
        started.set()
        mandel.mandel_render_ex(*big.args(), "fp64", "fcfs", 1, out_host=out)

    seen_busy = False
    for _ in range(5):
        t = threading.Thread(target=long_render)
        started.clear()
        t.start()
        started.wait()
        for _ in range(200):
            try:
                got, _ = mandel.render(*small.args(), "fp64", "block", 1)
                codes.append(0)
                _assert_same(got, oracle.render(small), "render beside a busy library")
            except mandel.MandelError as e:
                assert e.code == mandel.MANDEL_EBUSY
                seen_busy = True
                break
        t.join()
        if seen_busy:
            break
    assert seen_busy


def test_shutdown_and_reuse(mandel, oracle):
    cfg = wl.C1.with_(W=300, H=200)
    want = oracle.render(cfg)
    for _ in range(3):
        got, st = mandel.render(*cfg.args(), "fp64", "fcfs", 1)
        _assert_same(got, want, "after shutdown")
        mandel.mandel_shutdown()
    mandel.mandel_shutdown()  # idempotent
    out, st = _render_dev(mandel, cfg, "cyclic", 3)
    _assert_same(_host(out), want, "device output after shutdown")


def test_largest_iter_max(mandel, oracle):
    # iterMax = 2^32 - 2 (the largest accepted): a window outside the set, every pixel
    # escapes at its first updates, counts exact
    cfg = wl.Config("far_out", 2.1, 2.9, 2.1, 2.5, 77, 33, 0xFFFFFFFE, 2.0, "fp64")
    want = oracle.render(cfg)
    for kernel in ("refill", "lazy2", "refill1", "batch16x2"):
        out, st = _render_dev(mandel, cfg, "fcfs", 1, kernel=kernel)
        _assert_same(_host(out), want, f"iterMax 2^32-2/{kernel}")


@pytest.mark.slow
def test_more_than_2_32_pixels(mandel, oracle):
    # 70000 x 65000 = 4.55e9 pixels (18.2 GB map): 64-bit pixel offsets and counters
    torch = _torch()
    cfg = wl.Config("huge", -2.5, 1.5, -2.0, 2.0, 70000, 65000, 6, 2.0, "fp64")
    out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device="cuda:0")
    st = mandel.mandel_render_ex(*cfg.args(), "fp64", "fcfs", 1, out_dev0=out)
    assert st["pixels"] == cfg.pixels
    assert int(out.min()) >= 1 and int(out.max()) <= cfg.iter_max
    assert st["sum_iters"] == int(out.to(torch.int64).sum())
    rows = [0, 1, 32499, 32500, 64998, 64999]
    want, _ = oracle.render_rows_mt(cfg, np.array(rows))
    _assert_same(_host(out[rows]), want, "rows of a 4.55e9-pixel map")
    del out
    torch.cuda.empty_cache()


def test_max_logical_ranks(mandel, oracle):
    cfg = wl.C1.with_(W=97, H=130, iter_max=400)
    want = oracle.render(cfg)
    for scheme in ("fcfs", "cyclic", "block", "fcfs_master"):
        out, st = _render_dev(mandel, cfg, scheme, mandel.MANDEL_MAX_GPUS)
        _assert_same(_host(out), want, f"{mandel.MANDEL_MAX_GPUS} ranks/{scheme}")
        assert st["kernel_launches"] == mandel.MANDEL_MAX_GPUS
    with pytest.raises(mandel.MandelError) as e:
        _render_dev(mandel, cfg, "fcfs", mandel.MANDEL_MAX_GPUS + 1)
    assert e.value.code == mandel.MANDEL_ENODEV


def test_async_host_pipeline(mandel, oracle):
    # options.async_host: calls return once enqueued, consecutive renders overlap
    # (alternate library maps); every host buffer is complete after mandel_finish
    views = [wl.C1.with_(W=301, H=211, iter_max=600), wl.C1.with_(W=128, H=96, iter_max=2000, dtype="fp32"),
             wl.Config("zoom", -0.7437, -0.7435, 0.1317, 0.1319, 160, 120, 3000, 2.0, "fp64"),
             wl.C1.with_(W=301, H=211, iter_max=600)]
    outs = [np.zeros((v.H, v.W), np.uint32) for v in views]
    for v, o in zip(views, outs):
        r = mandel.mandel_render_ex(*v.args(), v.dtype, "fcfs", 1, out_host=o, async_host=True,
                                    want_stats=False, bands=[0, 3, 1, 5][len(v.name) % 4])
        assert r is None
    # a synchronous call in between is ordered with the asynchronous ones
    got, _ = mandel.render(*views[0].args(), "fp64", "cyclic", 1)
    _assert_same(got, oracle.render(views[0]), "sync between async")
    mandel.mandel_finish()
    for v, o in zip(views, outs):
        _assert_same(o, oracle.render(v), f"async {v.name}/{v.dtype}")
    # one host buffer reused by a stream of renders of one view
    v = views[0]
    o = np.zeros((v.H, v.W), np.uint32)
    for _ in range(6):
        mandel.mandel_render_ex(*v.args(), "fp64", "fcfs", 1, out_host=o, async_host=True, want_stats=False)
    mandel.mandel_finish()
    _assert_same(o, oracle.render(v), "async reuse")


def test_async_host_rejects_misuse(mandel):
    torch = _torch()
    v = wl.C1.with_(W=64, H=64)
    o = np.zeros((v.H, v.W), np.uint32)
    with pytest.raises(mandel.MandelError):  # statistics need a synchronous call
        mandel.mandel_render_ex(*v.args(), "fp64", "fcfs", 1, out_host=o, async_host=True)
    d = torch.zeros((v.H, v.W), dtype=torch.int32, device="cuda:0")
    with pytest.raises(mandel.MandelError):  # library-owned maps only
        mandel.mandel_render_ex(*v.args(), "fp64", "fcfs", 1, out_host=o, out_dev0=d, async_host=True,
                                want_stats=False)
    with pytest.raises(mandel.MandelError):
        mandel.mandel_render_ex(*v.args(), "fp64", "fcfs", 2, out_host=o, async_host=True, want_stats=False,
                                logical_ranks=True)
    mandel.mandel_finish()


@pytest.mark.gpu
def test_view_probe_ignores_sm_slicing(mandel, oracle):
    """The EAGER/LAZY view probe characterises the view, not the launch: with
    options.max_sms it still runs on the whole GPU (its calibration geometry), so a
    sliced first render makes the same choice from the same statistic as a whole-GPU
    one (on a 4-SM slice the sample had no drain phase and read fewer iterations per
    exit: the paper grid picked LAZY, 16% slower there)."""
    cfg = wl.Config("probe", -2.5, 1.5, -2.0, 2.0, 2048, 2048, 2000, 20.0, "fp64")
    got = []
    for kw in ({"max_sms": 4}, {}):
        mandel.mandel_shutdown()  # clears the per-view choice cache
        out, st = _render_dev(mandel, cfg, "block", 1, **kw)
        got.append((st["kernel"], st["probe"][1]))
    (k0, ipe0), (k1, ipe1) = got
    assert k0 == k1, got
    assert abs(ipe0 - ipe1) <= 0.1 * ipe1, got


def test_explicit_ilp_and_budget_honoured(mandel, oracle):
    """options.ilp / min_ctas apply on top of the per-view kernel choice in both entry
    points (mandel_render_ex ignored them under MANDEL_KERNEL_REFILL)."""
    torch = _torch()
    cfg = wl.C1.with_(W=400, H=300, iter_max=900)
    want = oracle.render(cfg)
    for ilp, minb in ((1, 0), (4, 0), (2, 1), (1, 3)):
        out, st = _render_dev(mandel, cfg, "fcfs", 1, ilp=ilp, min_ctas=minb)
        _assert_same(_host(out), want, f"ilp={ilp}/min_ctas={minb}")
        assert st["kernel_ilp"] == ilp, st
        img = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device="cuda:0")
        ctr = torch.zeros(4, dtype=torch.int32, device="cuda:0")
        st = mandel.mandel_render_rank(*cfg.args(), "fp64", "fcfs", 0, 1, img, ctr, None, ilp=ilp, min_ctas=minb)
        _assert_same(_host(img), want, f"rank ilp={ilp}")
        assert st["kernel_ilp"] == ilp, st


def test_enqueued_renders_on_two_streams(mandel, oracle):
    """Enqueue-only renders (device output, no statistics) on different streams reuse the
    library's cached tile counter and rank state; the second must not reset them while
    the first still draws tiles."""
    torch = _torch()
    a = wl.C1.with_(W=1500, H=1400, iter_max=6000)
    b = wl.C1.with_(W=900, H=700, iter_max=3000, xmin=-2.0, xmax=0.5)
    wa, wb = oracle.render(a), oracle.render(b)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for rep in range(3):
        oa = torch.zeros((a.H, a.W), dtype=torch.int32, device="cuda:0")
        ob = torch.zeros((b.H, b.W), dtype=torch.int32, device="cuda:0")
        torch.cuda.synchronize()
        for scheme, n in (("fcfs", 1), ("cyclic", 3))[rep % 2:rep % 2 + 1]:
            mandel.mandel_render_ex(*a.args(), "fp64", scheme, n, out_dev0=oa, stream0=s1.cuda_stream,
                                    logical_ranks=n > 1, want_stats=False)
            mandel.mandel_render_ex(*b.args(), "fp64", scheme, n, out_dev0=ob, stream0=s2.cuda_stream,
                                    logical_ranks=n > 1, want_stats=False)
        torch.cuda.synchronize()
        _assert_same(_host(oa), wa, f"stream 1 rep {rep}")
        _assert_same(_host(ob), wb, f"stream 2 rep {rep}")
    # the same through mandel_render_rank (the multi-process entry point)
    oa = torch.zeros((a.H, a.W), dtype=torch.int32, device="cuda:0")
    ob = torch.zeros((b.H, b.W), dtype=torch.int32, device="cuda:0")
    ca = torch.zeros(4, dtype=torch.int32, device="cuda:0")
    cb = torch.zeros(4, dtype=torch.int32, device="cuda:0")
    torch.cuda.synchronize()
    mandel.mandel_render_rank(*a.args(), "fp64", "fcfs", 0, 1, oa, ca, s1.cuda_stream, want_stats=False)
    mandel.mandel_render_rank(*b.args(), "fp64", "fcfs", 0, 1, ob, cb, s2.cuda_stream, want_stats=False)
    torch.cuda.synchronize()
    _assert_same(_host(oa), wa, "rank stream 1")
    _assert_same(_host(ob), wb, "rank stream 2")


STAGE_CASES = [
    # (label, config, options, expected store mode)
    ("aligned", wl.C1.with_(W=640, H=480, iter_max=3000), {"stage": 1}, "staged_vec"),
    ("W%4", wl.C1.with_(W=641, H=233, iter_max=3000), {"stage": 1}, "staged"),
    ("tile_rows1", wl.C1.with_(W=512, H=97, iter_max=2000), {"stage": 1, "tile_rows": 1}, "staged_vec"),
    ("tiny_tiles", wl.C1.with_(W=96, H=77, iter_max=2000), {"stage": 1, "tile_px": 1, "tile_rows": 1}, "staged"),
    ("tile_px7", wl.C1.with_(W=203, H=64, iter_max=900), {"stage": 1, "tile_px": 7}, "staged"),
    ("direct", wl.C1.with_(W=640, H=480, iter_max=3000), {"stage": -1}, "direct"),
    # default: the map is this GPU's own HBM (logical ranks share the device) -> direct
    ("auto_local", wl.C1.with_(W=640, H=480, iter_max=3000), {}, "direct"),
    # interior-heavy: slow interior pixels hold their 8x8 blocks while the stream moves on,
    # so ring entries are evicted (partial blocks stored, the rest stored directly)
    ("evict", wl.Config("evict", -0.9, 0.3, -0.6, 0.6, 512, 384, 20000, 2.0, "fp64"), {"stage": 1}, "staged_vec"),
    ("evict_f32", wl.Config("evict", -0.9, 0.3, -0.6, 0.6, 512, 384, 20000, 2.0, "fp32"), {"stage": 1},
     "staged_vec"),
]


@pytest.mark.parametrize("kernel", ["refill", "batch8x2", "batch8x1", "batch8x4", "lazy2", "lazy1"])
@pytest.mark.parametrize("case", STAGE_CASES, ids=[c[0] for c in STAGE_CASES])
def test_store_staging(mandel, oracle, case, kernel):
    """Coalesced, vectorised stores (north_star): counts are staged per
    8x8 block in shared memory and whole blocks stored as 32-B rows with 16-B stores;
    misaligned maps and narrow blocks store count by count, evicted blocks partly
    directly.  Every mode gives the oracle's map, for every scheme and a misaligned
    destination."""
    torch = _torch()
    label, cfg, opts, mode = case
    want = oracle.render(cfg)
    for scheme, n in (("block", 1), ("fcfs", 1), ("cyclic", 3), ("fcfs", 4)):
        out, st = _render_dev(mandel, cfg, scheme, n, kernel=kernel, **opts)
        _assert_same(_host(out), want, f"{label}/{kernel}/{scheme}/N={n}")
        assert st["store_mode"] == mode, (label, st["store_mode"])
    # a destination 4 bytes past a 16-B boundary: staged, but no vector stores
    buf = torch.zeros(cfg.pixels + 4, dtype=torch.int32, device="cuda:0")
    st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 1, out_dev0=buf.data_ptr() + 4,
                                 kernel=kernel, **opts)
    got = buf[1:1 + cfg.pixels].reshape(cfg.H, cfg.W)
    _assert_same(_host(got), want, f"{label}/{kernel}/misaligned")
    assert int(buf[0]) == 0 and int(buf[1 + cfg.pixels]) == 0  # nothing outside the map
    assert st["store_mode"] == ("direct" if mode == "direct" else "staged")


def test_store_staging_variants_without_instantiation(mandel, oracle):
    """stage = 1 on a kernel with no staged instantiation (per-update EAGER, check every 4,
    ADAPTIVE, static) stores directly and says so."""
    cfg = wl.C1.with_(W=320, H=200, iter_max=1500)
    want = oracle.render(cfg)
    for kernel in ("refill1", "batch4x2", "adaptive2", "static"):
        out, st = _render_dev(mandel, cfg, "block", 2, kernel=kernel, stage=1)
        _assert_same(_host(out), want, kernel)
        assert st["store_mode"] == "direct", (kernel, st["store_mode"])


def test_back_to_back_renders_reset_state_in_kernel(mandel, oracle):
    """Consecutive renders need no host memset: each launch's first CTA zeroes the other
    half of the rank's work state and the other FCFS counter word for the next render.
    Enqueued renders of different sizes (a larger chunk map falls back to a host memset),
    schemes, rank counts and streams, then every map and a final statistics call checked."""
    torch = _torch()
    views = [wl.C1.with_(W=257, H=37, iter_max=700), wl.C1.with_(W=300, H=777, iter_max=400),
             wl.C1.with_(W=96, H=1500, iter_max=300), wl.C1.with_(W=257, H=37, iter_max=700)]
    want = [oracle.render(v) for v in views]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    outs, plan = [], []
    for rep in range(3):
        for k, v in enumerate(views):
            scheme, n = [("fcfs", 1), ("block", 1), ("fcfs", 3), ("cyclic", 2)][(k + rep) % 4]
            o = torch.zeros((v.H, v.W), dtype=torch.int32, device="cuda:0")
            torch.cuda.synchronize()
            st = [s1, s2][(k + rep) % 2].cuda_stream
            mandel.mandel_render_ex(*v.args(), "fp64", scheme, n, out_dev0=o, stream0=st, logical_ranks=n > 1,
                                    want_stats=False, kernel=["refill", "lazy2"][rep % 2])
            outs.append(o)
            plan.append(k)
    torch.cuda.synchronize()
    for o, k in zip(outs, plan):
        _assert_same(_host(o), want[k], f"view {k}")
    for v, w in zip(views, want):
        for scheme, n in (("fcfs", 1), ("fcfs", 3)):
            out, st = _render_dev(mandel, v, scheme, n)
            _assert_same(_host(out), w, f"stats {scheme}/{n}")
            assert st["chunks_claimed"] == -(-v.H // 16) and st["pixels"] == v.pixels


@pytest.mark.parametrize("dtype", ["fp64", "fp32", "fp64fma"])
def test_small_view_tuning(mandel, oracle, dtype):
    """Views up to 2^21 pixels pick their kernel by timing the candidates on the view
    itself, once (tune_small): whatever wins, the map is the oracle's, the choice is cached
    per view (the second render reports the same kernel), and it applies to every scheme
    and rank count."""
    mandel.mandel_shutdown()  # clears the per-view cache
    cfg = wl.C1.with_(W=700, H=500, iter_max=400, dtype=dtype)
    want = oracle.render(cfg)
    out, st = _render_dev(mandel, cfg, "block", 1)
    _assert_same(_host(out), want, f"tuned {dtype}")
    assert st["kernel"] in ("eager", "lazy")
    assert st["probe"][1] == 0.0 and st["probe"][0] > 0  # timed, not the ipe statistic
    first = (st["kernel"], st["kernel_ilp"])
    for scheme, n in (("block", 1), ("cyclic", 3), ("fcfs", 2), ("fcfs", 1)):
        out, st = _render_dev(mandel, cfg, scheme, n)
        _assert_same(_host(out), want, f"tuned {dtype} {scheme}/N={n}")
        assert (st["kernel"], st["kernel_ilp"]) == first
    # an SM-sliced render tunes on the whole GPU and still renders the view exactly
    mandel.mandel_shutdown()
    out, st = _render_dev(mandel, cfg, "block", 1, max_sms=3)
    _assert_same(_host(out), want, f"tuned {dtype} max_sms")


# ---------------------------------------------------------------------------
# fused-y form (R21): y' = fma(RN(x y), 2, ci) where it equals the oracle's
# RN(RN((x + x) y) + ci); unsafe pixels (cr = 0, tiny |c| components) and views with a
# huge R keep the three-operation form -- maps identical to the oracle either way
# ---------------------------------------------------------------------------
FUSED_VIEWS = {
    "c1": wl.C1.with_(W=400, H=300, iter_max=300),
    # a column at cr = 0 exactly (and a row at ci = 0)
    "zero_column": wl.Config("zc", -1.0, 1.0, -1.0, 1.0, 64, 64, 500, 2.0, "fp64"),
    # every |c| component below 2^-400 (fp64) / 2^-32 (fp32): all pixels take the exact form
    "tiny": wl.Config("tiny", -1e-125, 1e-125, -1e-125, 1e-125, 48, 40, 200, 2.0, "fp64"),
    "tiny32": wl.Config("tiny32", -1e-11, 1e-11, -1e-11, 1e-11, 48, 40, 200, 2.0, "fp64"),
    # a mix: columns either side of the 2^-400 bound in one tile
    "mixed": wl.Config("mix", -4e-120, 4e-120, -0.5, 0.5, 96, 64, 300, 2.0, "fp64"),
    # near the c = -2 tip and the real axis (|z| = 2 orbits, exact R^2 hits)
    "tip": wl.Config("tip", -2.0, -1.9, -0.05, 0.05, 128, 96, 1000, 2.0, "fp64"),
    # fp32's bound (2^-32) inside one tile
    "mixed32": wl.Config("mix32", -1e-9, 1e-9, -0.5, 0.5, 96, 64, 300, 2.0, "fp64"),
}
FP64_ONLY = ("tiny", "mixed")  # windows below fp32's range (they collapse to 0 in fp32)


@pytest.mark.parametrize("view", sorted(FUSED_VIEWS))
@pytest.mark.parametrize("kernel", ["refill", "lazy1", "lazy2", "batch8x1", "batch8x2", "refill1", "batch4x2"])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_fused_y_parity(mandel, oracle, view, kernel, dtype):
    if dtype == "fp32" and view in FP64_ONLY:
        return  # not representable in fp32 (covered by tiny32 / mixed32)
    cfg = FUSED_VIEWS[view].with_(dtype=dtype)
    want = oracle.render(cfg)
    for fy in (0, -1):
        out, st = _render_dev(mandel, cfg, "block", 1, kernel=kernel, fused_y=fy)
        _assert_same(_host(out), want, f"fused_y={fy}/{view}/{kernel}/{dtype}")
        assert st["fused_y"] == (1 if fy == 0 else 0)


@pytest.mark.parametrize("dtype,R,on", [("fp64", 2.0 ** 128, 1), ("fp64", 2.0 ** 128 * 1.5, 0),
                                        ("fp32", 2.0 ** 32, 1), ("fp32", 2.0 ** 32 * 1.5, 0)])
def test_fused_y_needs_bounded_r(mandel, oracle, dtype, R, on):
    # R^2 <= 2^256 (fp64) / 2^64 (fp32) keeps 2 RN(x y) finite before the escape
    cfg = wl.C1.with_(W=120, H=90, iter_max=60, R=R, dtype=dtype)
    out, st = _render_dev(mandel, cfg, "cyclic", 2, kernel="lazy2")
    _assert_same(_host(out), oracle.render(cfg), f"R={R}/{dtype}")
    assert st["fused_y"] == on
    with pytest.raises(mandel.MandelError):
        _render_dev(mandel, cfg, "block", 1, fused_y=2)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_fused_y_whole_map_matches_exact_form(mandel, name):
    # the whole bench map with and without the fused-y form, element by element
    cfg = wl.CONFIGS[name]
    a, sa = _render_dev(mandel, cfg, "block", 1, fused_y=0)
    b, sb = _render_dev(mandel, cfg, "block", 1, fused_y=-1)
    assert sa["fused_y"] == 1 and sb["fused_y"] == 0
    assert bool((a == b).all()), f"{name}: fused-y map differs from the three-operation form"
    assert sa["sum_iters"] == sb["sum_iters"]


# ---------------------------------------------------------------------------
# per-device host hand-off (options.host_handoff = 1): every rank's band copied to the
# host by its own device -- forced here, where all logical ranks share cuda:0
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("scheme", ["block", "cyclic", "fcfs", "fcfs_master"])
@pytest.mark.parametrize("ngpus", [2, 3, 5, 8])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_host_handoff_per_device(mandel, oracle, dtype, scheme, ngpus):
    cfg = wl.C1.with_(dtype=dtype, W=517, H=389)  # ragged: H not a multiple of the chunk or N
    want = oracle.render(cfg)
    got = np.full((cfg.H, cfg.W), 0xDEADBEEF, np.uint32)
    kw = dict(chunk_rows=[0, 5, 16, 1][ngpus % 4]) if scheme == "fcfs" else {}
    st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, ngpus, out_host=got, logical_ranks=True,
                                 host_handoff=1, **kw)
    _assert_same(got, want, f"per-device hand-off {dtype}/{scheme}/N={ngpus}")
    assert st["host_handoff"] == "per_device"
    assert st["sum_iters"] == int(want.sum(dtype=np.uint64)) and st["pixels"] == cfg.pixels
    assert st["transfers"] >= 1 and st["d2h_ms"] >= 0
    if scheme in ("block", "cyclic"):
        # static plans: one (strided) copy per rank plus the cyclic tail on rank 0
        plans = [mandel.mandel_plan_rows(scheme, cfg.H, ngpus, r) for r in range(ngpus)]
        assert ngpus <= st["transfers"] <= ngpus + 1, (st["transfers"], [len(p) for p in plans])
    # the default with one device is the gather through GPU 0; a repeated call reuses the bands
    got2 = np.zeros_like(got)
    st2 = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, ngpus, out_host=got2, logical_ranks=True,
                                  **kw)
    _assert_same(got2, want, "through GPU 0")
    assert st2["host_handoff"] == "gpu0"
    got3 = np.zeros_like(got)
    mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, ngpus, out_host=got3, logical_ranks=True,
                            host_handoff=1, **kw)
    _assert_same(got3, want, "per-device hand-off, second call")


def test_host_handoff_rejects_bad_value(mandel):
    cfg = wl.C1.with_(W=32, H=32)
    o = np.zeros((cfg.H, cfg.W), np.uint32)
    for v in (-2, 2):
        with pytest.raises(mandel.MandelError):
            mandel.mandel_render_ex(*cfg.args(), "fp64", "block", 2, out_host=o, logical_ranks=True,
                                    host_handoff=v)


def test_host_handoff_large_pinned(mandel, oracle):
    """C2-shaped map through the per-device hand-off into pinned memory: sampled rows
    against the oracle, Σcounts against the map."""
    torch = _torch()
    cfg = wl.C2
    host = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, pin_memory=True)
    st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 4, out_host=host, logical_ranks=True,
                                 host_handoff=1)
    m = host.numpy().view(np.uint32)
    assert st["host_handoff"] == "per_device"
    assert int(m.sum(dtype=np.uint64)) == st["sum_iters"] and m.min() >= 1
    rows = np.sort(np.random.default_rng(7).choice(cfg.H, 24, replace=False))
    want, _ = oracle.render_rows_mt(cfg, rows)
    _assert_same(m[rows], want, "C2 per-device hand-off rows")


# ---------------------------------------------------------------------------
# first block (options.first_block): a refill of many fresh pixels
# starts with one exactly recorded block instead of a batch + replay -- counts unchanged
# ---------------------------------------------------------------------------
FIRST_BLOCK_VIEWS = {
    "full": wl.C1.with_(W=328, H=203),                                   # exterior, boundary, interior
    "far": wl.Config("far", 2.0, 9.0, -3.0, 3.0, 260, 130, 50, 2.0, "fp64"),  # every count 1 or 2
    "seahorse": wl.Config("sea", -0.76, -0.73, 0.09, 0.12, 192, 160, 600, 2.0, "fp64"),
}


@pytest.mark.parametrize("view", sorted(FIRST_BLOCK_VIEWS))
@pytest.mark.parametrize("kernel", ["refill", "batch8x1", "batch8x2", "batch8x3", "batch8x4", "batch4x2", "batch16x2"])
@pytest.mark.parametrize("dtype", ["fp64", "fp32", "fp64fma"])
def test_first_block_parity(mandel, oracle, view, kernel, dtype):
    if dtype == "fp32" and kernel.startswith("batch16"):
        return  # fp32 allows check_every <= 8 (R18)
    cfg = FIRST_BLOCK_VIEWS[view].with_(dtype=dtype)
    want = oracle.render(cfg)
    for fb in (0, -1, 1, 32):
        out, st = _render_dev(mandel, cfg, "cyclic" if fb == 1 else "block", 1, kernel=kernel, first_block=fb)
        _assert_same(_host(out), want, f"first_block={fb}/{view}/{kernel}/{dtype}")
        if st["kernel"] == "eager" and st["kernel_batch"] > 1:
            assert st["first_block"] == {0: 2, -1: 0, 1: 1, 32: 32}[fb]
        else:
            assert st["first_block"] == 0
        assert st["sum_iters"] == int(want.sum(dtype=np.uint64))


@pytest.mark.parametrize("iter_max", [1, 2, 7, 8, 9, 15, 16, 17, 25])
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_first_block_short_budgets(mandel, oracle, iter_max, dtype):
    # budgets around the block length: below 8 the block is skipped, at 8 it is the whole
    # budget (a slot that did not escape retires with iterMax), above it the batched loop follows
    cfg = wl.C1.with_(W=200, H=120, iter_max=iter_max, dtype=dtype)
    want = oracle.render(cfg)
    for kernel in ("batch8x2", "batch8x1", "batch4x4"):
        for fb in (1, 16):
            out, st = _render_dev(mandel, cfg, "fcfs", 1, kernel=kernel, first_block=fb, chunk_rows=4)
            _assert_same(_host(out), want, f"iterMax={iter_max}/{kernel}/first_block={fb}/{dtype}")


def test_first_block_large_radius_and_bad_value(mandel, oracle):
    # R = 2^100: slots past their escape inside the block overflow to inf/NaN; only the
    # first escaping update is recorded
    for dtype, R in (("fp64", 2.0 ** 100), ("fp32", 2.0 ** 20), ("fp64", 2.0 ** 200)):
        cfg = wl.C1.with_(W=160, H=96, iter_max=40, R=R, dtype=dtype)
        out, st = _render_dev(mandel, cfg, "block", 1, kernel="batch8x2", first_block=1)
        _assert_same(_host(out), oracle.render(cfg), f"R={R}/{dtype}")
    for bad in (-2, 33):
        with pytest.raises(mandel.MandelError):
            _render_dev(mandel, wl.C1.with_(W=64, H=64), "block", 1, first_block=bad)


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_first_block_whole_map_matches_batched_form(mandel, name):
    # the whole bench map with and without the first block, element by element
    cfg = wl.CONFIGS[name]
    a, sa = _render_dev(mandel, cfg, "block", 1, first_block=0)
    b, sb = _render_dev(mandel, cfg, "block", 1, first_block=-1)
    assert sa["first_block"] == 2 and sb["first_block"] == 0
    assert bool((a == b).all()), f"{name}: the map with the first block differs from the batched form"
    assert sa["sum_iters"] == sb["sum_iters"]
