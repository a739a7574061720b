"""Output stage (NEXT-3): colour map and binary PPM.
CPU tests pin the oracle colour map and the library's PPM writer; GPU tests compare
the device colour kernel with the oracle byte for byte."""
import os

import numpy as np
import pytest

import workloads as wl
from oracle import colour as C


def test_colour_pins():
    # interior black in every mode; the ramp starts at 0 for n = 1
    m = 2000
    n = np.array([m, 1, m - 1, 1000], dtype=np.uint32)
    g = C.colour(n, m, C.GRAY)
    assert g[0].tolist() == [0, 0, 0] and g[1].tolist() == [0, 0, 0]
    assert g[2].tolist() == [255, 255, 255]          # 255 * 1998/1999 = 254.87 -> 255
    assert g[3].tolist() == [127, 127, 127]          # 255 * 999/1999 = 127.44 -> 127
    assert C.colour(np.array([m]), m, C.CLASSIC)[0].tolist() == [0, 0, 0]
    assert C.colour(np.array([5]), m, C.CLASSIC)[0].tolist() == [35, 65, 145]
    assert C.colour(np.array([1, 1]), 1, C.GRAY).tolist() == [[0, 0, 0], [0, 0, 0]]


def test_ppm_layout_and_writer(mandel, tmp_path):
    # 1x1 interior -> "P6\n1 1\n255\n" + 00 00 00
    assert C.ppm_bytes(np.zeros((1, 1, 3), np.uint8)) == b"P6\n1 1\n255\n\x00\x00\x00"
    rgb = C.colour(np.arange(1, 7 * 5 + 1, dtype=np.uint32).reshape(5, 7), 40, C.CLASSIC)
    p = tmp_path / "x.ppm"
    n = mandel.mandel_write_ppm(str(p), np.ascontiguousarray(rgb), 7, 5)
    data = p.read_bytes()
    assert data == C.ppm_bytes(rgb) and n == len(data) == len(b"P6\n7 5\n255\n") + 3 * 35
    with pytest.raises(mandel.MandelError) as e:
        mandel.mandel_write_ppm(str(tmp_path / "no" / "such" / "dir.ppm"), rgb, 7, 5)
    assert e.value.code == mandel.MANDEL_EIO


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["gray", "classic"])
@pytest.mark.parametrize("shape", [(800, 800), (333, 217), (1, 1), (5, 3)])
def test_device_colour_matches_oracle(mandel, oracle, mode, shape):
    import torch
    W, H = shape
    cfg = wl.C1.with_(W=W, H=H, iter_max=300)
    counts = torch.zeros((H, W), dtype=torch.int32, device="cuda:0")
    mandel.mandel_render_ex(*cfg.args(), "fp64", "block", 1, out_dev0=counts,
                            stream0=torch.cuda.current_stream().cuda_stream)
    rgb = torch.zeros((H, W, 3), dtype=torch.uint8, device="cuda:0")
    mandel.mandel_colorize(counts, rgb, W, H, cfg.iter_max, mode,
                           torch.cuda.current_stream().cuda_stream)
    want = C.colour(oracle.render(cfg), cfg.iter_max, C.GRAY if mode == "gray" else C.CLASSIC)
    assert np.array_equal(rgb.cpu().numpy(), want)
    # unaligned destination (scalar kernel path)
    big = torch.zeros(H * W * 3 + 1, dtype=torch.uint8, device="cuda:0")
    mandel.mandel_colorize(counts, big.data_ptr() + 1, W, H, cfg.iter_max, mode, None)
    assert np.array_equal(big[1:].cpu().numpy().reshape(H, W, 3), want)


def _gray_probe_counts(M: int) -> np.ndarray:
    """Every count for small iterMax; for large ones the ends and, for each grey level k,
    the counts around the half-up rounding point t = (2k+1)(M-1)/510 (t = n-1)."""
    if M <= 4096:
        return np.arange(1, M + 1, dtype=np.uint64)
    K = M - 1
    ns = {1, 2, 3, M - 2, M - 1, M}
    for k in range(256):
        t0 = ((2 * k + 1) * K) // 510
        for d in (-2, -1, 0, 1, 2):
            t = t0 + d
            if 0 <= t <= K:
                ns.add(t + 1)
    return np.array(sorted(ns), dtype=np.uint64)


@pytest.mark.gpu
@pytest.mark.parametrize("M", [2, 3, 255, 256, 257, 511, 1000, 4096, 65537, 10_000_019, 2**24 + 1,
                               2**31 + 11, 2**32 - 2])
def test_device_gray_rounding_points(mandel, M):
    """The gray ramp's float estimate + exact correction against the integer formula
    (oracle/colour.py) at every rounding point, iterMax up to 2^32 - 2."""
    import torch
    n = _gray_probe_counts(M)
    pad = (-len(n)) % 4 + 4  # an aligned multiple of 4 plus a few more pixels
    n = np.concatenate([n, np.full(pad, M, dtype=np.uint64)]).astype(np.uint32)
    want = C.colour(n, M, C.GRAY)
    dev = torch.from_numpy(n.view(np.int32)).to("cuda:0")
    for W, H, off in ((len(n), 1, 0), (len(n) - 3, 1, 1)):  # vector and scalar kernel paths
        rgb = torch.zeros(W * 3 + 1, dtype=torch.uint8, device="cuda:0")
        mandel.mandel_colorize(dev, rgb.data_ptr() + off, W, H, M, "gray", None)
        torch.cuda.synchronize()
        got = rgb[off:off + W * 3].cpu().numpy().reshape(W, 3)
        assert np.array_equal(got, want[:W]), M
