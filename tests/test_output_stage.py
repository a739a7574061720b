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
