#!/usr/bin/env python3
"""Bandwidth of the auxiliary device kernels against the measured HBM peak
(development tool): mandel_colorize (4 B read + 3 B written per pixel) and the K4
row scatter mandel_scatter_rows (4 B read + 4 B written per pixel), CUDA events on
the launching stream, best of N after a warm-up.

    python tools/aux_bench.py --sizes 8000,32768 --reps 10
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2007_00745_b200 import mandel  # noqa: E402


def timed(fn, stream, reps):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="8000,32768")
    ap.add_argument("--iter-max", type=int, default=5000)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs")
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    s = st.cuda_stream
    g = torch.Generator(device=dev).manual_seed(1)
    for n in (int(v) for v in a.sizes.split(",")):
        counts = torch.randint(1, a.iter_max + 1, (n, n), dtype=torch.int32, device=dev, generator=g)
        rgb = torch.empty(n * n * 3, dtype=torch.uint8, device=dev)
        for mode in ("gray", "classic"):
            ms = timed(lambda: mandel.mandel_colorize(counts, rgb, n, n, a.iter_max, mode, s), st, a.reps)
            gbs = 7.0 * n * n / (ms * 1e-3) / 1e9
            print(json.dumps({"kernel": "colorize", "mode": mode, "W": n, "H": n, "ms": round(ms, 4),
                              "algorithmic_GBs": round(gbs, 1), "hbm_peak_GBs": peak,
                              "frac": round(gbs / peak, 3) if peak else None}), flush=True)
        del rgb
        # K4: scatter every other row of a half-height band into the image
        nb = n // 2
        band = counts[:nb]
        img = torch.empty_like(counts)
        rows = torch.arange(0, 2 * nb, 2, dtype=torch.int32, device=dev)
        ms = timed(lambda: mandel.mandel_scatter_rows(band, rows, nb, n, img, s), st, a.reps)
        gbs = 8.0 * nb * n / (ms * 1e-3) / 1e9
        assert torch.equal(img[0::2][:nb], band)
        print(json.dumps({"kernel": "scatter_rows", "W": n, "rows": nb, "ms": round(ms, 4),
                          "algorithmic_GBs": round(gbs, 1), "hbm_peak_GBs": peak,
                          "frac": round(gbs / peak, 3) if peak else None}), flush=True)
        del counts, img
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
