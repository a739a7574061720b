#!/usr/bin/env python3
"""Randomised parity campaign on a B200 (development tool; its summary is evidence).

Windows are drawn where the escape test is hardest: around points of the main
cardioid and period-2 disc boundaries, the Misiurewicz points +-i, the real-axis
tip c = -2 (where an escaped orbit grows slowest, R18) and random points,
with widths down to 1e-13 (fp64) / 1e-5 (fp32), iterMax up to 20000, R in
{2, 2.5, 20, 1e3}.  Every map from every kernel variant is compared with the C oracle
(all host threads) pixel by pixel.

    python tools/fuzz.py --seconds 300 --seed 1 > fuzz.jsonl
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402

KERNELS = {"fp64": ["refill", "batch4x2", "batch8x2", "batch16x2", "batch8x1", "lazy2", "adaptb8x2", "refill2"],
           "fp64fma": ["refill", "batch8x2", "batch16x1", "lazy2"],
           "fp32": ["refill", "batch8x1", "batch8x2", "batch4x4", "lazy2", "refill4"]}


def centre(rng):
    k = rng.integers(0, 6)
    t = rng.uniform(0, 2 * math.pi)
    if k == 0:  # main cardioid boundary
        z = complex(math.cos(t), math.sin(t))
        c = z / 2 - z * z / 4
    elif k == 1:  # period-2 disc boundary
        c = -1 + complex(math.cos(t), math.sin(t)) / 4
    elif k == 2:
        c = complex(0.0, 1.0 if rng.random() < 0.5 else -1.0)
    elif k == 3:
        c = complex(-2.0, 0.0)
    elif k == 4:
        c = complex(-0.743643887, 0.131825904)
    else:
        c = complex(rng.uniform(-2.2, 0.7), rng.uniform(-1.3, 1.3))
    return c, k


def draw(rng, dtype):
    c, kind = centre(rng)
    lo = -13 if dtype != "fp32" else -5
    w = 10 ** rng.uniform(lo, -0.5)
    h = w * rng.uniform(0.5, 1.5)
    ox, oy = rng.uniform(-0.5, 0.5) * w, rng.uniform(-0.5, 0.5) * h
    W, H = int(rng.integers(48, 257)), int(rng.integers(40, 200))
    it = int(rng.choice([500, 2000, 5000, 20000]))
    R = float(rng.choice([2.0, 2.0, 2.0, 2.5, 20.0, 1000.0]))
    xmin, ymin = c.real + ox - w / 2, c.imag + oy - h / 2
    cfg = wl.Config(f"fuzz{kind}", xmin, xmin + w, ymin, ymin + h, W, H, it, R, dtype)
    return cfg


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=120)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    rng = np.random.default_rng(a.seed)
    t0 = time.time()
    n_cfg = n_maps = n_px = n_bad = 0
    fails = []
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev).cuda_stream
    while time.time() - t0 < a.seconds:
        dtype = ["fp64", "fp64", "fp32", "fp64fma"][n_cfg % 4]
        cfg = draw(rng, dtype)
        try:
            want, _ = oracle.render_rows_mt(cfg, np.arange(cfg.H), chunk=4)
        except Exception as e:  # a window the ABI rejects (collapsed in fp32, ...)
            print(json.dumps({"skip": cfg.name, "why": str(e)[:80]}), flush=True)
            continue
        n_cfg += 1
        out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
        # the host-output path (pipelined bands, tapers) with random options
        hkw = dict(bands=int(rng.choice([0, 1, 2, 3, 5, 8, 12])), band_taper=int(rng.choice([0, 40, 70, 100])),
                   tile_rows=int(rng.choice([0, 1, 2, 4, 8, 16])), tile_px=int(rng.choice([0, 32, 64, 100, 256])),
                   chunk_rows=int(rng.choice([0, 1, 3, 16])))
        hscheme = ["block", "cyclic", "fcfs"][n_cfg % 3]
        try:
            if n_cfg % 5 == 0:  # several logical ranks, the per-device host hand-off (bands)
                nr = int(rng.choice([2, 3, 5, 8]))
                hs = hscheme if rng.random() < 0.8 else "fcfs_master"
                if hs in ("block", "cyclic") and cfg.H < nr:
                    nr = 2 if cfg.H >= 2 else 1
                got = np.zeros((cfg.H, cfg.W), np.uint32)
                hkw = dict(chunk_rows=hkw["chunk_rows"], tile_rows=hkw["tile_rows"], tile_px=hkw["tile_px"],
                           host_handoff=1, ngpus=nr, scheme=hs)
                mandel.mandel_render_ex(*cfg.args(), dtype, hs, nr, out_host=got, logical_ranks=True,
                                        host_handoff=1, chunk_rows=hkw["chunk_rows"], tile_rows=hkw["tile_rows"],
                                        tile_px=hkw["tile_px"])
            elif n_cfg % 2:  # asynchronous pipelined host output (finished right away)
                got = np.zeros((cfg.H, cfg.W), np.uint32)
                mandel.mandel_render_ex(*cfg.args(), dtype, hscheme, 1, out_host=got, async_host=True,
                                        want_stats=False, **hkw)
                mandel.mandel_finish()
            else:
                got, _ = mandel.render(*cfg.args(), dtype, hscheme, 1, **hkw)
            bad = int((got != want).sum())
            n_maps += 1
            n_px += got.size
            n_bad += bad
            if bad:
                fails.append({"cfg": cfg.__dict__, "host_output": hkw, "scheme": hscheme, "bad": bad})
                print(json.dumps(fails[-1]), flush=True)
        except mandel.MandelError as e:
            print(json.dumps({"skip": cfg.name, "host_output": hkw, "why": str(e)[:80]}), flush=True)
        for kern in KERNELS[dtype]:
            kw = {}
            if mandel.KERNELS[kern][2:] and cfg.R < 2.0:
                kw["check_every"] = 1
            if mandel.KERNELS[kern][2:] or kern == "refill":  # first-block threshold (a scheduling decision only)
                kw["first_block"] = int(rng.choice([0, 0, -1, 1, 2, 8, 31, 32]))
            if kern.startswith("lazy"):  # the LAZY exit threshold (a refill decision only)
                kw["refill_lanes"] = int(rng.choice([1, 2, 7, 16, 31, 32]))
            for scheme, n in (("fcfs", 1), ("cyclic", 3)):
                out.zero_()
                try:
                    mandel.mandel_render_ex(*cfg.args(), dtype, scheme, n, out_dev0=out, stream0=stream,
                                            logical_ranks=n > 1, kernel=kern, **kw)
                except mandel.MandelError as e:
                    print(json.dumps({"skip": cfg.name, "kernel": kern, "why": str(e)[:80]}), flush=True)
                    continue
                got = out.cpu().numpy().view(np.uint32)
                bad = int((got != want).sum())
                n_maps += 1
                n_px += got.size
                n_bad += bad
                if bad:
                    i, j = np.argwhere(got != want)[0]
                    fails.append({"cfg": cfg.__dict__, "kernel": kern, "scheme": scheme, "bad": bad,
                                  "first": [int(i), int(j), int(got[i, j]), int(want[i, j])]})
                    print(json.dumps(fails[-1]), flush=True)
    print(json.dumps({"summary": True, "seed": a.seed, "seconds": round(time.time() - t0, 1),
                      "configs": n_cfg, "maps": n_maps, "pixels_compared": n_px,
                      "mismatched_pixels": n_bad, "failing_maps": len(fails)}), flush=True)


if __name__ == "__main__":
    main()
