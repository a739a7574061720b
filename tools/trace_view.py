#!/usr/bin/env python3
"""Per-warp timeline of one render (development tool; needs libmandel_trace.so).

    python -c "from paper_2007_00745_b200 import build; build.build_trace()"
    MANDEL_LIB=paper_2007_00745_b200/libmandel_trace.so python tools/trace_view.py --config C1 --kernel lazy

Prints one JSON summary per variant: kernel span, warp finish-time quantiles, per-SM busy
spans, and the last warps to finish (what holds the tail).
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402


class Rec(ctypes.Structure):
    _fields_ = [("t0", ctypes.c_uint64), ("t1", ctypes.c_uint64), ("iters", ctypes.c_uint64),
                ("smid", ctypes.c_uint32), ("tiles", ctypes.c_uint32), ("pixels", ctypes.c_uint32),
                ("warp", ctypes.c_uint32)]


def main():
    assert "trace" in os.environ.get("MANDEL_LIB", ""), "run with MANDEL_LIB=.../libmandel_trace.so"
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--kernels", default="refill")
    ap.add_argument("--scheme", default="block")
    ap.add_argument("--tiles", default="0")
    ap.add_argument("--iter-max", type=int, default=0)
    a = ap.parse_args()
    L = mandel.lib()
    L.mandel_dev_trace.argtypes = [ctypes.c_void_p, ctypes.c_uint]
    L.mandel_dev_trace.restype = ctypes.c_int
    cfg = wl.CONFIGS[a.config]
    if a.iter_max:
        cfg = cfg.with_(iter_max=a.iter_max)
    dev = torch.device("cuda", 0)
    out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
    n = 1 << 16
    buf = (Rec * n)()
    for kern in a.kernels.split(","):
        for tile in a.tiles.split(","):
            kw = dict(out_dev0=out, kernel=kern, tile_px=int(tile))
            for _ in range(3):
                st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, a.scheme, 1, **kw)
            L.mandel_dev_trace(ctypes.addressof(buf), n)  # clears
            st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, a.scheme, 1, **kw)
            assert L.mandel_dev_trace(ctypes.addressof(buf), n) == 0
            r = np.frombuffer(buf, dtype=np.dtype([("t0", "u8"), ("t1", "u8"), ("iters", "u8"), ("smid", "u4"),
                                                   ("tiles", "u4"), ("pixels", "u4"), ("warp", "u4")]))
            r = r[r["t1"] > 0]
            t0 = int(r["t0"].min())
            start = (r["t0"] - t0) / 1e3
            end = (r["t1"] - t0) / 1e3
            dur = end - start
            span = float(end.max())
            sm_end = np.zeros(int(r["smid"].max()) + 1)
            sm_start = np.full_like(sm_end, 1e9)
            np.maximum.at(sm_end, r["smid"], end)
            np.minimum.at(sm_start, r["smid"], start)
            last = np.argsort(-end)[:12]
            res = {
                "config": cfg.name, "iter_max": cfg.iter_max, "kernel": kern, "tile": int(tile),
                "ran": f"{st['kernel']}{st['kernel_ilp']}",
                "kernel_ms_event": round(st["kernel_ms_max"] * 1e3, 2),
                "span_us": round(span, 2), "warps": int(len(r)),
                "start_us_max": round(float(start.max()), 2),
                "finish_us_q": {q: round(float(np.quantile(end, q)), 2) for q in (0.1, 0.5, 0.9, 0.99, 1.0)},
                "sm_end_us": {"min": round(float(sm_end.min()), 2), "mean": round(float(sm_end.mean()), 2),
                              "max": round(float(sm_end.max()), 2)},
                "sm_start_us_max": round(float(sm_start.max()), 2),
                "tiles_per_warp": {"mean": round(float(r["tiles"].mean()), 2), "max": int(r["tiles"].max())},
                "iters_per_warp": {"mean": round(float(r["iters"].mean()), 1), "max": int(r["iters"].max())},
                "last_warps": [{"sm": int(r["smid"][i]), "start": round(float(start[i]), 2), "end": round(float(end[i]), 2),
                                "tiles": int(r["tiles"][i]), "pixels": int(r["pixels"][i]), "iters": int(r["iters"][i])}
                               for i in last],
            }
            # iterations finished by warps ending in each 10% slice of the span
            edges = np.linspace(0, span, 11)
            res["iters_by_end_decile"] = [int(r["iters"][(end >= edges[k]) & (end < edges[k + 1] + 1e-9)].sum())
                                         for k in range(10)]
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
