#!/usr/bin/env python3
"""Small-view (C1-class) latency study on one GPU (development tool, not the bench).

For each variant: mean device time per render over back-to-back enqueue-only renders
(CUDA events on the launching stream; the renders are queued behind a sleep kernel so
the host's per-call cost is hidden), and the same with iterMax cut to 1 (the
fixed cost: launch, ramp, pixel mapping, stores).

    python tools/small_view.py --kernels lazy,refill --tiles 32,64 --ctas 0,2
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402


def host_us(cfg, kw, steps):
    """Host cost of one enqueue-only call (wall clock while the GPU sleeps)."""
    import time
    torch.cuda.synchronize()
    torch.cuda._sleep(int(steps * 100e3 * 2))
    t0 = time.perf_counter()
    for _ in range(steps):
        mandel.mandel_render_ex(*cfg.args(), cfg.dtype, SCHEME, 1, want_stats=False, **kw)
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    return dt / steps * 1e6


def timed(cfg, kw, steps, stream):
    for _ in range(5):
        mandel.mandel_render_ex(*cfg.args(), cfg.dtype, SCHEME, 1, want_stats=False, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the GPU sleeps while the host enqueues every render, so they run back to back with
    # no host gap: the per-render time is the device's own
    torch.cuda._sleep(int(steps * 40e3 * 2))
    e0.record(stream)
    for _ in range(steps):
        mandel.mandel_render_ex(*cfg.args(), cfg.dtype, SCHEME, 1, want_stats=False, **kw)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


SCHEME = "block"


def main():
    global SCHEME
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--view", default="", help="xmin,xmax,ymin,ymax,W,H,iterMax (overrides --config's)")
    ap.add_argument("--kernels", default="lazy,refill")
    ap.add_argument("--tiles", default="0")
    ap.add_argument("--tile-rows", default="0")
    ap.add_argument("--ctas", default="0")
    ap.add_argument("--lanes", default="0")
    ap.add_argument("--minb", default="0")
    ap.add_argument("--iters", default="", help="extra iterMax values (comma list) besides the config's and 1")
    ap.add_argument("--scheme", default="block")
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    SCHEME = a.scheme
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    base = wl.CONFIGS[a.config]
    if a.view:
        v = a.view.split(",")
        base = base.with_(xmin=float(v[0]), xmax=float(v[1]), ymin=float(v[2]), ymax=float(v[3]),
                          W=int(v[4]), H=int(v[5]), iter_max=int(v[6]))
    out = torch.zeros((base.H, base.W), dtype=torch.int32, device=dev)
    iters = [base.iter_max, 1] + [int(v) for v in a.iters.split(",") if v]
    for kern, tile, trows, ctas, lanes, minb in itertools.product(
            a.kernels.split(","), a.tiles.split(","), a.tile_rows.split(","), a.ctas.split(","),
            a.lanes.split(","), a.minb.split(",")):
        kw = dict(out_dev0=out, stream0=stream.cuda_stream, kernel=kern, tile_px=int(tile),
                  tile_rows=int(trows), ctas_per_sm=int(ctas), refill_lanes=int(lanes), min_ctas=int(minb))
        rec = {"view": [base.xmin, base.xmax, base.ymin, base.ymax, base.W, base.H, base.iter_max], "kernel": kern, "tile": int(tile), "tile_rows": int(trows), "ctas": int(ctas), "lanes": int(lanes),
               "minb": int(minb)}
        try:
            st = mandel.mandel_render_ex(*base.args(), base.dtype, SCHEME, 1, **kw)
        except Exception as ex:  # noqa: BLE001
            rec["error"] = str(ex)
            print(json.dumps(rec), flush=True)
            continue
        rec.update(ran=f"{st['kernel']}{st['kernel_ilp']}", sum_iters=st["sum_iters"])
        for im in iters:
            cfg = base.with_(iter_max=im)
            ms = timed(cfg, dict(kw), a.steps, stream)
            rec[f"ms_it{im}"] = round(ms, 5)
        rec["host_us_per_call"] = round(host_us(base, dict(kw), 50), 2)
        rec["giter_s"] = round(st["sum_iters"] / (rec[f"ms_it{base.iter_max}"] * 1e-3) / 1e9, 1)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
