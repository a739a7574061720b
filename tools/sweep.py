#!/usr/bin/env python3
"""Kernel-variant sweep on one GPU (development tool, not the bench).

    python tools/sweep.py --configs C2,C4 --kernels refill1,refill2,static \
        --schemes block,fcfs --tiles 256,512 --steps 10

Every variant's map is compared with the first variant's map on the device
(all variants must be bit-identical; parity with the oracle is the tests' job).
Prints one JSON line per variant.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2")
    ap.add_argument("--dtype", default=None, help="override the configs' dtype (fp64, fp32, fp64fma)")
    ap.add_argument("--kernels", default="refill1,refill2")
    ap.add_argument("--schemes", default="block,fcfs")
    ap.add_argument("--tiles", default="256")
    ap.add_argument("--tile-rows", default="0", help="rows per tile, comma separated (0 = default)")
    ap.add_argument("--pack", default="1", help="fp32 packed batched loop: 1, 0 or 1,0")
    ap.add_argument("--stage", default="0", help="store staging: 1 staged, -1 direct, 0 default (comma list)")
    ap.add_argument("--fused-y", default="0", help="options.fused_y (0 on, -1 off)")
    ap.add_argument("--first-block", default="0", help="options.first_block (0 default, -1 off, 1..32 lanes)")
    ap.add_argument("--ctas", default="0", help="resident CTAs per SM cap (0 = occupancy max), comma list")
    ap.add_argument("--chunks", default="16")
    ap.add_argument("--lanes", default="0", help="LAZY refill_lanes (0 = the library default, 16)")
    ap.add_argument("--minb", default="1")
    ap.add_argument("--adapt", default="16:64", help="lo:hi pairs, comma separated")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    for name in a.configs.split(","):
        cfg = wl.CONFIGS[name]
        if a.dtype:
            cfg = cfg.with_(dtype=a.dtype)
        ref = None
        out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
        for kern, scheme, tile, trows, chunk, lanes, minb, adapt, pack, stage, ctas in itertools.product(
                a.kernels.split(","), a.schemes.split(","), a.tiles.split(","), a.tile_rows.split(","),
                a.chunks.split(","), a.lanes.split(","), a.minb.split(","), a.adapt.split(","),
                a.pack.split(","), a.stage.split(","), a.ctas.split(",")):
            if not kern.startswith("adapt") and adapt != a.adapt.split(",")[0]:
                continue
            alo, ahi = (int(v) for v in adapt.split(":"))
            if kern == "static" and scheme == "fcfs":
                continue
            if not kern.startswith(("lazy", "adapt")) and lanes != a.lanes.split(",")[0]:
                continue
            if kern == "static" and minb != a.minb.split(",")[0]:
                continue
            kw = dict(out_dev0=out, stream0=stream.cuda_stream, kernel=kern,
                      tile_px=int(tile), tile_rows=int(trows), chunk_rows=int(chunk), refill_lanes=int(lanes),
                      no_pack=pack == "0", stage=int(stage), ctas_per_sm=int(ctas), fused_y=int(a.fused_y), first_block=int(a.first_block),
                      min_ctas=int(minb) if kern != "static" else 0, adapt_lo=alo, adapt_hi=ahi)
            out.zero_()
            for _ in range(a.warmup):
                mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, 1, **kw)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ks = []
            for _ in range(a.steps):
                st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, 1, **kw)
                ks.append(st["kernel_ms_max"])
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            if ref is None:
                ref = out.clone()
                same = True
            else:
                same = bool((ref == out).all())
            giter = st["sum_iters"] / (ms * 1e-3) / 1e9
            # pixel-iterations/s at the FP pipe peak: 8 ops/iteration (6 for the FMA dtype)
            ops = 6 if cfg.dtype == "fp64fma" else 8
            peak = 148 * (128 if cfg.dtype == "fp32" else 64) * 1.965e9 / ops / 1e9
            print(json.dumps({"config": name, "dtype": cfg.dtype, "kernel": kern, "scheme": scheme, "tile": int(tile), "tile_rows": int(trows),
                              "packed": st["kernel_packed"], "batch": st["kernel_batch"], "stage": int(stage), "ctas": int(ctas), "store": st["store_mode"], "fused_y": st["fused_y"],
                              "chunk": int(chunk), "lanes": int(lanes), "minb": int(minb), "adapt": adapt, "ms": round(ms, 4),
                              "kernel_ms": round(sum(ks) / len(ks), 4),
                              "giter_s": round(giter, 2), "frac": round(giter / peak, 4),
                              "ran": f"{st['kernel']}{st['kernel_ilp']}", "probe": st["probe"],
                              "iters_per_exit": round(st["warp_iters"] / max(st["loop_exits"], 1), 2),
                              "pix_per_exit": round(st["pixels"] / max(st["loop_exits"], 1), 2),
                              "identical": same}), flush=True)
        del out, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
