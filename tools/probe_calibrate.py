#!/usr/bin/env python3
"""Calibrate MANDEL_KERNEL_REFILL's per-view choice (EAGER batched vs LAZY) on a family
of views between the full set and deep zooms (development tool).

For each view: the probe's eager iterations per loop exit (stats['probe'][1]), and the
kernel time of the EAGER default and of LAZY; prints one JSON line per view.

    python tools/probe_calibrate.py --size 4096
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402

CENTRES = {"seahorse": (-0.743643887, 0.131825904), "elephant": (0.2925, 0.0145),
           "spiral": (-0.761574, -0.0847596), "tip": (-1.985540371, 0.0)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=5000)
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev).cuda_stream
    out = torch.zeros((a.size, a.size), dtype=torch.int32, device=dev)
    for name, (cx, cy) in CENTRES.items():
        for w in (3.0, 1.0, 0.3, 0.1, 3e-2, 1e-2, 3e-3, 1e-3, 1e-4, 1e-5, 1e-6):
            cfg = wl.Config(f"{name}-{w:g}", cx - w / 2, cx + w / 2, cy - w / 2, cy + w / 2, a.size, a.size,
                            a.iters, 2.0, "fp64")
            res = {"view": cfg.name}
            for kern in ("refill", "batch8x2", "lazy2"):
                ms = []
                for i in range(a.steps + 1):
                    st = mandel.mandel_render_ex(*cfg.args(), "fp64", "fcfs", 1, out_dev0=out, stream0=s,
                                                 kernel=kern)
                    if i:
                        ms.append(st["kernel_ms_max"])
                res[kern] = round(min(ms), 4)
                if kern == "refill":
                    res["probe_ipe"] = round(st["probe"][1], 2)
                    res["auto"] = st["kernel"]
            res["giter"] = st["sum_iters"] / 1e9
            res["best"] = "lazy" if res["lazy2"] < res["batch8x2"] else "eager"
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
