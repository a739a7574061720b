#!/usr/bin/env python3
"""Register budget of the batched EAGER default across views (development tool):
kernel time of batch8x2 at min_ctas 1 (ptxas' 82 registers, 2 CTAs/SM) and 3 (74
registers, 3 CTAs/SM) on the probe-calibration views and the bench configs.

    python tools/minb_views.py --size 4096
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
    ap.add_argument("--kernel", default="batch8x2")
    ap.add_argument("--dtype", default="fp64")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev).cuda_stream
    views = [wl.CONFIGS[c] for c in ("C2", "C5")] if a.dtype == "fp64" else [wl.CONFIGS["C3"]]
    for name, (cx, cy) in CENTRES.items():
        for w in (3.0, 1.0, 0.3, 0.1, 3e-2, 1e-2, 3e-3, 1e-3, 1e-4, 1e-5, 1e-6):
            views.append(wl.Config(f"{name}-{w:g}", cx - w / 2, cx + w / 2, cy - w / 2, cy + w / 2, a.size,
                                   a.size, a.iters, 2.0, a.dtype))
    for cfg in views:
        out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
        res = {"view": cfg.name}
        for mb in (1, 3):
            ms = []
            for i in range(a.steps + 1):
                st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 1, out_dev0=out, stream0=s,
                                             kernel=a.kernel, min_ctas=mb)
                if i:
                    ms.append(st["kernel_ms_max"])
            res[f"minb{mb}"] = round(min(ms), 4)
        res["ratio_1_over_3"] = round(res["minb1"] / res["minb3"], 4)
        print(json.dumps(res), flush=True)
        del out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
