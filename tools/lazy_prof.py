#!/usr/bin/env python3
"""Where the LAZY loop's slot-updates go (development tool): live, finished-but-waiting
for a refill, idle (no pixel), while tiles remain and in the final drain.

Needs the instrumented library (build.build_prof(); loaded through MANDEL_LIB):

    MANDEL_LIB=paper_2007_00745_b200/libmandel_prof.so python tools/lazy_prof.py --configs C4,C2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C4")
    ap.add_argument("--kernels", default="lazy2")
    ap.add_argument("--lanes", default="16")
    a = ap.parse_args()
    assert "prof" in os.environ.get("MANDEL_LIB", ""), "run with MANDEL_LIB=.../libmandel_prof.so"
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev).cuda_stream
    for name in a.configs.split(","):
        cfg = wl.CONFIGS[name]
        out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
        for kern in a.kernels.split(","):
            for lanes in a.lanes.split(","):
                st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 1, out_dev0=out, stream0=s,
                                             kernel=kern, refill_lanes=int(lanes))
                torch.cuda.synchronize()
                print(f"^ {name} {kern} lanes {lanes}: sum_iters {st['sum_iters']} pixels {st['pixels']} "
                      f"kernel_ms {st['kernel_ms_max']:.3f}", flush=True)


if __name__ == "__main__":
    main()
