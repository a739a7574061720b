#!/usr/bin/env python3
"""Divergence evidence (BASELINE north_star: "warp execution efficiency showing the
divergence mitigation"): render one config with one kernel a few times, so that ncu can
capture a late launch of the escape kernel.

    ncu --metrics ... -k regex:escape_ -s 5 -c 1 --csv --log-file X.csv \
        python tools/warp_eff.py --config C4 --kernel static --renders 6 > X.json

Prints one JSON line: config, kernel, the kernel that ran, Σcounts of a render and the
FP instructions per z-update of that kernel's loop form (tools/warp_eff_table.py turns
the ncu CSV and this line into the table in DESIGN.md §6).
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--kernel", default="refill")
    ap.add_argument("--renders", type=int, default=6)
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    st = None
    for _ in range(a.renders):
        st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "block", 1, out_dev0=out,
                                     stream0=stream.cuda_stream, kernel=a.kernel)
    torch.cuda.synchronize()
    assert int(out.to(torch.int64).sum()) == st["sum_iters"]
    print(json.dumps({"config": a.config, "kernel": a.kernel, "ran": f"{st['kernel']}{st['kernel_ilp']}",
                      "batch": st["kernel_batch"], "fused_y": st["fused_y"], "dtype": cfg.dtype,
                      "sum_iters": st["sum_iters"], "pixels": cfg.W * cfg.H}), flush=True)


if __name__ == "__main__":
    main()
