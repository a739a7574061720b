#!/usr/bin/env python3
"""Repeat renders of one configuration and compare every map with the oracle
(development tool: hunts nondeterministic failures)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C1")
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--kernels", default="lazy1")
    ap.add_argument("--schemes", default="block")
    ap.add_argument("--ngpus", default="5")
    ap.add_argument("--lanes", default="1")
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    cfg = wl.CONFIGS[a.config]
    if a.dtype:
        cfg = cfg.with_(dtype=a.dtype)
    want = oracle.render(cfg)
    out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device="cuda:0")
    for kern in a.kernels.split(","):
        for scheme in a.schemes.split(","):
            for n in (int(v) for v in a.ngpus.split(",")):
                for lanes in (int(v) for v in a.lanes.split(",")):
                    bad_runs = []
                    for rep in range(a.reps):
                        out.zero_()
                        st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, n, out_dev0=out,
                                                     logical_ranks=n > 1, kernel=kern,
                                                     refill_lanes=lanes)
                        got = out.cpu().numpy().view(np.uint32)
                        nbad = int((got != want).sum())
                        if nbad or st["pixels"] != cfg.pixels:
                            idx = np.argwhere(got != want)
                            bad_runs.append({"rep": rep, "bad": nbad, "pixels": st["pixels"],
                                             "first": idx[:3].tolist(),
                                             "zeros": int((got == 0).sum()),
                                             "rank_pixels": st["rank_pixels"]})
                    print(json.dumps({"kernel": kern, "scheme": scheme, "ngpus": n, "lanes": lanes,
                                      "reps": a.reps, "failures": len(bad_runs),
                                      "examples": bad_runs[:3]}), flush=True)


if __name__ == "__main__":
    main()
