#!/usr/bin/env python3
"""FCFS claim-protocol stress under injected delays (SPEC.md:281, 487
"injected adversarial per-row delays").

Run with MANDEL_LIB pointing at libmandel_delay.so (build.build_delay(): random
__nanosleep before every claim, between a claim and its binding, at each warp's start
and before one store in 32): N logical ranks on this GPU claim 16-row chunks (FCFS) or
single rows (FCFS_MASTER, the paper's protocol) from one counter; every map must equal
the oracle's and every chunk be claimed exactly once.  Prints one JSON line; exit 1 on
any mismatch.

    MANDEL_LIB=paper_2007_00745_b200/libmandel_delay.so python tools/fcfs_delay_stress.py --reps 20
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ranks", default="2,3,5,8")
    a = ap.parse_args()
    import torch

    from paper_2007_00745_b200 import mandel
    assert os.path.basename(mandel.LIB_PATH) == "libmandel_delay.so", mandel.LIB_PATH
    cfgs = [wl.Config("64x64", -2.2, 0.8, -1.3, 1.3, 64, 64, 300, 2.0, "fp64"),
            wl.C1.with_(W=800, H=600, iter_max=200)]
    want = {c.name: oracle.render(c) for c in cfgs}
    ranks = [int(x) for x in a.ranks.split(",")]
    renders, bad, kernels = 0, 0, set()
    for cfg in cfgs:
        for scheme in ("fcfs", "fcfs_master"):
            # one claimant (N = 1, FCFS only) claims 16-chunk batches; the others one chunk
            for n in ([1] if scheme == "fcfs" else []) + ranks:
                for rep in range(a.reps):
                    out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device="cuda:0")
                    kernel = ["refill", "lazy2", "batch8x2", "refill1"][rep % 4]
                    chunk = [0, 1, 3, 16][(rep // 4) % 4] if scheme == "fcfs" else 0
                    st = mandel.mandel_render_ex(*cfg.args(), "fp64", scheme, n, out_dev0=out,
                                                 logical_ranks=True, kernel=kernel, chunk_rows=chunk)
                    got = out.cpu().numpy().view(np.uint32)
                    c = chunk or (16 if scheme == "fcfs" else 1)
                    ok = np.array_equal(got, want[cfg.name]) and st["pixels"] == cfg.pixels and \
                        st["chunks_claimed"] == -(-cfg.H // c) and sum(st["rank_rows"]) == cfg.H
                    if scheme == "fcfs_master":
                        ok = ok and st["rank_rows"][0] == 0
                    renders += 1
                    kernels.add(kernel)
                    if not ok:
                        bad += 1
                        print(f"MISMATCH {cfg.name} {scheme} N={n} rep={rep} kernel={kernel} chunk={chunk}: "
                              f"{int((got != want[cfg.name]).sum())} px, claims {st['chunks_claimed']}",
                              file=sys.stderr)
    print(json.dumps({"renders": renders, "mismatched_renders": bad, "reps": a.reps, "ranks": ranks,
                      "configs": [c.name for c in cfgs], "kernels": sorted(kernels),
                      "library": os.path.basename(mandel.LIB_PATH)}))
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
