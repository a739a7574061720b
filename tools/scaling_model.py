#!/usr/bin/env python3
"""Load-balance model of the paper's three schemes on N GPUs, from real per-row work.

One GPU renders the configuration (through the C ABI); the per-row work
(pixel-iterations) then gives, for N equally fast GPUs and no communication cost:
  block / cyclic  : speed-up bound sum(w) / max_r(w_r) from mandel_plan_rows (Eq. 14-17,
                    PAPER.md:217-218) -- exact for the static plans;
  fcfs (chunk c)  : greedy list scheduling of c-row chunks in row order, each GPU taking
                    the next chunk when it finishes -> makespan;
  fcfs_master     : the paper's protocol: N-1 workers, single rows, master computes none.
Efficiency = speed-up / N.  With --paper it also forms "Table II on B200 (model)":
Amdahl (Eq. 13) from r_p = kernel time / end-to-end time (Eq. 12) measured on this GPU,
and Eq. 22 percentage differences of each scheme's modelled speed-up.
This is a model (the box has one GPU); multi-GPU runs replace it when available.
"""
import argparse
import heapq
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import analysis as A  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402


def list_schedule(chunk_work, workers):
    heap = [0.0] * workers
    for w in chunk_work:
        t = heapq.heappop(heap)
        heapq.heappush(heap, t + w)
    return max(heap)


def model(row_work, N, chunk=16):
    H = len(row_work)
    total = float(row_work.sum())
    out = {}
    for scheme in ("block", "cyclic"):
        if H < N:
            continue
        loads = [float(row_work[mandel.mandel_plan_rows(scheme, H, N, r).astype(np.int64)].sum())
                 for r in range(N)]
        s = A.load_balance_bound(loads)
        out[scheme] = {"speedup": s, "efficiency": A.efficiency(s, N)}
    chunks = [float(row_work[i:i + chunk].sum()) for i in range(0, H, chunk)]
    s = total / list_schedule(chunks, N)
    out[f"fcfs{chunk}"] = {"speedup": s, "efficiency": A.efficiency(s, N)}
    if N >= 2:
        s = total / list_schedule([float(v) for v in row_work], N - 1)
        out["fcfs_master"] = {"speedup": s, "efficiency": A.efficiency(s, N)}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C4,C5")
    ap.add_argument("--ns", default="2,4,8,16,32")
    ap.add_argument("--paper", action="store_true", help="also the R=20 paper grid + Eq. 12/13/22")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev).cuda_stream
    res = {}
    names = a.configs.split(",") + (["PAPER"] if a.paper else [])
    for name in names:
        cfg = wl.PAPER_GRID if name == "PAPER" else wl.CONFIGS[name]
        out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
        st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "block", 1, out_dev0=out, stream0=stream)
        row_work = out.to(torch.int64).sum(dim=1).cpu().numpy()
        assert int(row_work.sum()) == st["sum_iters"]
        entry = {"sum_iters": st["sum_iters"], "by_n": {}}
        for N in (int(v) for v in a.ns.split(",")):
            entry["by_n"][N] = model(row_work, N)
        if name == "PAPER":
            host = torch.empty((cfg.H, cfg.W), dtype=torch.int32, pin_memory=True)
            st_e = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "block", 1, out_host=host,
                                           stream0=stream)
            t_p, t_s = st_e["kernel_ms_max"], st_e["kernel_ms_max"] + st_e["d2h_ms"]
            r_p = A.parallel_fraction(t_p, t_s)
            entry["r_p"] = {"t_p_ms": t_p, "t_s_ms": t_s, "r_p": r_p}
            table = {}
            for N, m in entry["by_n"].items():
                T = A.amdahl_speedup(r_p, N)
                table[N] = {"theoretical": T}
                for sch, v in m.items():
                    table[N][sch] = {"speedup": v["speedup"],
                                     "pct_diff": A.percentage_difference(T, v["speedup"])}
            entry["table2_model"] = table
        res[name] = entry
        del out
        torch.cuda.empty_cache()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
