#!/usr/bin/env python3
"""Divergence table from the tools/warp_eff.py captures (ncu CSV + the script's JSON line).

    python tools/warp_eff_table.py gpurun_out r02an > profiles/r02an_warp_efficiency.json

Per config and kernel:
- warp_exec_eff: ncu's smsp__thread_inst_executed_per_inst_executed.ratio / 32 -- the
  share of lanes active per executed warp instruction (north_star's "warp execution
  efficiency").  A lane iterating an idle slot (refill kernels: z = c = 0 after the work
  ran out) or a finished one (LAZY: past its escape inside a block) counts as active.
- useful_lane_frac: the counted iterations' share of the FP lane work actually executed:
  Σcounts x (FP instructions per z-update of the kernel's loop form) / executed FP
  thread-instructions (DADD+DMUL+DFMA, FADD+FMUL+FFMA).  Per-update forms: static 8
  (Eq. 1 unfused, |z|^2 every update), EAGER batched fused 6 + 1/8 (R18, R21), LAZY fused 7;
  the unfused EAGER batched form 7 + 1/8.  Everything else -- masked-off lanes, idle and
  finished slots, replays, updates past an escape, c mapping -- lowers it.
"""
import csv
import glob
import json
import os
import sys


def form_fp(ran, batch, fused):
    if ran.startswith("static"):
        return 8.0
    if ran.startswith("lazy"):
        return 7.0 if fused else 8.0
    if batch and batch > 1:
        return (6.0 if fused else 7.0) + 1.0 / batch
    return 7.0 if fused else 8.0


def read_csv(path):
    vals = {}
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for row in csv.DictReader(lines):
        vals[row["Metric Name"]] = (row["Metric Value"].replace(",", ""), row["Metric Unit"], row["Kernel Name"])
    return vals


def main():
    d, tag = sys.argv[1], sys.argv[2]
    rows = []
    for js in sorted(glob.glob(os.path.join(d, f"{tag}_weff_*.json"))):
        csvp = js[:-5] + ".csv"
        try:
            meta = json.loads(open(js).read().strip().splitlines()[-1])
            m = read_csv(csvp)
        except (OSError, ValueError, IndexError):
            continue
        f = lambda k: float(m[k][0]) if k in m else 0.0  # noqa: E731
        fp = sum(f(f"sm__sass_thread_inst_executed_op_{o}_pred_on.sum")
                 for o in ("dadd", "dmul", "dfma", "fadd", "fmul", "ffma"))
        per = form_fp(meta["ran"], meta.get("batch", 1), meta.get("fused_y", 0))
        dur = m.get("gpu__time_duration.sum")
        ms = float(dur[0]) * {"ms": 1.0, "msecond": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6,
                              "nsecond": 1e-6}.get(dur[1], 1.0) if dur else None
        rows.append({
            "config": meta["config"], "kernel": meta["kernel"], "ran": meta["ran"],
            "ncu_kernel": m.get("gpu__time_duration.sum", ("", "", ""))[2],
            "duration_ms_ncu": ms,
            "warp_exec_eff": round(f("smsp__thread_inst_executed_per_inst_executed.ratio") / 32.0, 4),
            "pred_on_eff": round(f("smsp__thread_inst_executed_pred_on_per_inst_executed.ratio") / 32.0, 4),
            "branch_uniform_pct": f("smsp__sass_average_branch_targets_threads_uniform.pct"),
            "fp_thread_inst": fp, "sum_iters": meta["sum_iters"], "fp_per_update_form": per,
            "useful_lane_frac": round(meta["sum_iters"] * per / fp, 4) if fp else None,
            "fp64_pipe_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "source": os.path.basename(csvp),
        })
    print(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
