#!/usr/bin/env python3
"""Region breakdown of an ncu source page (SASS): consecutive instructions executed the
same number of times form one basic-block-like region; prints each region's share of
executed instructions and of warp-stall samples, its execution count and its first
instructions -- so the hot loop, the hit replay, the refill and the retire path can be
told apart and weighed (where C3's loss outside the loop goes).

    python tools/ncu_regions.py report.ncu-rep [--min 0.3] [--json out.json]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_source import rows  # noqa: E402


def regions(rs):
    out, cur = [], None
    for r in rs:
        ins = float(r["Instructions Executed"] or 0)
        smp = float(r["Warp Stall Sampling (All Samples)"] or 0)
        src = r["Source"].strip()
        if cur is None or ins != cur["exec"]:
            cur = {"exec": ins, "n": 0, "inst": 0.0, "samples": 0.0, "first": r["Address"], "code": []}
            out.append(cur)
        cur["n"] += 1
        cur["inst"] += ins
        cur["samples"] += smp
        if len(cur["code"]) < 6:
            cur["code"].append(src)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--min", type=float, default=0.3, help="only regions with at least this %% of instructions")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    rs = rows(a.rep)
    regs = regions(rs)
    itot = sum(g["inst"] for g in regs) or 1.0
    stot = sum(g["samples"] for g in regs) or 1.0
    top = max(regs, key=lambda g: g["exec"])
    res = []
    for g in regs:
        pi, ps = 100 * g["inst"] / itot, 100 * g["samples"] / stot
        if pi < a.min and ps < a.min:
            continue
        res.append({"first": g["first"], "instructions": g["n"], "exec_per_instruction": g["exec"],
                    "exec_vs_hot_loop": round(g["exec"] / top["exec"], 4), "pct_instructions": round(pi, 2),
                    "pct_stall_samples": round(ps, 2), "code": g["code"]})
        print(f'{g["first"]:>16} {g["n"]:4d} instr x {g["exec"]:12.0f} ({g["exec"] / top["exec"]:6.3f} of loop)'
              f'  {pi:6.2f}% inst  {ps:6.2f}% samples   {" | ".join(g["code"][:3])[:90]}')
    if a.json:
        json.dump({"report": os.path.basename(a.rep), "regions": res,
                   "hot_loop_share_instructions": round(100 * top["inst"] / itot, 2)}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
