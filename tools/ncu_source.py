#!/usr/bin/env python3
"""Per-region breakdown of an ncu source page (SASS): warp-stall samples and executed
instructions grouped into address ranges split at labelled branch targets.

    python tools/ncu_source.py report.ncu-rep [--top 40]
Prints each SASS line with its share of samples (and the instruction count), so the
hot loop, the replay and the refill path can be told apart by address."""
import argparse
import csv
import io
import subprocess


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rd = csv.DictReader(io.StringIO("\n".join(lines[start:])))
    return list(rd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--min", type=float, default=0.0, help="only lines with at least this %% of samples")
    a = ap.parse_args()
    rs = rows(a.rep)
    tot = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in rs)
    itot = sum(float(r["Instructions Executed"] or 0) for r in rs)
    for r in rs:
        smp = float(r["Warp Stall Sampling (All Samples)"] or 0)
        ins = float(r["Instructions Executed"] or 0)
        if 100 * smp / tot < a.min and ins == 0:
            continue
        print(f'{r["Address"]:>8} {100*smp/tot:6.2f}% {100*ins/itot:6.2f}%i  {r["Source"][:90]}')


if __name__ == "__main__":
    main()
