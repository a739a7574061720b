#!/usr/bin/env python3
"""Registers / spills / shared memory per kernel from paper_2007_00745_b200/ptxas_resources.txt.
    python tools/ptxas_regs.py [substring ...]"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
txt = open(os.path.join(ROOT, "paper_2007_00745_b200", "ptxas_resources.txt")).read()
pats = sys.argv[1:]
cur = None
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        spill = ""
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = f"spill {m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers.*?(?:(\d+) bytes smem)?", line)
    if m and cur and (not pats or any(p in cur for p in pats)):
        print(f"{m.group(1):>4} regs  {spill:14s} {line.split(',')[-1].strip():>22s}  {cur}")
