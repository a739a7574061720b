#!/usr/bin/env python3
"""Summarise an ncu --set full report (raw page CSV) into the numbers DESIGN.md and
bench.py use: duration, FP pipe utilisation, issue, stall reasons, DRAM traffic."""
import csv
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active",
    "smsp__inst_executed_pipe_fp64.sum", "sm__inst_executed_pipe_fp64.sum",
    "smsp__inst_executed_pipe_fma.sum", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmalite_cycles_active.avg.pct_of_peak_sustained_active",
]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        res.append((d, dict(zip(hdr, units))))
    return res


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def scaled(v, unit):
    """Value in bytes (byte units) or milliseconds (time units); others unchanged."""
    x = num(v)
    if x is None:
        return None
    return x * SCALE.get(unit, 1)


def summarise(rep):
    out = []
    for d, u in load(rep):
        s = {"kernel": d.get("Kernel Name"), "id": d.get("ID")}
        for k in KEYS:
            if k in d:
                s[k] = scaled(d[k], u.get(k, ""))
        s["units"] = {"bytes": "byte", "gpu__time_duration.sum": "ms"}
        stalls = {}
        for k, v in d.items():
            if k.startswith("smsp__average_warp_latency_issue_stalled_") and k.endswith(".ratio"):
                x = num(v)
                if x and x > 0.05:
                    stalls[k[len("smsp__average_warp_latency_issue_stalled_"):-len(".ratio")]] = x
        s["stall_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda t: -t[1]))
        s["dram_bytes_per_launch"] = (s.get("dram__bytes_read.sum") or 0) + (s.get("dram__bytes_write.sum") or 0)
        out.append(s)
    return out


def write_traffic(rep, config, n_gpus, path, summary_path):
    """profiles/<tag>_traffic.json: what bench.py quotes beside its live roofline --
    DRAM bytes per launch and the executed FP pipe utilisation of the escape kernel."""
    s = [x for x in summarise(rep) if "escape" in (x["kernel"] or "")][0]
    fp64 = s.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active")
    fma = s.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active")
    d = {"config": config, "n_gpus": n_gpus, "kernel": s["kernel"],
         "dram_bytes_per_launch": s["dram_bytes_per_launch"],
         "fp64_pipe_active_pct": fp64, "fma_pipe_active_pct": fma,
         "warp_execution_efficiency": (s.get("smsp__thread_inst_executed_per_inst_executed.ratio") or 0) / 32,
         "duration_ms_ncu": s.get("gpu__time_duration.sum"), "source": summary_path}
    with open(path, "w") as f:
        json.dump(d, f, indent=1)
    return d


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--traffic":
        # --traffic REP CONFIG NGPUS OUT.json SUMMARY.json
        rep, cfg, n, outp, summ = sys.argv[2:7]
        with open(summ, "w") as f:
            json.dump(summarise(rep), f, indent=1)
        print(json.dumps(write_traffic(rep, cfg, int(n), outp, summ), indent=1))
    else:
        print(json.dumps([summarise(r) for r in sys.argv[1:]], indent=1))
