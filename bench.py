#!/usr/bin/env python3
"""Benchmark of the escape-time hot path (arXiv 2007.00745) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2] [--scheme fcfs]

Metric (BASELINE.json): pixel-iterations per second (Giter/s) = sum of the per-pixel
iteration counts of one map / device time of one step.  A step is one full
render of the configured map -- steps a1..a6 of SURVEY.md §8(a): host constants,
partition, pixel->c, escape loop, store, gather to rank 0 -- through the C ABI.
The default workload is BASELINE.json configs[1] (C2: 8000x8000, iterMax 2000,
R 2, fp64, [-2.5,1.5]x[-2,2]).  Inputs are the deterministic grid itself
(no dataset; data "synthetic").

N = 1: one process, one GPU.  N > 1 (torchrun, one process per GPU): each rank
renders its rows of the same map (strong scaling) through mandel_render_rank,
storing straight into rank 0's image mapped over CUDA IPC; FCFS ranks share
one chunk counter in rank 0's memory.

--impl reference: the CPU oracle (oracle/, plain C) timed on the host cores on
bounded row samples of the same workload (the only other place bench.py runs
oracle code is the cpu_baseline leg).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as wl  # noqa: E402

# FP pipe peaks derived from unit counts and clocks:
# 148 SMs x 64 FP64 lanes (or 128 FP32 lanes) x 1965 MHz max SM clock, one op per
# lane per cycle (no FMA in this path, so ops = flops).
SMS, FP64_LANES, FP32_LANES, SM_MAX_MHZ = 148, 64, 128, 1965.0
FLOPS_PER_ITER = 8  # 3 mul + 5 add/sub per z-update
MIN_FP_INSTR_PER_ITER = 6.125  # fused y (R21): 6 FP instructions per update + |z|^2 per 8 (R18)


def fp_peak_tflops(dtype: str, mhz: float = SM_MAX_MHZ) -> float:
    lanes = FP64_LANES if dtype == "fp64" else FP32_LANES
    return SMS * lanes * mhz * 1e6 / 1e12


def parse():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2", choices=sorted(wl.CONFIGS))
    ap.add_argument("--scheme", default=None, choices=["block", "cyclic", "fcfs"],
                    help="row partition (PAPER.md §III); default: fcfs over N > 1 GPUs, and on one GPU "
                         "the plain row order (block: one rank owns every row -- there is nothing to "
                         "partition; FCFS on one rank would only add its claim lookups, per_scheme "
                         "times all three)")
    ap.add_argument("--chunk-rows", type=int, default=16)
    ap.add_argument("--kernel", default="refill",
                    help="refill (default), static, eager, lazy, adaptive, refill1..4, lazy1/2")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="target CPU work (core-seconds) of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-schemes", action="store_true", help="skip the per-scheme lines")
    ap.add_argument("--gather", choices=["fused", "nccl"], default="fused",
                    help="N>1: fused peer stores into rank 0's map (default) or the NCCL path "
                         "(rank bands, point-to-point to rank 0, K4 row scatter)")
    ap.add_argument("--share-device", action="store_true",
                    help="TEST ONLY: every rank on cuda:0 with gloo plumbing (checks the N>1 "
                         "code path on a one-GPU box; not a measurement)")
    ap.add_argument("--profile", action="store_true",
                    help="short run for ncu: warmup + steps only, no e2e/cpu/schemes legs")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks: nvidia-smi sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None
        self.thread = None
        self.windows = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, t0, t1):
        self.windows.append((t0, t1))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return None
        inwin = [s for t, s in self.samples if any(a - 0.05 <= t <= b + 0.05 for a, b in self.windows)]
        use = inwin or [s for _, s in self.samples]
        mhz, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for s in use:
            try:
                mhz.append(float(s[1]))
                mx.append(float(s[2]))
                power.append(float(s[3]))
            except (ValueError, IndexError):
                continue
            for k, n in enumerate(names):
                if len(s) > 5 + k and s[5 + k].lower().startswith("active"):
                    reasons.add(n)
        if not mhz:
            return None
        return {"sm_mhz": statistics.median(mhz), "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(power) if power else None, "reasons": sorted(reasons),
                "samples": len(use), "in_window": bool(inwin)}


# ---------------------------------------------------------------------------
# distributed plumbing (torchrun): one process per GPU
# ---------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


def aggregate(dist, rank_ms: float, rank_iters: int, device=None):
    from paper_2007_00745_b200.multiproc import aggregate as _agg
    return _agg(dist, rank_ms, rank_iters, device)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    if args.scheme is None:
        args.scheme = "block" if dist_env()[0] == 1 else "fcfs"

    from paper_2007_00745_b200 import mandel

    cfg = wl.CONFIGS[args.config]
    world, rank, local = dist_env()
    if args.gpus != world:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    dist = None
    if args.share_device:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist_mod
        if args.share_device:
            dist_mod.init_process_group("gloo")
        else:
            dist_mod.init_process_group("nccl", device_id=dev)
        dist = dist_mod
    adev = None if args.share_device else dev  # gloo reduces host tensors
    mandel.lib()
    if args.kernel not in mandel.KERNELS:
        raise SystemExit(f"unknown --kernel {args.kernel}; choose from {sorted(mandel.KERNELS)}")
    kernel = args.kernel
    stream = torch.cuda.current_stream(dev)
    s_handle = stream.cuda_stream
    nbytes = cfg.W * cfg.H * 4

    # the root image (rank 0) and the shared FCFS counter, IPC-mapped on the other ranks
    rr = None
    if world == 1:
        img = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
        img_ptr = img.data_ptr()
    else:
        from paper_2007_00745_b200.multiproc import GatherRenderer, RankRenderer
        if args.gather == "nccl":
            rr = GatherRenderer(dist, rank, world, local, cfg.args(), cfg.dtype, s_handle,
                                chunk_rows=args.chunk_rows)
        else:
            rr = RankRenderer(dist, rank, world, local, cfg.args(), cfg.dtype, s_handle, images=2)
        img_ptr = rr.img
        img = None

    shared = None  # N > 1 e2e: the shared host image every rank drains a slice into

    def step(scheme, out_host=None, e2e=False, sync=True):
        """One render (N > 1: this rank's rows; the caller adds the device barrier)."""
        if world == 1:
            if e2e:
                # host output through the library, asynchronous and pipelined: render n+1
                # overlaps the banded device->host copy of render n (mandel_finish at the end)
                return mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, 1, out_host=out_host,
                                               stream0=s_handle, chunk_rows=args.chunk_rows,
                                               kernel=kernel, async_host=True, want_stats=False)
            # timed device-output renders are enqueued back to back; the last returns stats
            return mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, 1,
                                           out_host=out_host, out_dev0=img_ptr,
                                           stream0=s_handle, chunk_rows=args.chunk_rows,
                                           kernel=kernel, want_stats=sync or out_host is not None)
        # renders follow each other without a barrier (one FCFS counter slot per render);
        # e2e ends each render with one so that rank 0 copies a complete map
        st = rr.step(scheme, barrier=e2e, sync=sync or e2e, chunk_rows=args.chunk_rows, kernel=kernel)
        if e2e and shared is not None and shared.ok:
            # every rank pulls its slice of rank 0's map over NVLink and pushes it through
            # its own PCIe link into the shared host image; the barrier makes it whole
            shared.drain(img_ptr, cfg.W, cfg.H, world, s_handle)
            dist.barrier()
        elif out_host is not None and rank == 0:
            _d2h(out_host, img_ptr, nbytes, s_handle)  # rank 0 holds the whole map
        return st

    def timed(scheme, steps, warmup, sampler=None, out_host=None, e2e=False, barriered=True, per_render=False):
        """K renders bracketed by barrier + synchronize, max over ranks (the caller reduces).
        N > 1 and barriered: a device-side barrier (rr.device_barrier: an all_reduce on the
        render stream) follows every render, so render n+1 starts on every rank only after
        every rank finished render n -- each step is one whole render to the moment rank 0
        holds the map, FCFS tail included.  barriered=False: renders follow
        each other without a barrier (render n+1 fills render n's tail; pipelined).
        per_render: also bracket every render with its own pair of events (render_ms; a
        separate pass -- the two event records cost the host ~8 us per step, which on a
        small view would make the timed loop host-bound)."""
        stats = []
        for _ in range(warmup):
            step(scheme, out_host, e2e)
            if world > 1 and barriered and not e2e:
                rr.device_barrier()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.time()
        # per-render events on the launching stream (per_render pass only)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)] if per_render and not e2e else []
        e0.record(stream)
        for i in range(steps):
            # renders are enqueued back to back (no host round trip between them); the last
            # one returns the statistics
            if ev:
                ev[i][0].record(stream)
            st = step(scheme, out_host, e2e, sync=(i == steps - 1))
            if ev:
                ev[i][1].record(stream)
            if world > 1 and barriered and not e2e:
                rr.device_barrier()
            if st is not None:
                stats.append(st)
        if e2e and world == 1:
            mandel.mandel_finish()  # every render's map is in host memory
        e1.record(stream)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t1 = time.time()
        if sampler:
            sampler.mark(t0, t1)
        ms = e0.elapsed_time(e1)
        if ev:
            per = [a.elapsed_time(b) for a, b in ev]
            stats[-1]["render_ms_mean"] = statistics.mean(per)
            stats[-1]["render_ms_median"] = statistics.median(per)
            stats[-1]["render_ms_min"] = min(per)
        return ms, stats

    def e2e_pipelined(scheme, steps):
        """N > 1 end to end with the hand-off overlapped: render n+1 (into the other of
        rank 0's two maps) runs while every rank drains its slice of render n to the shared
        host image on a copy stream.  Per render: all ranks finish it (sync + barrier)
        before anyone drains it, and every drain of a map ends (sync + barrier) before
        anyone renders into that map again."""
        cstream = torch.cuda.Stream(dev)
        c_handle = cstream.cuda_stream

        def settle():
            mandel.mandel_sync(s_handle)
            mandel.mandel_sync(c_handle)
            dist.barrier()

        for _ in range(2):  # warm-up of the same sequence
            rr.step(scheme, sync=False, image=0, chunk_rows=args.chunk_rows, kernel=kernel)
            settle()
            shared.drain(rr.imgs[0], cfg.W, cfg.H, world, c_handle, wait=False)
            settle()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rr.step(scheme, sync=False, image=0, chunk_rows=args.chunk_rows, kernel=kernel)
        for n in range(steps):
            settle()  # render n done everywhere; drain n-1 done everywhere
            if n + 1 < steps:
                rr.step(scheme, sync=False, image=(n + 1) % 2, chunk_rows=args.chunk_rows, kernel=kernel)
            shared.drain(rr.imgs[n % 2], cfg.W, cfg.H, world, c_handle, wait=False)
        settle()
        stream.wait_stream(cstream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return e0.elapsed_time(e1)

    # the FP pipe peak of this GPU, measured live before the timed region (tools/fp_peak)
    peak_meas = measured_fp_peak(cfg.dtype) if rank == 0 else None
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ms, stats = timed(args.scheme, args.steps, args.warmup, sampler)
    sampler.stop()
    # per-render durations in a second pass (diagnostic: render_ms)
    _, rstats = timed(args.scheme, min(args.steps, 50), 2, per_render=True)
    from paper_2007_00745_b200.multiproc import sum_over_ranks
    iters_rank = stats[-1]["sum_iters"]  # this rank's share of the last step (FCFS: varies)
    iters_launch = statistics.mean(s["sum_iters"] for s in stats)  # per launch of this rank
    per_step = sum_over_ranks(dist, [s["sum_iters"] for s in stats], adev)
    assert all(v == per_step[0] for v in per_step), "the map's work differs between steps"
    tot_ms, _ = aggregate(dist, ms, 0, adev)
    iters_job = per_step[0]
    ms_per_step = tot_ms / args.steps
    value = iters_job / (ms_per_step * 1e-3) / 1e9  # Giter/s
    # the escape kernel's average launch duration: at N = 1 every timed step is exactly one
    # launch, back to back on the launching stream, so the timed region's events / K; at
    # N > 1 a step also holds the device barrier, so the per-render event pass
    kern_ms = ms / args.steps if world == 1 else rstats[-1]["render_ms_mean"]
    kern_basis = ("CUDA events around the K timed launches on the launching stream / K" if world == 1 else
                  "mean of per-render CUDA-event brackets on this rank's launching stream")
    clocks = sampler.summary()
    if clocks is not None:
        # the SM clock the escape kernels themselves measured (clock64 / %globaltimer per
        # CTA, mandel_stats.sm_clock_mhz) on the last timed render, next to nvidia-smi's
        clocks["sm_mhz_in_kernel"] = round(stats[-1].get("sm_clock_mhz", 0.0), 1)

    # roofline of the dominant kernel (the escape kernel): algorithmic FP ops per launch
    # (8 per pixel-iteration of this rank) / its CUDA-event duration on the launching stream
    achieved = iters_launch * FLOPS_PER_ITER / (kern_ms * 1e-3) / 1e12
    peak_uc = fp_peak_tflops(cfg.dtype)
    peak, peak_src = (peak_meas["tflops"], peak_meas["source"]) if peak_meas else (peak_uc, "unit counts")
    lanes = FP64_LANES if cfg.dtype == "fp64" else FP32_LANES
    roof = {"bound": "alu", "unit": "TFLOP/s", "achieved": round(achieved, 4),
            "peak": round(peak, 4), "frac": round(achieved / peak, 4),
            "traffic": None,
            "peak_basis": f"measured: {peak_src}",
            # the guide's unit-count figure beside the measured one
            "peak_unit_count": round(peak_uc, 4), "frac_unit_count": round(achieved / peak_uc, 4),
            "peak_unit_count_basis": f"{SMS} SMs x {lanes} {cfg.dtype.upper()} lanes x {SM_MAX_MHZ:.0f} MHz "
                                     "(max SM clock; DESIGN.md Roofline)",
            "kernel_ms": round(kern_ms, 4),
            "kernel_ms_basis": kern_basis,
            "ops_per_launch": int(iters_launch * FLOPS_PER_ITER),
            "ops_per_launch_basis": f"{FLOPS_PER_ITER} FP ops (3 mul + 5 add/sub) x {iters_launch:.0f} "
                                    "pixel-iterations (sum of this rank's counts) per launch",
            # the peak above is the FP pipe's lane-instruction rate (DADD/DMUL/DFMA: one each);
            # the path executes fewer FP instructions than the 8 counted flops per iteration --
            # the fused-y form does the *2 and +ci of Eq. 1's y-update in one FMA (R21)
            # and the batched test forms |z|^2 once per 8 updates (R18) -- so frac can pass 1.
            # Against the FMA flop peak (2 flops per lane-instruction) the same work is:
            "peak_fma_flops": round(2 * peak, 4),
            "frac_of_fma_flop_peak": round(achieved / (2 * peak), 4),
            "executed_vs_counted": "fewer than 8 FP instructions per counted iteration (fused-y FMA; "
                                   "batched |z|^2); ncu_pipe_active is the executed pipe utilisation",
            # the same time against the fewest FP instructions an exact evaluation needs per
            # iteration -- 6 per z-update in the fused form (x*x, y*y, x*y, -, +cr, fma) and the
            # |z|^2 add once per 8 updates (R18) -- so this fraction cannot pass 1
            "frac_min_fp_instr": round(iters_launch * MIN_FP_INSTR_PER_ITER / (kern_ms * 1e-3) / 1e12 / peak, 4),
            "min_fp_instr_per_iter": MIN_FP_INSTR_PER_ITER}
    prof = _traffic_from_profiles(cfg, world)
    if prof:
        # NOT measured in this run: read from the committed ncu --set full capture of this
        # kernel (profiles/): DRAM bytes per launch, and the FP pipe utilisation the kernel
        # actually EXECUTED -- the batched escape check (R18) executes fewer than 8 FP ops
        # per counted iteration, so `frac` (counted ops) can exceed the executed utilisation
        roof["traffic"] = prof.get("dram_bytes_per_launch")
        pipe = prof.get("fp64_pipe_active_pct" if cfg.dtype != "fp32" else "fma_pipe_active_pct")
        if pipe is not None:
            roof["ncu_pipe_active"] = round(pipe / 100.0, 4)
        # north_star's divergence evidence: active lanes per executed warp instruction
        # (smsp__thread_inst_executed_per_inst_executed.ratio / 32); the static
        # one-pixel-per-thread baseline beside it is in profiles/*_warp_efficiency.json
        if prof.get("warp_execution_efficiency") is not None:
            roof["ncu_warp_exec_eff"] = round(prof["warp_execution_efficiency"], 4)
        roof["ncu_kernel"] = prof.get("kernel")
        roof["traffic_source"] = (f"profiles/{os.path.basename(prof['_path'])}: committed ncu --set full "
                                  "capture of this kernel on this config (not measured in this run)")
    if clocks and clocks.get("sm_mhz"):
        roof["frac_unit_count_at_measured_clock"] = round(
            achieved / fp_peak_tflops(cfg.dtype, clocks["sm_mhz"]), 4)

    line = {
        "metric": "pixel-iterations/sec (Giter/s)",
        "value": round(value, 3),
        "unit": "Giter/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 4),
        # per-render CUDA-event times on rank 0's launching stream (PAPER.md:237 reports
        # repetitions; median and minimum)
        "render_ms": {"mean": round(rstats[-1]["render_ms_mean"], 4),
                      "median": round(rstats[-1]["render_ms_median"], 4),
                      "min": round(rstats[-1]["render_ms_min"], 4),
                      "steps": min(args.steps, 50),
                      "note": "a second pass with an event pair around every render (the timed "
                              "loop has events only around all K steps)"},
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "strong",
        "vs_baseline": None,
        "dtype": "f64" if cfg.dtype == "fp64" else "f32",
        "data": "synthetic (deterministic grid; no dataset)",
        "config": {
            "workload": f"{cfg.name}: {cfg.W}x{cfg.H} grid, [{cfg.xmin},{cfg.xmax}]x[{cfg.ymin},{cfg.ymax}], "
                        f"iterMax {cfg.iter_max}, R {cfg.R}, {cfg.dtype}",
            "scheme": args.scheme, "chunk_rows": args.chunk_rows, "kernel": args.kernel,
            "sum_iters_per_step": iters_job, "pixels": cfg.pixels,
            # what the kernels ran: the row order, and the FCFS claims the device counted
            # (Eq. 19 analog; ceil(H/chunk) per render when complete), summed over ranks
            "kernel_scheme": stats[-1].get("kernel_scheme"),
            "chunks_claimed_per_step": sum_over_ranks(dist, [stats[-1]["chunks_claimed"]], adev)[0],
            "kernel_variant": stats[-1].get("kernel"),
            "first_block_lanes": stats[-1].get("first_block"),
            "parallelism": f"{args.scheme} rows over {world} GPU(s)",
            "gather": "none (1 GPU)" if world == 1 else (
                "fused: every rank's kernel stores into rank 0's map over NVLink (CUDA IPC)"
                if args.gather == "fused" else
                "nccl: rank bands sent point-to-point to rank 0, K4 row scatter"),
            "l2": f"no input reads; each step writes a {nbytes / 2**20:.0f} MiB map "
                  "(> 126 MB L2) -- nothing to flush",
        },
        "gpu_launches": int(args.steps * stats[-1]["kernel_launches"]),  # one stats per timed loop
        "roofline": roof,
        "clocks": clocks,
    }

    if world > 1:
        # the headline steps above are barriered (each render whole before the next);
        # efficiency is judged on them.  Pipelined throughput beside it: the same renders
        # with no barrier between them (render n+1 fills render n's tail)
        line["render_ms_barriered"] = line["ms_per_step"]
        pms, _ = timed(args.scheme, args.steps, 2, barriered=False)
        pms_job, _ = aggregate(dist, pms, 0, adev)
        line["pipelined"] = {"value": round(iters_job / (pms_job / args.steps * 1e-3) / 1e9, 3),
                             "ms_per_step": round(pms_job / args.steps, 4),
                             "note": "renders back to back with no barrier between them: a fast rank's "
                                     "render n+1 overlaps render n's tail -- not the paper's per-render "
                                     "time; scaling efficiency is judged on `value` (barriered)"}
        line["timing"] = ("each timed step is one render followed by a device-side barrier (a 1-element "
                          "NCCL all_reduce on the render stream): render n+1 starts on every rank after "
                          "every rank finished render n; K steps bracketed by barrier + synchronize, "
                          "max over ranks")

    if not args.profile:
        # e2e: the same metric through the C ABI with a HOST destination (pinned), the
        # device->host copy of each step's map inside the timed region
        host = torch.empty((cfg.H, cfg.W), dtype=torch.int32, pin_memory=True) \
            if rank == 0 else None
        if world > 1:
            from paper_2007_00745_b200.multiproc import SharedHostImage
            shared = SharedHostImage(dist, rank, nbytes, _cudart())
        ne = max(1, args.e2e_steps)
        if world > 1 and shared.ok and args.gather == "fused":
            ems = e2e_pipelined(args.scheme, ne)
        else:
            ems, _ = timed(args.scheme, ne, 1, None, out_host=host if rank == 0 else None, e2e=True)
        ems_job, _ = aggregate(dist, ems, 0, adev)
        e2e_val = iters_job / (ems_job / ne * 1e-3) / 1e9
        line["e2e"] = {"value": round(e2e_val, 3), "unit": "Giter/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": nbytes, "steps": ne,
                       "note": "inputs are scalar kernel arguments (window, sizes, iterMax, R); "
                               "the map is copied device->host into pinned memory every step"}
        if world == 1:
            line["e2e"]["hand_off"] = ("mandel_render_ex(out_host, async_host): banded device->host "
                                       "copies, render n+1 overlapping the copies of render n; "
                                       "mandel_finish() inside the timed region")
        if world > 1:
            line["e2e"]["hand_off"] = (
                f"every rank copies 1/{world} of rank 0's map (NVLink, then its own PCIe link) "
                "into one shared page-locked host image" + (
                    "; the copy of render n overlaps render n+1 (two maps on rank 0)"
                    if args.gather == "fused" else "") if shared.ok else
                f"rank 0 copies the whole map (shared host image unavailable: {shared.error})")
        if rank == 0 and host is not None:
            total = shared.checksum() if (world > 1 and shared.ok) else \
                int(host.numpy().view(np.uint32).sum(dtype=np.uint64))
            line["e2e"]["map_sum_check"] = total == (iters_rank if world == 1 else iters_job)
        # latency: ONE synchronous render with the whole map landing in host memory --
        # the paper's "total process time", no overlap between
        # renders; the median of a few calls, host wall clock around the call (max over ranks)
        lat = []
        for _ in range(5):
            if dist is not None:
                dist.barrier()
            t0 = time.perf_counter()
            if world == 1:
                mandel.mandel_render_ex(*cfg.args(), cfg.dtype, args.scheme, 1, out_host=host,
                                        stream0=s_handle, chunk_rows=args.chunk_rows, kernel=kernel)
            else:
                rr.step(args.scheme, barrier=True, sync=True, chunk_rows=args.chunk_rows, kernel=kernel)
                if shared.ok:
                    shared.drain(img_ptr, cfg.W, cfg.H, world, s_handle)
                    dist.barrier()
                elif rank == 0:
                    _d2h(host, img_ptr, nbytes, s_handle)
            lat_ms = (time.perf_counter() - t0) * 1e3
            lat_ms, _ = aggregate(dist, lat_ms, 0, adev)
            lat.append(lat_ms)
        line["e2e"]["latency_ms"] = round(statistics.median(lat), 4)
        line["e2e"]["latency_note"] = ("one synchronous render + the whole map in pinned host memory, "
                                       "host wall clock around the call, median of 5 (the paper's total "
                                       "process time); `value` above overlaps consecutive renders")
        if shared is not None:
            shared.close()
            shared = None

        if not args.no_schemes:
            per = {}
            for sch in ("block", "cyclic", "fcfs"):
                if args.kernel == "static" and sch == "fcfs":
                    continue
                k = max(5, args.steps // 4)
                sms, sst = timed(sch, k, 2)
                sms_job, _ = aggregate(dist, sms, 0, adev)
                per[sch] = {"value": round(iters_job / (sms_job / k * 1e-3) / 1e9, 3),
                            "ms_per_step": round(sms_job / k, 4), "steps": k,
                            "kernel_scheme": sst[-1].get("kernel_scheme"),
                            "chunks_claimed": sst[-1].get("chunks_claimed")}
                if world > 1:
                    per[sch]["render_ms_barriered"] = per[sch]["ms_per_step"]
                    pms, _ = timed(sch, k, 2, barriered=False)
                    pms_job, _ = aggregate(dist, pms, 0, adev)
                    per[sch]["pipelined_value"] = round(iters_job / (pms_job / k * 1e-3) / 1e9, 3)
            line["per_scheme"] = per

        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_seconds, img)
    if args.share_device:
        line["test_only_shared_device"] = True  # N ranks on one GPU: not a measurement
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        rr.close()
        dist.destroy_process_group()


def _d2h(out_host, dev_ptr, nbytes, stream):
    """cudaMemcpyAsync(device -> pinned host) + sync, through the CUDA runtime torch ships."""
    import ctypes
    libcudart = _cudart()
    rc = libcudart.cudaMemcpyAsync(ctypes.c_void_p(out_host.data_ptr()), ctypes.c_void_p(dev_ptr),
                                   ctypes.c_size_t(nbytes), ctypes.c_int(2), ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"cudaMemcpyAsync failed: {rc}")
    libcudart.cudaStreamSynchronize(ctypes.c_void_p(stream))


_CUDART = None


def _cudart():
    global _CUDART
    if _CUDART is None:
        import ctypes
        import glob

        import torch
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
        cands += glob.glob(os.path.join(os.path.dirname(os.path.dirname(torch.__file__)),
                                        "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
        cands += ["libcudart.so", "/usr/local/cuda/lib64/libcudart.so"]
        for c in cands:
            try:
                _CUDART = ctypes.CDLL(c)
                break
            except OSError:
                continue
    return _CUDART


def _traffic_from_profiles(cfg, world):
    """dram read+write bytes per launch of the escape kernel from the committed ncu
    capture summary (profiles/*_traffic.json), or None."""
    import glob
    best = None

    def round_tag(path):  # r01 < r01w < r02a < r02z < r02aa: newer tags are longer or later
        tag = os.path.basename(path).split("_")[0]
        return (len(tag), tag)

    for p in sorted(glob.glob(os.path.join(ROOT, "profiles", "*traffic*.json")), key=round_tag):
        try:
            d = json.load(open(p))
        except (OSError, ValueError):
            continue
        if d.get("config") == cfg.name and d.get("n_gpus", 1) == world:
            best = d
            best["_path"] = p
    return best


def measured_fp_peak(dtype: str):
    """The FP pipe peak measured on this GPU right now: tools/fp_peak (8 independent
    DADD/DMUL -- FADD/FMUL for fp32 -- chains per thread at full occupancy; no FMA, as in
    the path), mean of the add and mul figures, in T lane-ops/s.  Falls back to the newest
    committed profiles/*fp_peak.json when the tool is not built or fails."""
    import glob
    exe = os.path.join(ROOT, "tools", "fp_peak")
    keys = ("dadd", "dmul") if dtype != "fp32" else ("fadd", "fmul")
    if os.access(exe, os.X_OK):
        try:
            r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
            d = json.loads(r.stdout)
            return {"tflops": sum(d[k]["tops"] for k in keys) / 2,
                    "source": f"tools/fp_peak run live before the timed region ({keys[0]}/{keys[1]} chains, "
                              f"{d['sms']} SMs x {d['ctas_per_sm']} CTAs; implied clock "
                              f"{d[keys[0]].get('implied_mhz', 0):.0f} MHz)"}
        except (OSError, ValueError, KeyError, subprocess.SubprocessError):
            pass
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_fp_peak.json")))
    for p in reversed(files):
        try:
            d = json.load(open(p))
            return {"tflops": sum(d[k]["tops"] for k in keys) / 2,
                    "source": f"profiles/{os.path.basename(p)} (committed tools/fp_peak run on a B200; "
                              "the tool was not runnable here)"}
        except (OSError, ValueError, KeyError):
            continue
    return None


# ---------------------------------------------------------------------------
# CPU baseline (oracle on the host cores) -- rank 0, N = 1 only
# ---------------------------------------------------------------------------
def cpu_sample_rows(cfg, cpu_seconds: float, cores: int, rate_per_core: float = 2.5e8):
    """Evenly strided rows whose estimated work is ~cpu_seconds core-seconds."""
    mean_row = cfg.W * {"C1": 22.1, "C2": 192.1, "C3": 192.1, "C4": 137.7, "C5": 474.8}.get(cfg.name, 200)
    nrows = int(max(8, min(cfg.H, cpu_seconds * rate_per_core / mean_row)))
    stride = max(1, cfg.H // nrows)
    return np.arange(stride // 2, cfg.H, stride)[:nrows]


def cpu_baseline(cfg, cpu_seconds, gpu_img=None):
    import oracle
    cores = oracle.host_cores()
    rows = cpu_sample_rows(cfg, cpu_seconds, cores)
    oracle.lib()
    t0 = time.perf_counter()
    # FCFS chunks small enough that every host thread gets work on a short sample
    chunk = max(1, min(16, len(rows) // (8 * cores)))
    ref, used = oracle.render_rows_mt(cfg, rows, threads=cores, chunk=chunk)
    dt = time.perf_counter() - t0
    iters = int(ref.sum(dtype=np.uint64))
    out = {"value": round(iters / dt / 1e9, 4), "unit": "Giter/s", "cores": used, "kind": "oracle",
           "sample": f"{len(rows)} evenly strided rows of {cfg.name} ({len(rows)}/{cfg.H} rows, "
                     f"{iters} pixel-iterations), plain C oracle (-O2 -ffp-contract=off) on "
                     f"{used} host threads claiming {chunk}-row chunks", "seconds": round(dt, 3),
           "core_seconds": round(dt * used, 2),  # the sample's CPU work (target --cpu-seconds)
           "per_core": round(iters / dt / 1e9 / used, 5)}
    # single-threaded rate: every 8th row of the same sample, one thread
    srows = rows[::8]
    t0 = time.perf_counter()
    sref, _ = oracle.render_rows_mt(cfg, srows, threads=1, chunk=1)
    sdt = time.perf_counter() - t0
    out["single_thread"] = {"value": round(int(sref.sum(dtype=np.uint64)) / sdt / 1e9, 5), "unit": "Giter/s",
                            "rows": int(len(srows)), "seconds": round(sdt, 3)}
    if gpu_img is not None:
        got = gpu_img[rows.tolist()].cpu().numpy().view(np.uint32)
        out["parity_rows_vs_gpu"] = {"rows": int(len(rows)), "mismatched_pixels": int((got != ref).sum())}
    return out


# ---------------------------------------------------------------------------
# reference arm: the oracle on host cores, bounded samples of the same workload
# ---------------------------------------------------------------------------
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return  # rank 0 alone runs and prints; the other ranks exit 0 without work
    import oracle
    cfg = wl.CONFIGS[args.config]
    cores = oracle.host_cores()
    oracle.lib()
    total_budget_s = 150.0
    per_step_s = total_budget_s / max(1, args.steps + args.warmup)
    rows_per_step = cpu_sample_rows(cfg, per_step_s * cores, cores).shape[0]
    stride = max(1, cfg.H // max(1, rows_per_step))

    def step(k):
        off = (k * 7919) % stride
        rows = np.arange(off, cfg.H, stride)[:rows_per_step]
        ref, _ = oracle.render_rows_mt(cfg, rows, threads=cores)
        return int(ref.sum(dtype=np.uint64))

    for k in range(args.warmup):
        step(k)
    t0 = time.perf_counter()
    iters = 0
    for k in range(args.steps):
        iters += step(args.warmup + k)
    dt = time.perf_counter() - t0
    value = iters / dt / 1e9
    line = {
        "impl": "reference",
        "metric": "pixel-iterations/sec (Giter/s)", "value": round(value, 4), "unit": "Giter/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f64" if cfg.dtype == "fp64" else "f32", "data": "synthetic (deterministic grid)",
        "config": {"workload": f"{cfg.name}: {cfg.W}x{cfg.H} grid, iterMax {cfg.iter_max}, R {cfg.R}, "
                               f"{cfg.dtype}; each step a {rows_per_step}-row strided sample",
                   "scheme": "fcfs (host threads, 16-row chunks)"},
        "cpu_baseline": {"value": round(value, 4), "unit": "Giter/s", "cores": cores, "kind": "oracle",
                         "sample": f"{rows_per_step} strided rows of {cfg.name} per step"},
        "e2e": {"value": round(value, 4), "unit": "Giter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    import faulthandler
    import signal
    faulthandler.register(signal.SIGUSR1, all_threads=True)  # stack dump of a stuck rank on demand
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
