#!/usr/bin/env python3
"""Pipelined host hand-off probe: kernel-only vs banded end-to-end render times."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402

cfg = wl.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
dev = torch.device("cuda", 0)
s = torch.cuda.current_stream(dev).cuda_stream
host = torch.empty((cfg.H, cfg.W), dtype=torch.int32, pin_memory=True)
dmap = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
for _ in range(2):
    mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 1, out_dev0=dmap, stream0=s)
st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 1, out_dev0=dmap, stream0=s)
print(json.dumps({"mode": "device", "kernel_ms": st["kernel_ms_max"], "device_ms": st["device_ms"]}))
t0 = time.perf_counter(); torch.cuda.synchronize()
host.copy_(dmap, non_blocking=True); torch.cuda.synchronize()
print(json.dumps({"mode": "plain_d2h_copy_ms", "ms": (time.perf_counter() - t0) * 1e3,
                  "gbs": cfg.W * cfg.H * 4 / (time.perf_counter() - t0) / 1e9}))
tapers = [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["100", "70"])]
blist = [int(v) for v in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["1", "4", "8", "12", "16"])]
for bands in blist:
    for taper in tapers:
        if bands == 1 and taper != tapers[0]:
            continue
        res = []
        for _ in range(5):
            t0 = time.perf_counter()
            st = mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 1, out_host=host, stream0=s,
                                         bands=bands, band_taper=taper)
            res.append(((time.perf_counter() - t0) * 1e3, st["device_ms"], st["d2h_ms"]))
        best = min(res)
        print(json.dumps({"mode": "host", "config": cfg.name, "bands": bands, "taper": taper,
                          "wall_ms": round(best[0], 3), "compute_ms": round(best[1], 3),
                          "exposed_d2h_ms": round(best[2], 3)}), flush=True)
