#!/usr/bin/env python3
"""Host cost of the enqueue path (development tool): wall time per call while the GPU
sleeps (so nothing waits on the device), for each layer of a bench step."""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
s = stream.cuda_stream
N = 200


def per_call(fn):
    torch.cuda.synchronize()
    torch.cuda._sleep(int(N * 60e3 * 2))  # the GPU is busy for the whole loop
    t0 = time.perf_counter()
    for _ in range(N):
        fn()
    dt = (time.perf_counter() - t0) / N * 1e6
    torch.cuda.synchronize()
    return round(dt, 2)


res = {}
for cfg in (wl.C1.with_(W=8, H=8), wl.C1):
    out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
    for _ in range(3):
        mandel.mandel_render_ex(*cfg.args(), "fp64", "block", 1, out_dev0=out, stream0=s)
    torch.cuda.synchronize()
    res[f"{cfg.W}x{cfg.H} render_ex enqueue (python)"] = per_call(
        lambda: mandel.mandel_render_ex(*cfg.args(), "fp64", "block", 1, out_dev0=out, stream0=s, want_stats=False))
    # the C call alone: options and pointers prepared once
    L = mandel.lib()
    o = mandel._opts()
    ptr = ctypes.c_void_p(out.data_ptr())
    args = (*cfg.args(), 0, 0, 1, ctypes.byref(o), None, ptr, ctypes.c_void_p(s), None)
    res[f"{cfg.W}x{cfg.H} mandel_render_ex C call"] = per_call(lambda: L.mandel_render_ex(*args))
e = torch.cuda.Event(enable_timing=True)
res["torch event record"] = per_call(lambda: e.record(stream))
res["ctypes trivial call (abi_version)"] = per_call(lambda: mandel.mandel_abi_version())
res["_opts()"] = per_call(lambda: mandel._opts(0, 0, "refill"))
print(json.dumps(res, indent=1))
