import sys, time, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2007_00745_b200 import mandel
import workloads as wl
dev = torch.device("cuda", 0); s = torch.cuda.current_stream(dev).cuda_stream
for cfg in (wl.C1.with_(W=8, H=8), wl.C1):
    out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
    for _ in range(5): mandel.mandel_render_ex(*cfg.args(), "fp64", "fcfs", 1, out_dev0=out, stream0=s)
    torch.cuda.synchronize()
    for ws in (False, True):
        t0 = time.perf_counter(); n = 200
        for _ in range(n): mandel.mandel_render_ex(*cfg.args(), "fp64", "fcfs", 1, out_dev0=out, stream0=s, want_stats=ws)
        torch.cuda.synchronize(); dt = (time.perf_counter() - t0) / n * 1e6
        print(cfg.W, cfg.H, "stats" if ws else "async", round(dt, 1), "us/call")
t0 = time.perf_counter()
for _ in range(2000): mandel.mandel_abi_version()
print("ctypes trivial call", round((time.perf_counter() - t0) / 2000 * 1e6, 2), "us")
o = None
t0 = time.perf_counter()
for _ in range(2000): o = mandel._opts(0, 0, "refill")
print("_opts", round((time.perf_counter() - t0) / 2000 * 1e6, 2), "us")
