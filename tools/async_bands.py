import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import workloads as wl
from paper_2007_00745_b200 import mandel
dev = torch.device("cuda", 0)
for name in ("C2", "C3", "C4"):
    cfg = wl.CONFIGS[name]
    host = torch.empty((cfg.H, cfg.W), dtype=torch.int32, pin_memory=True)
    for _ in range(2):
        mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 1, out_host=host)
    for bands in (1, 2, 4, 0):
        for _ in range(2):
            mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 1, out_host=host, async_host=True, want_stats=False, bands=bands)
        mandel.mandel_finish()
        n = 10
        t0 = time.perf_counter()
        for _ in range(n):
            mandel.mandel_render_ex(*cfg.args(), cfg.dtype, "fcfs", 1, out_host=host, async_host=True, want_stats=False, bands=bands)
        mandel.mandel_finish()
        dt = (time.perf_counter() - t0) / n * 1e3
        print(json.dumps({"config": name, "bands": bands, "ms_per_frame": round(dt, 3)}), flush=True)
