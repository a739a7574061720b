#!/usr/bin/env python3
"""A compact tour of every kernel variant and host path, each render checked against
the oracle (written to run under compute-sanitizer, which this GPU pool disables;
it runs plain as a quick smoke of every path):

    python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import workloads as wl  # noqa: E402
from paper_2007_00745_b200 import mandel  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream(dev).cuda_stream
    cases = [wl.C1.with_(W=131, H=77, iter_max=300), wl.C1.with_(W=64, H=200, iter_max=150, dtype="fp32"),
             wl.C1.with_(W=100, H=61, iter_max=200, dtype="fp64fma"),
             wl.Config("zoom", -0.7437, -0.7435, 0.1317, 0.1319, 96, 64, 2000, 2.0, "fp64")]
    kernels = ["refill", "refill1", "refill2", "lazy2", "adaptive2", "batch4x2", "batch8x2", "batch16x1",
               "adaptb8x2", "static"]
    n = 0
    for cfg in cases:
        want = oracle.render(cfg)
        out = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
        for kern in kernels:
            if kern.startswith("batch16") and cfg.dtype == "fp32":
                continue
            for scheme, ng in (("block", 1), ("cyclic", 3), ("fcfs", 2), ("fcfs_master", 3)):
                if kern == "static" and scheme.startswith("fcfs"):
                    continue
                out.zero_()
                mandel.mandel_render_ex(*cfg.args(), cfg.dtype, scheme, ng, out_dev0=out, stream0=s,
                                        logical_ranks=ng > 1, kernel=kern, tile_rows=[0, 1, 4][n % 3])
                got = out.cpu().numpy().view(np.uint32)
                assert np.array_equal(got, want), (cfg.name, kern, scheme)
                n += 1
        # host output: pipelined bands, tapers
        for bands, taper in ((0, 0), (3, 40), (7, 100)):
            got, _ = mandel.render(*cfg.args(), cfg.dtype, "fcfs", 1, bands=bands, band_taper=taper)
            assert np.array_equal(got, want), (cfg.name, bands, taper)
            n += 1
        # band mode + K4 scatter, SM-sliced ranks
        img = torch.zeros((cfg.H, cfg.W), dtype=torch.int32, device=dev)
        ctr = torch.zeros(64, dtype=torch.int32, device=dev)
        cap = -(-cfg.H // 16) * 16
        for r in range(3):
            band = torch.zeros((cap, cfg.W), dtype=torch.int32, device=dev)
            mandel.mandel_render_rank(*cfg.args(), cfg.dtype, "fcfs", r, 3, band, ctr, s, band_out=True,
                                      max_sms=2)
            rows = mandel.mandel_band_rows()
            if len(rows):
                rd = torch.from_numpy(rows.view(np.int32)).to(dev)
                mandel.mandel_scatter_rows(band, rd, len(rows), cfg.W, img, s)
        torch.cuda.synchronize()
        assert np.array_equal(img.cpu().numpy().view(np.uint32), want), (cfg.name, "band")
        n += 1
        # output stage
        rgb = torch.zeros(cfg.pixels * 3, dtype=torch.uint8, device=dev)
        mandel.mandel_colorize(out, rgb, cfg.W, cfg.H, cfg.iter_max, "classic", s)
    print(f"sanitize_run: {n} renders bit-exact")


if __name__ == "__main__":
    main()
