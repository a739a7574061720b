#!/usr/bin/env python3
"""Render a view with the library and write it as a binary PPM (P6).

The whole pipeline runs through the C ABI: mandel_render_ex (escape counts into a
device map), mandel_colorize (device counts -> RGB bytes), mandel_write_ppm (host).

    python examples/render_ppm.py --out set.ppm                      # the full set, 2000 x 2000
    python examples/render_ppm.py --centre -0.743643887 0.131825904 --width 1e-4 \\
        --size 4096 --iter-max 10000 --palette classic --out zoom.ppm
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2007_00745_b200 import mandel  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--centre", type=float, nargs=2, default=(-0.5, 0.0))
    ap.add_argument("--width", type=float, default=4.0, help="window width (and height) in the complex plane")
    ap.add_argument("--size", type=int, default=2000, help="W = H in pixels")
    ap.add_argument("--iter-max", type=int, default=1000)
    ap.add_argument("--radius", type=float, default=2.0)
    ap.add_argument("--dtype", default="fp64", choices=sorted(mandel.DTYPES))
    ap.add_argument("--palette", default="gray", choices=["gray", "classic"])
    ap.add_argument("--out", default="mandelbrot.ppm")
    a = ap.parse_args()
    cx, cy = a.centre
    h = a.width / 2
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev).cuda_stream
    counts = torch.empty((a.size, a.size), dtype=torch.int32, device=dev)
    st = mandel.mandel_render_ex(cx - h, cx + h, cy - h, cy + h, a.size, a.size, a.iter_max, a.radius,
                                 a.dtype, "fcfs", 1, out_dev0=counts, stream0=stream)
    rgb = torch.empty(a.size * a.size * 3, dtype=torch.uint8, device=dev)
    mandel.mandel_colorize(counts, rgb, a.size, a.size, a.iter_max, a.palette, stream)
    host = rgb.cpu().numpy()
    n = mandel.mandel_write_ppm(a.out, host, a.size, a.size)
    print(f"{a.out}: {n} bytes; {st['sum_iters'] / 1e9:.3f} G pixel-iterations in {st['kernel_ms_max']:.2f} ms "
          f"({st['sum_iters'] / st['kernel_ms_max'] / 1e6:.0f} Giter/s, kernel {st['kernel']}{st['kernel_ilp']})")


if __name__ == "__main__":
    main()
