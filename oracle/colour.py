"""Colour map and PPM encoding (oracle side, TEST INFRASTRUCTURE ONLY).

PAPER.md:31 ("The iteration is then used to determine the pixel color") gives no
palette; SPEC.md:313-321 defines the grayscale ramp (interior black,
v = round(255 (n-1)/(M-1)) on escaped pixels) and SPEC.md:325-329 the P6 file:
"P6\\n<width> <height>\\n255\\n" + H*W RGB triples, row-major top to bottom.
Rounding is half up (R16); "classic" is this repo's integer palette
(7n, 13n, 29n mod 256).  Plain numpy, written independently of the CUDA kernel.
"""
from __future__ import annotations

import numpy as np

GRAY, CLASSIC = 0, 1


def colour(counts: np.ndarray, iter_max: int, mode: int = GRAY) -> np.ndarray:
    n = counts.astype(np.int64)
    out = np.zeros(n.shape + (3,), dtype=np.uint8)
    esc = n < iter_max
    if mode == GRAY:
        if iter_max >= 2:
            # round half up of 255 (n-1) / (M-1), exact in integers
            v = (510 * (n - 1) + (iter_max - 1)) // (2 * (iter_max - 1))
            for c in range(3):
                out[..., c] = np.where(esc, v, 0).astype(np.uint8)
    else:
        for c, k in enumerate((7, 13, 29)):
            out[..., c] = np.where(esc, (k * n) % 256, 0).astype(np.uint8)
    return out


def ppm_bytes(rgb: np.ndarray) -> bytes:
    H, W, _ = rgb.shape
    return f"P6\n{W} {H}\n255\n".encode() + np.ascontiguousarray(rgb, dtype=np.uint8).tobytes()
