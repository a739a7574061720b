"""Workload definitions and seeded input generators shared by tests, bench and smoke.

This module holds INPUTS only -- window bounds, grid sizes, iteration caps and
seeded random small configurations.  It contains none of the method's
arithmetic (no escape loop, no pixel->c mapping, no partition), so both the
oracle (``oracle/``) and the CUDA path (``paper_2007_00745_b200/``) may be fed
from it without sharing code.

The five configurations are BASELINE.json's ``configs``:

  C1  800 x 800,   [-2.5,1.5]x[-2,2], iterMax 200,   R 2, fp64  (small; oracle in ms)
  C2  8000 x 8000, same plane,        iterMax 2000,  R 2, fp64  (the paper's image size,
                                                              PAPER.md:237; bench workload)
  C3  8000 x 8000, same plane,        iterMax 2000,  R 2, fp32
  C4  16384^2 zoom centred at -0.743643887+0.131825904i, width = height = 1e-4,
      iterMax 10000, R 2, fp64  (boundary divergence / row imbalance stress)
  C5  32768^2, full plane, iterMax 5000, R 2, fp64  (4 GiB map; scaling config)

All inputs are deterministic grids: there is no dataset, and the paper prints
no per-pixel values.  The paper's window is never stated
(SPEC.md:107,118); [-2.5,1.5]x[-2,2] is BASELINE.json's choice (R6).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    xmin: float
    xmax: float
    ymin: float
    ymax: float
    W: int
    H: int
    iter_max: int
    R: float
    dtype: str  # "fp64" | "fp32"

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)

    @property
    def pixels(self) -> int:
        return self.W * self.H

    def args(self):
        """The scalar arguments of mandel_render / oracle_render_rows, in order."""
        return (self.xmin, self.xmax, self.ymin, self.ymax, self.W, self.H, self.iter_max, self.R)


FULL_PLANE = (-2.5, 1.5, -2.0, 2.0)

# C4 zoom window: centre -/+ half width, computed once in fp64 and passed as the
# same doubles to both sides.
_C4_CR, _C4_CI, _C4_HALF = -0.743643887, 0.131825904, 1e-4 / 2
ZOOM_WINDOW = (_C4_CR - _C4_HALF, _C4_CR + _C4_HALF, _C4_CI - _C4_HALF, _C4_CI + _C4_HALF)

C1 = Config("C1", *FULL_PLANE, 800, 800, 200, 2.0, "fp64")
C2 = Config("C2", *FULL_PLANE, 8000, 8000, 2000, 2.0, "fp64")
C3 = Config("C3", *FULL_PLANE, 8000, 8000, 2000, 2.0, "fp32")
C4 = Config("C4", *ZOOM_WINDOW, 16384, 16384, 10000, 2.0, "fp64")
C5 = Config("C5", *FULL_PLANE, 32768, 32768, 5000, 2.0, "fp64")

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}

# The paper's own experiment: 8000x8000, 2000 iterations,
# "Escape Radius 400" read as |z|^2 > 400, i.e. R = 20 (R1).
PAPER_GRID = Config("PAPER", *FULL_PLANE, 8000, 8000, 2000, 20.0, "fp64")


def random_small_configs(n: int = 50, seed0: int = 0, dtype: str = "fp64") -> list[Config]:
    """Seeded small configurations (SPEC.md:478-479 acceptance shape): H 5-64,
    W 4-32, iterMax 16-64, random windows intersecting the set's neighbourhood.
    numpy default_rng(seed) for seed in seed0..seed0+n-1."""
    out = []
    for s in range(seed0, seed0 + n):
        rng = np.random.default_rng(s)
        H = int(rng.integers(5, 65))
        W = int(rng.integers(4, 33))
        it = int(rng.integers(16, 65))
        cx = float(rng.uniform(-2.0, 0.6))
        cy = float(rng.uniform(-1.2, 1.2))
        w = float(10.0 ** rng.uniform(-3, 0.6))
        h = float(w * rng.uniform(0.5, 2.0))
        R = float(rng.choice([2.0, 2.0, 2.0, 20.0, 1.5]))
        out.append(Config(f"rand{s}", cx - w / 2, cx + w / 2, cy - h / 2, cy + h / 2,
                          W, H, it, R, dtype))
    return out


def sample_rows(H: int, n: int, seed: int = 0, include=(0,)) -> np.ndarray:
    """A seeded, sorted sample of n distinct rows, always including ``include``
    and the last row (ragged tails, mirror partners)."""
    rng = np.random.default_rng(seed)
    rows = set(int(r) for r in include if 0 <= r < H)
    rows.add(H - 1)
    rows.add(H // 2)
    while len(rows) < min(n, H):
        rows.add(int(rng.integers(0, H)))
    return np.array(sorted(rows), dtype=np.int64)


def sample_pixels(W: int, H: int, n: int, seed: int = 0):
    """A seeded sample of n pixel coordinates (ii, jj) including the four corners."""
    rng = np.random.default_rng(seed)
    ii = rng.integers(0, H, size=n).astype(np.uint32)
    jj = rng.integers(0, W, size=n).astype(np.uint32)
    ii[:4] = [0, 0, H - 1, H - 1]
    jj[:4] = [0, W - 1, 0, W - 1]
    return ii, jj
