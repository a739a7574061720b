#!/usr/bin/env python3
"""Development model: how often a warp's batched escape test hits, for two pixel
orders of the refill stream (row segments vs 2-D blocks), on a real count map.

A warp holds S slots; every B updates it tests; a batch in which >= 1 slot finishes
is a hit (replayed, then the finished slots are refilled from the stream).  The
model ignores tails and iterMax budget alignment; it only compares orders.

    python tools/sim_hits.py --config C2 --warps 400
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402


def warp_hits(counts, slots, B):
    """counts: the warp's pixel stream (escape counts in order). Returns (hits, batches)."""
    n = len(counts)
    rem = np.zeros(slots, dtype=np.int64)
    nxt = 0
    live = np.zeros(slots, dtype=bool)
    for s in range(slots):
        if nxt < n:
            rem[s] = counts[nxt]; live[s] = True; nxt += 1
    hits = batches = 0
    while live.any():
        fin = live & (rem <= B)
        batches += 1
        rem[live] -= B
        if fin.any():
            hits += 1
            for s in np.nonzero(fin)[0]:
                if nxt < n:
                    rem[s] = counts[nxt]; nxt += 1
                else:
                    live[s] = False
    return hits, batches


def stream(img, r0, c0, order, tile_w, tiles, tile_rows):
    out = []
    H, W = img.shape
    for t in range(tiles):
        if order == "row":
            r, c = r0 + t // max(1, W // tile_w), c0 + (t % max(1, W // tile_w)) * tile_w
            out.append(img[r, c:c + tile_w])
        else:  # tile_rows x (tile_w/tile_rows... ) block, 8-column sub-blocks, row-major inside
            cols = tile_w // tile_rows
            r = r0 + (t // max(1, W // cols)) * tile_rows
            c = c0 + (t % max(1, W // cols)) * cols
            blk = img[r:r + tile_rows, c:c + cols]
            for sb in range(0, blk.shape[1], 8):
                out.append(blk[:, sb:sb + 8].reshape(-1))
    return np.concatenate(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--warps", type=int, default=300)
    ap.add_argument("--slots", type=int, default=64)
    ap.add_argument("--B", type=int, default=8)
    ap.add_argument("--scale", type=int, default=4, help="render at 1/scale of the size (same pixel pitch window crop)")
    a = ap.parse_args()
    import oracle
    cfg = wl.CONFIGS[a.config]
    # a crop at the full resolution: the centre 1/scale of the image
    H = cfg.H // a.scale
    rows = np.arange((cfg.H - H) // 2, (cfg.H + H) // 2)
    img, _ = oracle.render_rows_mt(cfg, rows)
    c0 = (cfg.W - H) // 2
    img = img[:, c0:c0 + H]
    rng = np.random.default_rng(1)
    res = {}
    for order, tr in (("row", 1), ("block", 4), ("block", 8)):
        h = b = px = it = 0
        for _ in range(a.warps):
            r0 = int(rng.integers(0, img.shape[0] - 64))
            cc = int(rng.integers(0, img.shape[1] - 1024))
            s = stream(img[:, cc:], r0, 0, order, 256, 4, tr)
            hh, bb = warp_hits(s.astype(np.int64), a.slots, a.B)
            h += hh; b += bb; px += len(s); it += int(s.sum())
        res[f"{order}{tr}"] = {"hits_per_kpx": round(1000 * h / px, 2), "hit_frac": round(h / b, 4),
                               "batches": b, "iters_per_hit": round(it / max(1, h), 1)}
    print(res)


if __name__ == "__main__":
    main()
