"""An independent numpy re-implementation of the escape-time map (tests only).

Written from the paper's Eq. 1 and Eq. 2 and the Cx/Cy
mapping under DESIGN.md's readings, separately from oracle.c, so
that a transcription slip in either (an operand order, a sign, an index) shows
up as a disagreement.  numpy ufuncs round each operation on its own (no
contraction), and numpy 2 keeps float32 arrays in float32 when combined with
float32 scalars.
"""
from __future__ import annotations

import numpy as np


def np_map(xmin, xmax, ymin, ymax, W, H, iter_max, R, dtype="fp64", rows=None):
    T = np.float64 if dtype == "fp64" else np.float32
    lo_x, hi_x, lo_y, hi_y, rad = (T(v) for v in (xmin, xmax, ymin, ymax, R))
    dx = (hi_x - lo_x) / T(W)
    dy = (hi_y - lo_y) / T(H)
    r2 = rad * rad
    rows = np.arange(H) if rows is None else np.asarray(rows)
    cols = np.arange(W)
    re_axis = lo_x + cols.astype(T) * dx           # Cx[j] = xmin + j*dx
    im_axis = hi_y - rows.astype(T) * dy           # Cy[i] = ymax - i*dy
    cr = np.broadcast_to(re_axis[None, :], (rows.size, W)).ravel().copy()
    ci = np.broadcast_to(im_axis[:, None], (rows.size, W)).ravel().copy()
    assert cr.dtype == T and ci.dtype == T
    count = np.full(cr.size, iter_max, dtype=np.uint32)
    live = np.arange(cr.size)
    zr = np.zeros(cr.size, T)
    zi = np.zeros(cr.size, T)
    for n in range(1, iter_max + 1):
        a, b, c_r, c_i = zr[live], zi[live], cr[live], ci[live]
        re_new = (a * a - b * b) + c_r               # Re(z^2 + c)
        im_new = (a + a) * b + c_i                   # Im(z^2 + c)
        mag2 = re_new * re_new + im_new * im_new     # |z|^2
        zr[live] = re_new
        zi[live] = im_new
        gone = mag2 > r2
        count[live[gone]] = n
        live = live[~gone]
        if live.size == 0:
            break
    return count.reshape(rows.size, W)
