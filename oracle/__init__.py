"""CPU oracle for arXiv 2007.00745's escape-time Mandelbrot map.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2007_00745_b200`` never imports it and
shares no code with it (the only shared module is ``workloads.py``, which holds
configuration values and seeded generators, none of the method's arithmetic).

Layers:
  * ``oracle.c`` -> ``liboracle.so``: Eq. 1/Eq. 2 per pixel, the Cx/Cy mapping
    and row/pixel drivers (see its header for the passages it follows).
  * ``partition.py``: the paper's three row-partition schemes, Eq. 14-20.

Every function cites the passage it follows; DESIGN.md lists the readings taken
where the paper is silent.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

FP64 = 0
FP32 = 1
FP64_FMA = 2

_lib = None
_lock = threading.Lock()

BUILD_CMD = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math",
             "-fPIC", "-shared", "-o", _LIB_PATH, _SRC, "-lm"]


def build(force: bool = False) -> str:
    """Compile oracle.c with contraction off (no FMA), as the header states."""
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(BUILD_CMD)
    return _LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB_PATH)
            u32, f64, f32, i32 = ctypes.c_uint32, ctypes.c_double, ctypes.c_float, ctypes.c_int
            L.oracle_escape_f64.argtypes = [f64, f64, u32, f64]
            L.oracle_escape_f64.restype = u32
            L.oracle_escape_f64fma.argtypes = [f64, f64, u32, f64]
            L.oracle_escape_f64fma.restype = u32
            L.oracle_escape_f32.argtypes = [f32, f32, u32, f32]
            L.oracle_escape_f32.restype = u32
            L.oracle_derive_f64.argtypes = [f64, f64, f64, f64, u32, u32, f64, ctypes.c_void_p]
            L.oracle_derive_f64.restype = None
            L.oracle_derive_f32.argtypes = [f64, f64, f64, f64, u32, u32, f64, ctypes.c_void_p]
            L.oracle_derive_f32.restype = None
            for name, t in (("oracle_cx_f64", f64), ("oracle_cy_f64", f64),
                            ("oracle_cx_f32", f32), ("oracle_cy_f32", f32)):
                fn = getattr(L, name)
                fn.argtypes = [t, t, u32]
                fn.restype = t
            L.oracle_render_rows.argtypes = [f64, f64, f64, f64, u32, u32, u32, f64, i32,
                                             u32, u32, ctypes.c_void_p]
            L.oracle_render_rows.restype = i32
            L.oracle_render_pixels.argtypes = [f64, f64, f64, f64, u32, u32, u32, f64, i32,
                                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                               ctypes.c_void_p]
            L.oracle_render_pixels.restype = i32
            _lib = L
    return _lib


def _dt(dtype) -> int:
    if dtype in (FP64, "fp64", "f64", "float64"):
        return FP64
    if dtype in (FP32, "fp32", "f32", "float32"):
        return FP32
    if dtype in (FP64_FMA, "fp64fma"):
        return FP64_FMA
    raise ValueError(f"unknown dtype {dtype!r}")


def escape(cr: float, ci: float, iter_max: int, R: float, dtype="fp64") -> int:
    """Eq. 1 + Eq. 2 for one point; R is a radius (R2 = R*R in dtype)."""
    L = lib()
    if _dt(dtype) == FP64:
        return int(L.oracle_escape_f64(cr, ci, iter_max, R * R))
    if _dt(dtype) == FP64_FMA:
        return int(L.oracle_escape_f64fma(cr, ci, iter_max, R * R))
    rf = float(np.float32(R))
    r2 = float(np.float32(rf) * np.float32(rf))
    return int(L.oracle_escape_f32(float(np.float32(cr)), float(np.float32(ci)), iter_max, r2))


def derive(xmin, xmax, ymin, ymax, W, H, R, dtype="fp64"):
    """Step a1: (dx, dy, R2) in fp64, or (xmin_f, ymax_f, dx, dy, R2) in fp32."""
    L = lib()
    if _dt(dtype) in (FP64, FP64_FMA):
        out = (ctypes.c_double * 3)()
        L.oracle_derive_f64(xmin, xmax, ymin, ymax, W, H, R, ctypes.addressof(out))
        return tuple(out)
    out = (ctypes.c_float * 5)()
    L.oracle_derive_f32(xmin, xmax, ymin, ymax, W, H, R, ctypes.addressof(out))
    return tuple(out)


def axes(xmin, xmax, ymin, ymax, W, H, R, dtype="fp64"):
    """Step a3: the Cx and Cy arrays as numpy arrays."""
    L = lib()
    if _dt(dtype) in (FP64, FP64_FMA):
        dx, dy, _ = derive(xmin, xmax, ymin, ymax, W, H, R, "fp64")
        cx = np.array([L.oracle_cx_f64(xmin, dx, j) for j in range(W)], dtype=np.float64)
        cy = np.array([L.oracle_cy_f64(ymax, dy, i) for i in range(H)], dtype=np.float64)
        return cx, cy
    xa, yb, dx, dy, _ = derive(xmin, xmax, ymin, ymax, W, H, R, "fp32")
    cx = np.array([L.oracle_cx_f32(xa, dx, j) for j in range(W)], dtype=np.float32)
    cy = np.array([L.oracle_cy_f32(yb, dy, i) for i in range(H)], dtype=np.float32)
    return cx, cy


def render_rows(xmin, xmax, ymin, ymax, W, H, iter_max, R, dtype="fp64",
                row0: int = 0, row1: int | None = None) -> np.ndarray:
    """Rows [row0, row1) of the map as a (rows, W) uint32 array (single thread)."""
    if row1 is None:
        row1 = H
    out = np.zeros((row1 - row0, W), dtype=np.uint32)
    rc = lib().oracle_render_rows(xmin, xmax, ymin, ymax, W, H, iter_max, R, _dt(dtype),
                                  row0, row1, out.ctypes.data)
    if rc != 0:
        raise ValueError("oracle_render_rows rejected its arguments")
    return out


def render(cfg, dtype=None) -> np.ndarray:
    """The whole map of a workloads.Config (single thread)."""
    return render_rows(cfg.xmin, cfg.xmax, cfg.ymin, cfg.ymax, cfg.W, cfg.H, cfg.iter_max,
                       cfg.R, dtype or cfg.dtype)


def render_pixels(cfg, ii, jj, dtype=None) -> np.ndarray:
    """Counts at pixels (ii[p], jj[p]) of a workloads.Config."""
    ii = np.ascontiguousarray(ii, dtype=np.uint32)
    jj = np.ascontiguousarray(jj, dtype=np.uint32)
    out = np.zeros(ii.shape[0], dtype=np.uint32)
    rc = lib().oracle_render_pixels(cfg.xmin, cfg.xmax, cfg.ymin, cfg.ymax, cfg.W, cfg.H,
                                    cfg.iter_max, cfg.R, _dt(dtype or cfg.dtype),
                                    ii.ctypes.data, jj.ctypes.data, ii.shape[0],
                                    out.ctypes.data)
    if rc != 0:
        raise ValueError("oracle_render_pixels rejected its arguments")
    return out


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def render_rows_mt(cfg, rows, threads: int | None = None, chunk: int = 16, dtype=None):
    """Rows ``rows`` (an index array) of cfg on ``threads`` host threads.

    The row-level parallel driver of the CPU baseline: threads claim 16-row
    chunks first-come-first-served (the paper's FCFS scheme, PAPER.md:205-207,
    with a shared counter instead of a master).  ctypes releases the GIL during
    each oracle_render_rows call, so the threads run on separate cores.  The
    per-pixel arithmetic is exactly render_rows'.  Returns (map[len(rows), W],
    threads used).
    """
    rows = np.asarray(rows, dtype=np.int64)
    threads = threads or host_cores()
    out = np.zeros((rows.shape[0], cfg.W), dtype=np.uint32)
    nxt = [0]
    lk = threading.Lock()
    L = lib()
    dt = _dt(dtype or cfg.dtype)

    def worker():
        while True:
            with lk:
                s = nxt[0]
                nxt[0] += chunk
            if s >= rows.shape[0]:
                return
            for k in range(s, min(s + chunk, rows.shape[0])):
                r = int(rows[k])
                rc = L.oracle_render_rows(cfg.xmin, cfg.xmax, cfg.ymin, cfg.ymax, cfg.W, cfg.H,
                                          cfg.iter_max, cfg.R, dt, r, r + 1,
                                          out[k].ctypes.data)
                if rc != 0:
                    raise ValueError("oracle_render_rows rejected its arguments")

    with ThreadPoolExecutor(max_workers=threads) as ex:
        futs = [ex.submit(worker) for _ in range(threads)]
        for f in futs:
            f.result()
    return out, threads
