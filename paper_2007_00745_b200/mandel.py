"""Thin ctypes binding of libmandel.so (include/mandel.h), same names as the C ABI.

Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  There is no CPU fallback -- if the shared library is missing or
fails to load this module raises, and on a machine without a CUDA device the
compute calls return MANDEL_ENODEV (raised as MandelError).
"""
from __future__ import annotations

import ctypes
import os
import re
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# MANDEL_LIB: an alternative build of the same library (A/B measurements only)
LIB_PATH = os.environ.get("MANDEL_LIB") or os.path.join(_HERE, "libmandel.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "mandel.h")

MANDEL_FP64, MANDEL_FP32, MANDEL_FP64_FMA = 0, 1, 2
MANDEL_BLOCK, MANDEL_CYCLIC, MANDEL_FCFS, MANDEL_FCFS_MASTER = 0, 1, 2, 3
MANDEL_OK, MANDEL_EINVAL, MANDEL_ENODEV, MANDEL_ENOMEM = 0, -1, -2, -3
MANDEL_ECUDA, MANDEL_ECOMM, MANDEL_EBUSY, MANDEL_EIO = -4, -5, -6, -7
MANDEL_COLOUR_GRAY, MANDEL_COLOUR_CLASSIC = 0, 1
COLOURS = {"gray": MANDEL_COLOUR_GRAY, "grey": MANDEL_COLOUR_GRAY, "classic": MANDEL_COLOUR_CLASSIC}
MANDEL_KERNEL_REFILL, MANDEL_KERNEL_STATIC, MANDEL_KERNEL_EAGER, MANDEL_KERNEL_LAZY = 0, 1, 2, 3
MANDEL_KERNEL_ADAPTIVE = 4
# name -> (mandel_kernel, ilp); ilp 0 = the library's default for that kernel
KERNELS = {"refill": (0, 0), "static": (1, 0), "eager": (2, 0), "lazy": (3, 0),
           "refill1": (2, 1), "refill2": (2, 2), "refill3": (2, 3), "refill4": (2, 4),
           "lazy1": (3, 1), "lazy2": (3, 2), "adaptive": (4, 0), "adaptive1": (4, 1),
           "adaptive2": (4, 2),
           # EAGER with the batched escape check (check_every 4 / 8; R18)
           "batch4x1": (2, 1, 4), "batch4x2": (2, 2, 4), "batch4x4": (2, 4, 4),
           "batch8x1": (2, 1, 8), "batch8x2": (2, 2, 8), "batch8x3": (2, 3, 8), "batch8x4": (2, 4, 8),
           "batch16x1": (2, 1, 16), "batch16x2": (2, 2, 16), "batch16x4": (2, 4, 16),
           # ADAPTIVE on batched EAGER runs (lazy runs where escapes are dense)
           "adaptb4x1": (4, 1, 4), "adaptb4x2": (4, 2, 4), "adaptb8x1": (4, 1, 8), "adaptb8x2": (4, 2, 8)}
MANDEL_MAX_GPUS = 64
MANDEL_IPC_HANDLE_BYTES = 64

DTYPES = {"fp64": MANDEL_FP64, "fp32": MANDEL_FP32, "fp64fma": MANDEL_FP64_FMA}
SCHEMES = {"block": MANDEL_BLOCK, "naive": MANDEL_BLOCK, "cyclic": MANDEL_CYCLIC,
           "alternating": MANDEL_CYCLIC, "fcfs": MANDEL_FCFS, "fcfs_master": MANDEL_FCFS_MASTER}


class MandelError(RuntimeError):
    def __init__(self, code: int, where: str, detail: str = ""):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} ({code}) {detail}".strip())


class mandel_stats(ctypes.Structure):
    _fields_ = [
        ("device_ms", ctypes.c_double),
        ("kernel_ms_max", ctypes.c_double),
        ("kernel_ms", ctypes.c_double * MANDEL_MAX_GPUS),
        ("d2h_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("sum_iters", ctypes.c_uint64),
        ("pixels", ctypes.c_uint64),
        ("rank_iters", ctypes.c_uint64 * MANDEL_MAX_GPUS),
        ("rank_pixels", ctypes.c_uint64 * MANDEL_MAX_GPUS),
        ("rank_rows", ctypes.c_uint32 * MANDEL_MAX_GPUS),
        ("chunks_claimed", ctypes.c_uint32),
        ("transfers", ctypes.c_uint32),
        ("kernel_launches", ctypes.c_uint32),
        ("ngpus", ctypes.c_uint32),
        ("ndevices", ctypes.c_uint32),
        ("kernel_variant", ctypes.c_int32),
        ("kernel_ilp", ctypes.c_int32),
        ("probe", ctypes.c_float * 2),
        ("warp_iters", ctypes.c_uint64),
        ("loop_exits", ctypes.c_uint64),
        ("kernel_batch", ctypes.c_int32),
        ("kernel_packed", ctypes.c_int32),
        ("sm_clock_mhz", ctypes.c_double),
        ("kernel_scheme", ctypes.c_int32),
        ("store_mode", ctypes.c_int32),
        ("fused_y", ctypes.c_int32),
        ("host_handoff", ctypes.c_int32),
        ("first_block", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        n = max(int(self.ngpus), 1)
        return {
            "device_ms": self.device_ms, "kernel_ms_max": self.kernel_ms_max,
            "kernel_ms": list(self.kernel_ms[:n]), "d2h_ms": self.d2h_ms,
            "total_ms": self.total_ms, "sum_iters": int(self.sum_iters),
            "pixels": int(self.pixels), "rank_iters": [int(v) for v in self.rank_iters[:n]],
            "rank_pixels": [int(v) for v in self.rank_pixels[:n]],
            "rank_rows": [int(v) for v in self.rank_rows[:n]],
            "chunks_claimed": int(self.chunks_claimed), "transfers": int(self.transfers),
            "kernel_launches": int(self.kernel_launches), "ngpus": int(self.ngpus),
            "ndevices": int(self.ndevices),
            "kernel": {0: "refill", 1: "static", 2: "eager", 3: "lazy", 4: "adaptive"}.get(
                int(self.kernel_variant), str(self.kernel_variant)),
            "kernel_ilp": int(self.kernel_ilp), "probe": [float(v) for v in self.probe],
            "warp_iters": int(self.warp_iters), "loop_exits": int(self.loop_exits),
            "kernel_batch": int(self.kernel_batch), "kernel_packed": int(self.kernel_packed),
            "sm_clock_mhz": float(self.sm_clock_mhz),
            "fused_y": int(self.fused_y),
            "first_block": int(self.first_block),
            "host_handoff": "per_device" if int(self.host_handoff) else "gpu0",
            "store_mode": {0: "direct", 1: "staged", 2: "staged_vec"}.get(int(self.store_mode), str(self.store_mode)),
            "kernel_scheme": {v: k for k, v in SCHEMES.items() if k not in ("naive", "alternating")}.get(
                int(self.kernel_scheme), str(self.kernel_scheme)),
        }


class mandel_options(ctypes.Structure):
    _fields_ = [
        ("chunk_rows", ctypes.c_uint32),
        ("tile_px", ctypes.c_uint32),
        ("kernel", ctypes.c_int),
        ("logical_ranks", ctypes.c_int),
        ("refill_lanes", ctypes.c_int),
        ("ilp", ctypes.c_int),
        ("min_ctas", ctypes.c_int),
        ("adapt_lo", ctypes.c_int),
        ("adapt_hi", ctypes.c_int),
        ("bands", ctypes.c_int),
        ("band_taper", ctypes.c_int),
        ("tile_rows", ctypes.c_int),
        ("band_out", ctypes.c_int),
        ("no_pack", ctypes.c_int),
        ("max_sms", ctypes.c_int),
        ("async_host", ctypes.c_int),
        ("check_every", ctypes.c_int),
        ("stage", ctypes.c_int),
        ("ctas_per_sm", ctypes.c_int),
        ("fused_y", ctypes.c_int),
        ("host_handoff", ctypes.c_int),
        ("first_block", ctypes.c_int),
    ]


_lib = None
_lock = threading.Lock()

_SCALARS = [ctypes.c_double] * 4 + [ctypes.c_uint32] * 3 + [ctypes.c_double]


def lib():
    """Load libmandel.so; raise if it is missing (no fallback path exists)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                  "(the CUDA library is the only implementation)")
            L = ctypes.CDLL(LIB_PATH)
            i32, u32, vp = ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p
            L.mandel_render.argtypes = _SCALARS + [i32, i32, i32, vp]
            L.mandel_render.restype = i32
            L.mandel_render_ex.argtypes = _SCALARS + [i32, i32, i32, vp, vp, vp, vp, vp]
            L.mandel_render_ex.restype = i32
            L.mandel_render_rank.argtypes = _SCALARS + [i32, i32, i32, i32, vp, vp, vp, vp, vp]
            L.mandel_render_rank.restype = i32
            L.mandel_plan_rows.argtypes = [i32, u32, i32, i32, vp, vp]
            L.mandel_plan_rows.restype = i32
            L.mandel_strerror.argtypes = [i32]
            L.mandel_strerror.restype = ctypes.c_char_p
            L.mandel_last_error.argtypes = []
            L.mandel_last_error.restype = ctypes.c_char_p
            L.mandel_device_count.argtypes = []
            L.mandel_device_count.restype = i32
            L.mandel_shutdown.argtypes = []
            L.mandel_shutdown.restype = None
            L.mandel_abi_version.argtypes = []
            L.mandel_abi_version.restype = i32
            L.mandel_dev_alloc.argtypes = [i32, ctypes.c_size_t, vp]
            L.mandel_dev_alloc.restype = i32
            L.mandel_dev_free.argtypes = [vp]
            L.mandel_dev_free.restype = i32
            L.mandel_ipc_handle.argtypes = [vp, vp]
            L.mandel_ipc_handle.restype = i32
            L.mandel_ipc_open.argtypes = [i32, vp, vp]
            L.mandel_ipc_open.restype = i32
            L.mandel_colorize.argtypes = [vp, vp, u32, u32, u32, i32, vp]
            L.mandel_colorize.restype = i32
            L.mandel_write_ppm.argtypes = [ctypes.c_char_p, vp, u32, u32, vp]
            L.mandel_write_ppm.restype = i32
            L.mandel_dev_zero.argtypes = [vp, ctypes.c_size_t, vp]
            L.mandel_dev_zero.restype = i32
            L.mandel_ipc_close.argtypes = [vp]
            L.mandel_ipc_close.restype = i32
            L.mandel_finish.argtypes = []
            L.mandel_finish.restype = i32
            L.mandel_sync.argtypes = [vp]
            L.mandel_sync.restype = i32
            L.mandel_band_rows.argtypes = [vp, vp]
            L.mandel_band_rows.restype = i32
            L.mandel_scatter_rows.argtypes = [vp, vp, u32, u32, vp, vp]
            L.mandel_scatter_rows.restype = i32
            _lib = L
    return _lib


def header_symbols() -> list[str]:
    """Function names include/mandel.h declares (for the export test)."""
    text = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(mandel_\w+)\s*\(", text, re.M)))


def strerror(code: int) -> str:
    return lib().mandel_strerror(code).decode()


def last_error() -> str:
    return lib().mandel_last_error().decode()


def _check(rc: int, where: str):
    if rc != MANDEL_OK:
        raise MandelError(rc, where, last_error())


def _enum(v, table):
    return table[v] if isinstance(v, str) else int(v)


def _ptr(a) -> int | None:
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    raise TypeError(f"cannot take a pointer of {type(a)}")


def _buf(a, nbytes: int, name: str) -> int | None:
    """_ptr of an output buffer the library writes ``nbytes`` through: numpy arrays and
    torch tensors must be C-contiguous, have 4-byte elements and hold at least nbytes
    (a raw integer pointer is the caller's responsibility)."""
    if a is None or isinstance(a, int):
        return a
    if isinstance(a, np.ndarray):
        ok_layout = a.flags.c_contiguous and a.flags.writeable
        item, size = a.itemsize, a.nbytes
    elif hasattr(a, "data_ptr"):
        ok_layout = bool(a.is_contiguous())
        item, size = a.element_size(), a.numel() * a.element_size()
    else:
        raise TypeError(f"{name}: cannot take a pointer of {type(a)}")
    if not ok_layout:
        raise ValueError(f"{name} must be a C-contiguous, writable buffer")
    if item != 4:
        raise ValueError(f"{name} must have 4-byte elements (uint32/int32), not {item}-byte")
    if size < nbytes:
        raise ValueError(f"{name} holds {size} bytes; the map needs {nbytes} (W*H*4)")
    return _ptr(a)


def _opts(chunk_rows=0, tile_px=0, kernel=MANDEL_KERNEL_REFILL, logical_ranks=False,
          refill_lanes=0, ilp=0, min_ctas=0, adapt_lo=0, adapt_hi=0, bands=0, check_every=0,
          tile_rows=0, no_pack=False, band_out=False, band_taper=0, max_sms=0, async_host=False,
          stage=0, ctas_per_sm=0, fused_y=0, host_handoff=0, first_block=0):
    """kernel: a mandel_kernel value or a KERNELS name (which may also fix ilp)."""
    o = mandel_options()
    if isinstance(kernel, str):
        kernel, kilp, *kce = KERNELS[kernel]
        ilp = ilp or kilp
        check_every = check_every or (kce[0] if kce else 0)
    o.refill_lanes = refill_lanes or 0
    o.ilp = ilp or 0
    o.min_ctas = min_ctas or 0
    o.adapt_lo = adapt_lo or 0
    o.adapt_hi = adapt_hi or 0
    o.bands = bands or 0
    o.check_every = check_every or 0
    o.tile_rows = tile_rows or 0
    o.no_pack = 1 if no_pack else 0
    o.band_out = 1 if band_out else 0
    o.band_taper = band_taper or 0
    o.max_sms = max_sms or 0
    o.async_host = 1 if async_host else 0
    o.stage = int(stage)
    o.ctas_per_sm = int(ctas_per_sm)
    o.fused_y = int(fused_y)
    o.host_handoff = int(host_handoff)
    o.first_block = int(first_block)
    o.chunk_rows = chunk_rows or 0
    o.tile_px = tile_px or 0
    o.kernel = kernel
    o.logical_ranks = 1 if logical_ranks else 0
    return o


def mandel_device_count() -> int:
    return int(lib().mandel_device_count())


def mandel_abi_version() -> int:
    return int(lib().mandel_abi_version())


def mandel_shutdown() -> None:
    lib().mandel_shutdown()


def mandel_render(xmin, xmax, ymin, ymax, W, H, iter_max, R, dtype, scheme, ngpus, out) -> None:
    """C: mandel_render.  ``out``: host numpy uint32 array (or torch CPU tensor) of W*H."""
    rc = lib().mandel_render(xmin, xmax, ymin, ymax, W, H, iter_max, R, _enum(dtype, DTYPES),
                             _enum(scheme, SCHEMES), ngpus, _buf(out, W * H * 4, "out"))
    _check(rc, "mandel_render")


def mandel_render_ex(xmin, xmax, ymin, ymax, W, H, iter_max, R, dtype="fp64", scheme="block",
                     ngpus=1, *, out_host=None, out_dev0=None, stream0=None, chunk_rows=0,
                     tile_px=0, kernel=MANDEL_KERNEL_REFILL, logical_ranks=False,
                     refill_lanes=0, ilp=0, min_ctas=0, adapt_lo=0, adapt_hi=0,
                     bands=0, check_every=0, tile_rows=0, no_pack=False, band_taper=0,
                     max_sms=0, async_host=False, stage=0, ctas_per_sm=0, fused_y=0, host_handoff=0,
                     first_block=0, want_stats=True):
    """C: mandel_render_ex.  out_host: numpy/pinned tensor; out_dev0: CUDA tensor or
    device pointer on device 0; stream0: cudaStream_t handle (int) on device 0.
    Returns the call's statistics as a dict; want_stats=False (device output only)
    enqueues the render on stream0 without waiting and returns None."""
    need = W * H * 4
    host_p, dev_p = _buf(out_host, need, "out_host"), _buf(out_dev0, need, "out_dev0")
    st = mandel_stats() if want_stats else None
    o = _opts(chunk_rows=chunk_rows, tile_px=tile_px, kernel=kernel, logical_ranks=logical_ranks,
              refill_lanes=refill_lanes, ilp=ilp, min_ctas=min_ctas, adapt_lo=adapt_lo,
              adapt_hi=adapt_hi, bands=bands, check_every=check_every, tile_rows=tile_rows,
              no_pack=no_pack, band_taper=band_taper, max_sms=max_sms, async_host=async_host,
              stage=stage, ctas_per_sm=ctas_per_sm, fused_y=fused_y, host_handoff=host_handoff,
              first_block=first_block)
    rc = lib().mandel_render_ex(xmin, xmax, ymin, ymax, W, H, iter_max, R, _enum(dtype, DTYPES),
                                _enum(scheme, SCHEMES), ngpus, ctypes.byref(o), host_p,
                                dev_p, stream0, ctypes.byref(st) if st is not None else None)
    _check(rc, "mandel_render_ex")
    return st.as_dict() if st is not None else None


def mandel_render_rank(xmin, xmax, ymin, ymax, W, H, iter_max, R, dtype, scheme, rank, nranks,
                       out_root, fcfs_counter=None, stream=None, chunk_rows=0, tile_px=0,
                       kernel=MANDEL_KERNEL_REFILL, refill_lanes=0, ilp=0,
                       min_ctas=0, adapt_lo=0, adapt_hi=0, check_every=0, tile_rows=0,
                       no_pack=False, band_out=False, max_sms=0, stage=0, fused_y=0, first_block=0,
                       want_stats=True):
    """C: mandel_render_rank (one process per GPU).  out_root / fcfs_counter are device
    pointers valid in this process (own, or mapped with mandel_ipc_open).
    want_stats=False: the render is only enqueued on ``stream``; returns None."""
    # out_root: the whole image, or (band_out) this rank's band -- whose row count depends
    # on the plan, so only the layout is checked for a band
    root_p = _buf(out_root, 0 if band_out else W * H * 4, "out_root")
    st = mandel_stats() if want_stats else None
    o = _opts(chunk_rows=chunk_rows, tile_px=tile_px, kernel=kernel, refill_lanes=refill_lanes,
              ilp=ilp, min_ctas=min_ctas, adapt_lo=adapt_lo, adapt_hi=adapt_hi,
              check_every=check_every, tile_rows=tile_rows, no_pack=no_pack, band_out=band_out,
              max_sms=max_sms, stage=stage, fused_y=fused_y, first_block=first_block)
    rc = lib().mandel_render_rank(xmin, xmax, ymin, ymax, W, H, iter_max, R, _enum(dtype, DTYPES),
                                  _enum(scheme, SCHEMES), rank, nranks, ctypes.byref(o),
                                  root_p, _ptr(fcfs_counter), stream,
                                  ctypes.byref(st) if st is not None else None)
    _check(rc, "mandel_render_rank")
    return st.as_dict() if st is not None else None


def mandel_plan_rows(scheme, H: int, ngpus: int, rank: int) -> np.ndarray:
    """C: mandel_plan_rows (host-only planner of the static schemes)."""
    L = lib()
    cnt = ctypes.c_uint32(0)
    _check(L.mandel_plan_rows(_enum(scheme, SCHEMES), H, ngpus, rank, None, ctypes.byref(cnt)),
           "mandel_plan_rows")
    rows = np.zeros(cnt.value, dtype=np.uint32)
    _check(L.mandel_plan_rows(_enum(scheme, SCHEMES), H, ngpus, rank,
                              rows.ctypes.data if cnt.value else None, ctypes.byref(cnt)),
           "mandel_plan_rows")
    return rows


def mandel_band_rows() -> np.ndarray:
    """C: mandel_band_rows (image row of each band row of the last band_out render)."""
    L = lib()
    cnt = ctypes.c_uint32(0)
    _check(L.mandel_band_rows(None, ctypes.byref(cnt)), "mandel_band_rows")
    rows = np.zeros(cnt.value, dtype=np.uint32)
    if cnt.value:
        _check(L.mandel_band_rows(rows.ctypes.data, ctypes.byref(cnt)), "mandel_band_rows")
    return rows


def mandel_scatter_rows(band_dev, rows_dev, nrows: int, W: int, image_dev, stream=None) -> None:
    """C: mandel_scatter_rows (K4: image[rows[b]] = band[b], device pointers/tensors)."""
    _check(lib().mandel_scatter_rows(_ptr(band_dev), _ptr(rows_dev), nrows, W, _ptr(image_dev), stream),
           "mandel_scatter_rows")


def mandel_dev_alloc(device: int, nbytes: int) -> int:
    p = ctypes.c_void_p(0)
    _check(lib().mandel_dev_alloc(device, nbytes, ctypes.byref(p)), "mandel_dev_alloc")
    return int(p.value)


def mandel_dev_free(ptr: int) -> None:
    _check(lib().mandel_dev_free(ptr), "mandel_dev_free")


def mandel_finish() -> None:
    """C: mandel_finish (every asynchronous render's host output complete)."""
    _check(lib().mandel_finish(), "mandel_finish")


def mandel_sync(stream=None) -> None:
    """C: mandel_sync (wait for the stream, or the current device when None)."""
    _check(lib().mandel_sync(stream), "mandel_sync")


def mandel_dev_zero(ptr: int, nbytes: int, stream=None) -> None:
    _check(lib().mandel_dev_zero(ptr, nbytes, stream), "mandel_dev_zero")


def mandel_ipc_handle(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(MANDEL_IPC_HANDLE_BYTES)
    _check(lib().mandel_ipc_handle(ptr, buf), "mandel_ipc_handle")
    return buf.raw


def mandel_ipc_open(device: int, handle: bytes) -> int:
    if len(handle) != MANDEL_IPC_HANDLE_BYTES:
        raise ValueError("IPC handle must be MANDEL_IPC_HANDLE_BYTES long")
    p = ctypes.c_void_p(0)
    _check(lib().mandel_ipc_open(device, handle, ctypes.byref(p)), "mandel_ipc_open")
    return int(p.value)


def mandel_ipc_close(ptr: int) -> None:
    _check(lib().mandel_ipc_close(ptr), "mandel_ipc_close")


def mandel_colorize(counts_dev, rgb_dev, W, H, iter_max, mode="gray", stream=None) -> None:
    """C: mandel_colorize (device counts -> device RGB bytes)."""
    _check(lib().mandel_colorize(_ptr(counts_dev), _ptr(rgb_dev), W, H, iter_max,
                                 _enum(mode, COLOURS), stream), "mandel_colorize")


def mandel_write_ppm(path: str, rgb_host, W: int, H: int) -> int:
    """C: mandel_write_ppm (binary P6); returns the bytes written."""
    n = ctypes.c_uint64(0)
    _check(lib().mandel_write_ppm(os.fsencode(path), _ptr(rgb_host), W, H, ctypes.byref(n)),
           "mandel_write_ppm")
    return int(n.value)


def render(xmin, xmax, ymin, ymax, W, H, iter_max, R, dtype="fp64", scheme="block", ngpus=1,
           **kw):
    """Convenience: the map as a (H, W) numpy uint32 array plus the stats dict."""
    out = np.zeros((H, W), dtype=np.uint32)
    st = mandel_render_ex(xmin, xmax, ymin, ymax, W, H, iter_max, R, dtype, scheme, ngpus,
                          out_host=out, **kw)
    return out, st
