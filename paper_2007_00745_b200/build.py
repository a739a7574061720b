"""In-tree build of libmandel.so (sm_100a) -- invoked by __graft_entry__.build().

The library is compiled with -fmad=false as a second guard on top of the
explicit __dadd_rn/__dmul_rn intrinsics (no FMA contraction anywhere on the
device), and the host code with -ffp-contract=off (step a1 constants).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libmandel.so")
SOURCES = [os.path.join(CSRC, "mandel.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "mandel_kernels.cuh"), os.path.join(CSRC, "mandel_image.cuh"),
                  os.path.join(ROOT, "include", "mandel.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def src_hash(define: str = "") -> str:
    """Content hash of the sources (and the build flags) a library is built from: a copy of
    the tree with fresh file times (the gpurun snapshot) must not look up to date."""
    import hashlib
    h = hashlib.sha1(" ".join(NVCC_FLAGS + [define]).encode())
    for d in DEPS:
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _stale(lib: str, define: str = "") -> bool:
    try:
        with open(lib + ".srchash") as f:
            return f.read().strip() != src_hash(define)
    except OSError:
        return True


def _stamp(lib: str, define: str = "") -> None:
    with open(lib + ".srchash", "w") as f:
        f.write(src_hash(define) + "\n")


def needs_build() -> bool:
    return not os.path.exists(LIB) or _stale(LIB)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-o", LIB + ".tmp", *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libmandel.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    _stamp(LIB)
    with open(os.path.join(PKG, "ptxas_resources.txt"), "w") as f:
        f.write(res.stderr)
    return LIB


def build_debug(out: str = None, define: str = "MANDEL_DEBUG_CHECKS=1", name: str = "libmandel_debug.so") -> str:
    """libmandel_debug.so: the same library with device-side bounds/alignment checks
    (MANDEL_DEBUG_CHECKS=1); load it with MANDEL_LIB=... to run the tests against it.
    build_prof() uses it for the LAZY-loop instrumentation (MANDEL_LAZY_PROF=1)."""
    out = out or os.path.join(PKG, name)
    cmd = [nvcc(), *NVCC_FLAGS, "-D" + define, "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           "-o", out, *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {name}")
    _stamp(out, define)
    return out


def build_delay(force: bool = False) -> str:
    """libmandel_delay.so: random sleeps around every FCFS claim, binding and some stores
    (MANDEL_FCFS_DELAY=1; tests/test_fcfs_stress.py runs it through tools/fcfs_delay_stress.py)."""
    out = os.path.join(PKG, "libmandel_delay.so")
    if force or not os.path.exists(out) or _stale(out, "MANDEL_FCFS_DELAY=1"):
        build_debug(out, "MANDEL_FCFS_DELAY=1", "libmandel_delay.so")
    return out


def build_trace(out: str = None) -> str:
    """libmandel_trace.so: one timeline record per warp (tools/trace_view.py)."""
    return build_debug(out, "MANDEL_TRACE=1", "libmandel_trace.so")


def build_prof(out: str = None) -> str:
    """libmandel_prof.so: LAZY slot-state counters printed per launch (tools/lazy_prof.py)."""
    return build_debug(out, "MANDEL_LAZY_PROF=1", "libmandel_prof.so")


TOOLS = ["fp_peak", "loop_bench", "fp_latency"]  # FP-pipe micro-benchmarks (tools/*.cu)


def build_tools(force: bool = False) -> list:
    """nvcc the micro-benchmarks the roofline peak and issue model rest on."""
    procs, outs = [], []
    for t in TOOLS:
        src, out = os.path.join(ROOT, "tools", t + ".cu"), os.path.join(ROOT, "tools", t)
        outs.append(out)
        if not force and os.path.exists(out) and os.path.getmtime(out) >= os.path.getmtime(src):
            continue
        procs.append((t, subprocess.Popen([nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                                           "-lineinfo", "-fmad=false", "-o", out, src],
                                          stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    for t, pr in procs:
        o, e = pr.communicate()
        if pr.returncode != 0:
            sys.stderr.write(o + e)
            raise RuntimeError(f"nvcc failed building tools/{t}")
    return outs


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
