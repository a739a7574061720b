"""The C-ABI boundary without a GPU: the library loads, exports every symbol the
header declares, validates arguments (EINVAL before any device work), and
reports ENODEV instead of falling back to the CPU when no device is present."""
import ctypes
import math
import subprocess

import numpy as np
import pytest

import workloads as wl


def test_exports_every_header_symbol(mandel):
    names = mandel.header_symbols()
    assert "mandel_render" in names and "mandel_plan_rows" in names and len(names) >= 14
    L = mandel.lib()
    for n in names:
        assert hasattr(L, n), n
    # and the dynamic symbol table really has them (extern "C", unmangled)
    out = subprocess.run(["nm", "-D", "--defined-only", mandel.LIB_PATH],
                         capture_output=True, text=True).stdout
    for n in names:
        assert f" T {n}\n" in out or out.endswith(f" T {n}"), n


def test_library_is_sm100a_only(mandel):
    out = subprocess.run(["cuobjdump", "--list-elf", mandel.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", mandel.LIB_PATH], capture_output=True,
                          text=True).stdout
    # no FMA contraction in any kernel except the explicit FMA dtype's (R10, R17);
    # elsewhere the only FMA is the fused-y form fma(RN(x y), 2, ci) (R21): an exact doubling
    # of its first operand, the immediate 2 -- never a contracted multiply-add pair
    import re
    fn, fma_fns, fused = None, 0, 0
    doubling = re.compile(r"\b[DF]FMA R\d+, R\d+(\.reuse)?, 2, R\d+(\.reuse)? ;")
    for line in sass.splitlines():
        if "Function :" in line:
            fn = line.split("Function :")[1].strip()
            continue
        if "DFMA" in line or "FFMA" in line:
            if fn and "ArithF64Fma" in fn:
                fma_fns += 1
            else:
                assert doubling.search(line), (fn, line)
                fused += 1
    assert fma_fns > 0 and fused > 0


def test_abi_version_and_strerror(mandel):
    assert mandel.mandel_abi_version() == 10
    for code in range(-7, 1):
        assert mandel.strerror(code) and mandel.strerror(code) != "unknown status"


def _call(mandel, **kw):
    a = dict(xmin=-2.5, xmax=1.5, ymin=-2.0, ymax=2.0, W=8, H=8, iter_max=10, R=2.0,
             dtype=0, scheme=0, ngpus=1)
    a.update(kw)
    out = np.zeros(max(a["W"] * a["H"], 1), dtype=np.uint32)
    return mandel.lib().mandel_render(a["xmin"], a["xmax"], a["ymin"], a["ymax"], a["W"], a["H"],
                                      a["iter_max"], a["R"], a["dtype"], a["scheme"], a["ngpus"],
                                      out.ctypes.data)


BAD_ARGS = [
    dict(W=0), dict(H=0), dict(iter_max=0), dict(iter_max=0xFFFFFFFF), dict(R=0.0), dict(R=-1.0), dict(R=math.inf),
    dict(R=1e200), dict(xmin=math.nan), dict(ymax=math.inf), dict(xmin=1.5), dict(ymin=2.0),
    dict(dtype=3), dict(dtype=-1), dict(dtype=2, R=1e200), dict(scheme=4), dict(scheme=3, ngpus=1), dict(H=3, ngpus=4),
    dict(dtype=1, R=1e20), dict(dtype=1, xmin=-1e39), dict(dtype=1, xmin=1.0, xmax=1.0 + 1e-12),
    dict(W=0xFFFFFFFF, H=0xFFFFFFFF) if ctypes.sizeof(ctypes.c_size_t) == 4 else dict(W=0),
]


@pytest.mark.parametrize("kw", BAD_ARGS)
def test_einval(mandel, kw):
    assert _call(mandel, **kw) == mandel.MANDEL_EINVAL, kw
    assert mandel.last_error()


def test_null_outputs_rejected(mandel):
    L = mandel.lib()
    rc = L.mandel_render(-2.5, 1.5, -2.0, 2.0, 8, 8, 10, 2.0, 0, 0, 1, None)
    assert rc == mandel.MANDEL_EINVAL
    rc = L.mandel_render_ex(-2.5, 1.5, -2.0, 2.0, 8, 8, 10, 2.0, 0, 0, 1, None, None, None,
                            None, None)
    assert rc == mandel.MANDEL_EINVAL
    rc = L.mandel_render_rank(-2.5, 1.5, -2.0, 2.0, 8, 8, 10, 2.0, 0, 0, 0, 1, None, None,
                              None, None, None)
    assert rc == mandel.MANDEL_EINVAL
    rc = L.mandel_render_rank(-2.5, 1.5, -2.0, 2.0, 8, 8, 10, 2.0, 0, 0, 2, 2, None,
                              ctypes.c_void_p(16), None, None, None)
    assert rc == mandel.MANDEL_EINVAL


def test_no_device_means_enodev_not_fallback(mandel):
    if mandel.mandel_device_count() > 0:
        pytest.skip("a CUDA device is present")
    assert _call(mandel) == mandel.MANDEL_ENODEV
    with pytest.raises(mandel.MandelError) as e:
        mandel.render(*wl.C1.args())
    assert e.value.code == mandel.MANDEL_ENODEV


def test_band_api_host_checks(mandel):
    # band_out belongs to mandel_render_rank; the band row list is empty before any band render
    L = mandel.lib()
    o = mandel._opts(band_out=True)
    out = np.zeros(wl.C1.pixels, np.uint32)
    rc = L.mandel_render_ex(*wl.C1.args(), 0, 0, 1, ctypes.byref(o), out.ctypes.data, None, None, None)
    assert rc == mandel.MANDEL_EINVAL and "band_out" in mandel.last_error()
    assert mandel.mandel_band_rows().size == 0
    assert L.mandel_scatter_rows(None, None, 0, 8, None, None) == mandel.MANDEL_OK  # nothing to do
    assert L.mandel_scatter_rows(None, None, 4, 8, None, None) == mandel.MANDEL_EINVAL
    cnt = ctypes.c_uint32(0)
    assert L.mandel_band_rows(None, None) == mandel.MANDEL_EINVAL
    assert L.mandel_band_rows(None, ctypes.byref(cnt)) == mandel.MANDEL_OK and cnt.value == 0


def test_binding_validates_output_buffers(mandel):
    """The binding checks caller buffers before the library writes W*H*4 bytes through
    them: too small, wrong element size and non-contiguous are rejected
    with ValueError before any library call."""
    import torch
    cfg = wl.C1.with_(W=16, H=12)
    bad = [np.zeros(cfg.pixels - 1, np.uint32),              # one element short
           np.zeros(cfg.pixels, np.uint16),                  # 2-byte elements
           np.zeros((cfg.H, 2 * cfg.W), np.uint32)[:, ::2],  # strided view
           torch.zeros(cfg.pixels, dtype=torch.float64),     # 8-byte elements
           torch.zeros((cfg.W, cfg.H), dtype=torch.int32).t()]  # non-contiguous tensor
    for b in bad:
        with pytest.raises(ValueError):
            mandel.mandel_render(*cfg.args(), "fp64", "block", 1, b)
        with pytest.raises(ValueError):
            mandel.mandel_render_ex(*cfg.args(), "fp64", "block", 1, out_host=b)
        with pytest.raises(ValueError):
            mandel.mandel_render_ex(*cfg.args(), "fp64", "block", 1, out_dev0=b)
        with pytest.raises(ValueError):
            mandel.mandel_render_rank(*cfg.args(), "fp64", "block", 0, 1, b)
    ro = np.zeros(cfg.pixels, np.uint32)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        mandel.mandel_render(*cfg.args(), "fp64", "block", 1, ro)
    # a correctly sized buffer passes validation (then ENODEV without a device)
    if mandel.mandel_device_count() == 0:
        with pytest.raises(mandel.MandelError) as e:
            mandel.mandel_render(*cfg.args(), "fp64", "block", 1, np.zeros((cfg.H, cfg.W), np.uint32))
        assert e.value.code == mandel.MANDEL_ENODEV


def test_binding_structs_match_the_header(mandel, tmp_path):
    """The ctypes mirrors of mandel_options / mandel_stats have the header's layout: a C
    program compiled against include/mandel.h prints every field's offset and the struct
    sizes (a field added to one side only would shift everything after it silently)."""
    import ctypes
    import os
    import re
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    hdr = open(os.path.join(root, "include", "mandel.h")).read()
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "mandel.h"', 'int main(void) {']
    want = {}
    for cname, ctype in (("mandel_options", mandel.mandel_options), ("mandel_stats", mandel.mandel_stats)):
        end = re.search(r"\}\s*" + cname + r"\s*;", hdr).start()
        body = hdr[hdr.rindex("{", 0, end) + 1:end]
        body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
        fields = [re.sub(r"\[.*", "", f.strip().split()[-1]) for f in body.split(";") if f.strip()]
        assert fields == [f[0] for f in ctype._fields_], f"{cname}: field names/order differ from the header"
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        want[cname] = ctypes.sizeof(ctype)
        for f in fields:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
            want[f"{cname}.{f}"] = getattr(ctype, f).offset
    lines += ["return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(root, "include"), "-o", str(exe), str(src)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    got = {k: int(v) for k, v in (l.split() for l in out.splitlines())}
    assert got == want
