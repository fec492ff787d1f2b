"""Reference-side binding: what a ``halftile`` maintainer adds to route the
package's hot path through the B200 C ABI (include/tc_collectives.h).

Torch-free on purpose: the reference depends only on numpy
(pkg/pyproject.toml:10-13), so this stub drives the CUDA runtime directly
through ctypes (cudaMalloc / cudaMemcpy / cudaMemset / cudaFree) and calls
``tc_seg_reduce`` / ``tc_seg_scan``.  Drop it in as
``halftile/_b200.py`` and dispatch from the two drivers:

    # halftile/reduce.py, top of segmented_reduce (reduce.py:379-446)
    from . import _b200
    if _b200.available():
        <keep the reference's variant / length validation, reduce.py:398-418>
        return _b200.seg_reduce(values, seg_size, engine.acc_dtype)

    # halftile/scan.py, top of segmented_scan (scan.py:316-388)
    if _b200.available():
        <keep the reference's validation, scan.py:326-348>
        return _b200.seg_scan(values, seg_size, engine.acc_dtype, inclusive)

Status codes map onto halftile.errors exactly like
paper_1811_09736_b200/_device.py does.  tests/test_integration_gpu.py runs
this module on the B200 against the oracle.
"""

from __future__ import annotations

import ctypes
import ctypes.util
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB = os.environ.get("TC_COLLECTIVES_LIB",
                     str(_HERE.parent / "paper_1811_09736_b200" / "_tc_collectives.so"))

TC_OK, TC_BAD_LENGTH, TC_BAD_CONFIG = 0, 1, 2
TC_F16, TC_F32 = 0, 1
TC_OP_REDUCE, TC_OP_SCAN = 0, 1
_H2D, _D2H = 1, 2


class B200Error(RuntimeError):
    pass


def _load():
    tc = ctypes.CDLL(LIB)
    vp, i64, sz, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_size_t, ctypes.c_int
    tc.tc_workspace_bytes.restype = sz
    tc.tc_workspace_bytes.argtypes = [ci, i64, i64]
    tc.tc_seg_reduce.restype = ci
    tc.tc_seg_reduce.argtypes = [vp, i64, i64, vp, ci, vp, sz, vp]
    tc.tc_seg_scan.restype = ci
    tc.tc_seg_scan.argtypes = [vp, i64, i64, vp, ci, ci, vp, vp, vp, sz, vp]
    tc.tc_irreg_reduce.restype = ci
    tc.tc_irreg_reduce.argtypes = [vp, ci, i64, vp, i64, vp, ci, vp, sz, vp]
    tc.tc_h2d_pageable.restype = ci
    tc.tc_h2d_pageable.argtypes = [vp, vp, sz, vp]
    tc.tc_d2h_pageable.restype = ci
    tc.tc_d2h_pageable.argtypes = [vp, vp, sz, vp]
    tc.tc_last_error.restype = ctypes.c_char_p
    name = ctypes.util.find_library("cudart") or "libcudart.so"
    try:
        rt = ctypes.CDLL(name)
    except OSError:
        # the CUDA runtime the extension itself links against is already loaded
        rt = tc
    rt.cudaMalloc.argtypes = [ctypes.POINTER(vp), sz]
    rt.cudaMemcpy.argtypes = [vp, vp, sz, ci]
    rt.cudaMemset.argtypes = [vp, ci, sz]
    rt.cudaFree.argtypes = [vp]
    rt.cudaDeviceSynchronize.argtypes = []
    return tc, rt


_tc = _rt = None


def available() -> bool:
    global _tc, _rt
    if _tc is None:
        try:
            _tc, _rt = _load()
            n = ctypes.c_int(0)
            _rt.cudaGetDeviceCount.argtypes = [ctypes.POINTER(ctypes.c_int)]
            if _rt.cudaGetDeviceCount(ctypes.byref(n)) != 0 or n.value == 0:
                return False
        except OSError:
            return False
    return True


def _cuda(rc):
    if rc != 0:
        raise B200Error(f"CUDA runtime error {rc}")


class _Dev:
    """A cudaMalloc'd buffer freed on exit."""

    def __init__(self, nbytes):
        self.p = ctypes.c_void_p()
        _cuda(_rt.cudaMalloc(ctypes.byref(self.p), max(int(nbytes), 256)))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        _rt.cudaFree(self.p)


def _check(rc):
    if rc == TC_OK:
        return
    from_halftile = None
    try:  # inside the reference package these are halftile.errors.*
        from halftile.errors import BadConfigError, BadLengthError
        from_halftile = {TC_BAD_LENGTH: BadLengthError, TC_BAD_CONFIG: BadConfigError}
    except ImportError:
        pass
    msg = (_tc.tc_last_error() or b"").decode()
    if from_halftile and rc in from_halftile:
        raise from_halftile[rc](msg)
    raise B200Error(f"tc status {rc}: {msg}")


def _run(values, seg_size, acc_dtype, op, inclusive=True):
    if not available():
        raise B200Error("no CUDA device / library")
    x = np.ascontiguousarray(values, dtype=np.float16)  # reduce.py:69-73 coercion
    n = x.size
    out_dt = np.dtype(acc_dtype)
    code = TC_F32 if out_dt == np.float32 else TC_F16
    n_out = -(-n // seg_size) if op == TC_OP_REDUCE else n
    out = np.empty(n_out, dtype=out_dt)
    wsb = _tc.tc_workspace_bytes(op, n, seg_size)
    with _Dev(x.nbytes) as dx, _Dev(out.nbytes) as do, _Dev(wsb) as dw:
        _cuda(_rt.cudaMemset(dw.p, 0, wsb))
        # the numpy buffers move through the library's pinned-ring stager
        # (a plain pageable cudaMemcpy runs at ~11 GB/s); both are ordered on
        # the legacy default stream, like the kernel launch
        _check(_tc.tc_h2d_pageable(dx.p, x.ctypes.data, x.nbytes, None))
        if op == TC_OP_REDUCE:
            _check(_tc.tc_seg_reduce(dx.p, n, seg_size, do.p, code, dw.p, wsb, None))
        else:
            _check(_tc.tc_seg_scan(dx.p, n, seg_size, do.p, code, 0 if inclusive else 1,
                                   None, None, dw.p, wsb, None))
        _check(_tc.tc_d2h_pageable(out.ctypes.data, do.p, out.nbytes, None))  # returns with the data
    return out


def seg_reduce(values, seg_size, acc_dtype=np.float16):
    """ceil(n/s) segment sums (halftile.segmented_reduce semantics)."""
    return _run(values, seg_size, acc_dtype, TC_OP_REDUCE)


def seg_scan(values, seg_size, acc_dtype=np.float16, inclusive=True):
    """n segmented prefix sums (halftile.segmented_scan semantics)."""
    return _run(values, seg_size, acc_dtype, TC_OP_SCAN, inclusive)


def irregular_reduce(values, offsets, acc_dtype=np.float32):
    """Sums of values[offsets[k]:offsets[k+1]] (tc_irreg_reduce; extension)."""
    if not available():
        raise B200Error("no CUDA device / library")
    x = np.ascontiguousarray(values, dtype=np.float16)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    n, nseg = x.size, off.size - 1
    if nseg < 1 or off[0] != 0 or off[-1] != n or np.any(np.diff(off) < 0):
        raise B200Error("offsets must be non-decreasing from 0 to len(values)")
    out_dt = np.dtype(acc_dtype)
    out = np.empty(nseg, dtype=out_dt)
    code = TC_F32 if out_dt == np.float32 else TC_F16
    wsb = _tc.tc_workspace_bytes(TC_OP_REDUCE, n, n)
    with _Dev(x.nbytes) as dx, _Dev(off.nbytes) as dof, _Dev(out.nbytes) as do, _Dev(wsb) as dw:
        _cuda(_rt.cudaMemset(dw.p, 0, wsb))
        _cuda(_rt.cudaMemcpy(dx.p, x.ctypes.data, x.nbytes, _H2D))
        _cuda(_rt.cudaMemcpy(dof.p, off.ctypes.data, off.nbytes, _H2D))
        _check(_tc.tc_irreg_reduce(dx.p, TC_F16, n, dof.p, nseg, do.p, code, dw.p, wsb, None))
        _cuda(_rt.cudaMemcpy(out.ctypes.data, do.p, out.nbytes, _D2H))
    return out
