"""Device-side entry points: torch CUDA tensors in, torch CUDA tensors out.

Thin wrappers over the C ABI (include/tc_collectives.h): they own output
and workspace allocation on the caller's current CUDA stream and map status
codes onto the reference's exceptions (BadLengthError / BadConfigError,
pkg/src/halftile/errors.py:29-38).  Everything is stream-ordered; nothing
here synchronises.
"""

from __future__ import annotations

import torch

from . import _lib
from .errors import STATUS_ERRORS, BadConfigError, BadLengthError

_DT = {torch.float16: _lib.TC_F16, torch.float32: _lib.TC_F32, torch.float64: _lib.TC_F64}

_ws_cache: dict = {}


def _check(rc: int) -> None:
    if rc == _lib.TC_OK:
        return
    msg = _lib.last_error()
    exc = STATUS_ERRORS.get(rc)
    if exc is not None:
        raise exc(msg)
    raise RuntimeError(f"tc_collectives: {_lib.status_string(rc)}: {msg}")


def _stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def workspace(op: int, n: int, seg: int, device: torch.device) -> torch.Tensor:
    """Zero-initialised workspace cached per (device, stream); grows on demand.

    The kernels leave a workspace reusable (ticket reset, epoch-tagged
    look-back flags), so one allocation serves every later call on that
    stream."""
    need = int(_lib.lib.tc_workspace_bytes(op, n, seg))
    key = (device.index, _stream_ptr(device))
    ws = _ws_cache.get(key)
    if ws is None or ws.numel() < need:
        size = max(need, 1 << 20)
        if ws is not None:
            size = max(size, 2 * ws.numel())
        ws = torch.zeros(size, dtype=torch.uint8, device=device)
        _ws_cache[key] = ws
    return ws


_IN = {torch.float16: _lib.TC_F16, torch.bfloat16: _lib.TC_BF16}


def _prep(x: torch.Tensor) -> torch.Tensor:
    """fp16 (the reference's input type) or bf16 (extension) stay as they
    are; anything else is converted to fp16 like reduce._as_flat_half.

    A non-contiguous view, or one whose data pointer is not 16-byte aligned
    (TMA rows need it, e.g. ``x[3:]``), costs ONE extra device copy here;
    aligned contiguous fp16 / bf16 tensors are used in place."""
    if not x.is_cuda:
        raise ValueError("device entry points take CUDA tensors")
    if x.dim() != 1:
        raise BadLengthError("collectives operate on flat vectors")
    if x.dtype not in _IN:
        x = x.to(torch.float16)
    if not x.is_contiguous() or x.data_ptr() % 16:
        x = x.contiguous().clone()
    return x


def seg_reduce(x: torch.Tensor, seg: int, out_dtype=torch.float16, out=None) -> torch.Tensor:
    """ceil(n/seg) segment sums of a CUDA fp16 vector (tc_seg_reduce)."""
    x = _prep(x)
    n = x.numel()
    if n == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    if seg < 1:
        raise BadLengthError(f"segment size must be positive, got {seg}")
    nseg = -(-n // seg)
    if out is None:
        out = torch.empty(nseg, dtype=out_dtype, device=x.device)
    ws = workspace(_lib.TC_OP_REDUCE, n, seg, x.device)
    _check(_lib.lib.tc_seg_reduce_ex(x.data_ptr(), _IN[x.dtype], n, seg, out.data_ptr(),
                                     _DT[out.dtype], ws.data_ptr(), ws.numel(),
                                     _stream_ptr(x.device)))
    return out


def full_reduce(x: torch.Tensor, out_dtype=torch.float16, out=None) -> torch.Tensor:
    """Sum of all n elements as a 1-element tensor (tc_full_reduce)."""
    x = _prep(x)
    n = x.numel()
    if n == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    if out is None:
        out = torch.empty(1, dtype=out_dtype, device=x.device)
    ws = workspace(_lib.TC_OP_REDUCE, n, n, x.device)
    _check(_lib.lib.tc_seg_reduce_ex(x.data_ptr(), _IN[x.dtype], n, n, out.data_ptr(),
                                     _DT[out.dtype], ws.data_ptr(), ws.numel(),
                                     _stream_ptr(x.device)))
    return out


def seg_scan(x: torch.Tensor, seg: int, out_dtype=torch.float16, exclusive=False,
             carry_in: torch.Tensor | None = None, total_out: torch.Tensor | None = None,
             out=None) -> torch.Tensor:
    """Segmented inclusive/exclusive prefix sums (tc_seg_scan).

    ``carry_in`` / ``total_out`` are optional 1-element float64 CUDA tensors
    (cross-GPU carry of a sharded full scan)."""
    x = _prep(x)
    n = x.numel()
    if n == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    if seg < 1:
        raise BadLengthError(f"segment size must be positive, got {seg}")
    if out is None:
        out = torch.empty(n, dtype=out_dtype, device=x.device)
    ws = workspace(_lib.TC_OP_SCAN, n, seg, x.device)
    cin = carry_in.data_ptr() if carry_in is not None else None
    tout = total_out.data_ptr() if total_out is not None else None
    _check(_lib.lib.tc_seg_scan_ex(x.data_ptr(), _IN[x.dtype], n, seg, out.data_ptr(),
                                   _DT[out.dtype], 1 if exclusive else 0, cin, tout,
                                   ws.data_ptr(), ws.numel(), _stream_ptr(x.device)))
    return out


def full_scan(x: torch.Tensor, out_dtype=torch.float16, exclusive=False,
              carry_in: torch.Tensor | None = None, total_out: torch.Tensor | None = None,
              out=None) -> torch.Tensor:
    """One-segment scan of the whole vector (tc_full_scan)."""
    x = _prep(x)
    return seg_scan(x, max(x.numel(), 1), out_dtype, exclusive, carry_in, total_out, out)


def _prep_offsets(offsets: torch.Tensor, n: int, device: torch.device, validate: bool) -> torch.Tensor:
    """int64 CUDA offsets (nseg + 1 entries, offsets[0] = 0, offsets[-1] = n,
    non-decreasing).  ``validate`` checks that on the device (one host sync)."""
    if not isinstance(offsets, torch.Tensor):
        raise ValueError("device entry points take CUDA tensors")
    if offsets.dim() != 1 or offsets.numel() < 2:
        raise BadLengthError("offsets must be a flat vector of nseg + 1 >= 2 entries")
    offsets = offsets.to(device=device, dtype=torch.int64)
    if not offsets.is_contiguous():
        offsets = offsets.contiguous()
    if validate:
        ok = ((offsets[0] == 0) & (offsets[-1] == n)
              & (offsets[1:] >= offsets[:-1]).all())
        if not bool(ok):
            raise BadConfigError(
                "offsets must be non-decreasing with offsets[0] = 0 and offsets[-1] = len(values)")
    return offsets


def irreg_reduce(x: torch.Tensor, offsets: torch.Tensor, out_dtype=torch.float16, out=None,
                 validate: bool = True) -> torch.Tensor:
    """Sums of the irregular segments x[offsets[k]:offsets[k+1]] (tc_irreg_reduce)."""
    x = _prep(x)
    n = x.numel()
    if n == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    offsets = _prep_offsets(offsets, n, x.device, validate)
    nseg = offsets.numel() - 1
    if out is None:
        out = torch.empty(nseg, dtype=out_dtype, device=x.device)
    ws = workspace(_lib.TC_OP_REDUCE, n, n, x.device)
    _check(_lib.lib.tc_irreg_reduce(x.data_ptr(), _IN[x.dtype], n, offsets.data_ptr(), nseg,
                                    out.data_ptr(), _DT[out.dtype], ws.data_ptr(), ws.numel(),
                                    _stream_ptr(x.device)))
    return out


def irreg_scan(x: torch.Tensor, offsets: torch.Tensor, out_dtype=torch.float16, exclusive=False,
               out=None, validate: bool = True) -> torch.Tensor:
    """Prefix sums restarted at every offsets[k] (tc_irreg_scan)."""
    x = _prep(x)
    n = x.numel()
    if n == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    offsets = _prep_offsets(offsets, n, x.device, validate)
    nseg = offsets.numel() - 1
    if out is None:
        out = torch.empty(n, dtype=out_dtype, device=x.device)
    ws = workspace(_lib.TC_OP_SCAN, n, n, x.device)
    _check(_lib.lib.tc_irreg_scan(x.data_ptr(), _IN[x.dtype], n, offsets.data_ptr(), nseg,
                                  out.data_ptr(), _DT[out.dtype], 1 if exclusive else 0,
                                  ws.data_ptr(), ws.numel(), _stream_ptr(x.device)))
    return out


def bn_stats(x: torch.Tensor, out_dtype=torch.float32):
    """Per-channel (mean, biased variance) of an NCHW-contiguous CUDA tensor
    x of shape (N, C, *spatial), fp16 or bf16 (tc_bn_stats)."""
    if not x.is_cuda:
        raise ValueError("device entry points take CUDA tensors")
    if x.dim() < 2:
        raise BadLengthError("batch-norm statistics need an (N, C, ...) tensor")
    N, C = int(x.shape[0]), int(x.shape[1])
    HW = 1
    for d in x.shape[2:]:
        HW *= int(d)
    if N * C * HW == 0:
        raise BadLengthError("batch-norm statistics of an empty tensor")
    if x.dtype not in _IN:
        raise TypeError(f"batch-norm statistics take fp16 or bf16 input, got {x.dtype} "
                        "(convert explicitly; fp32 activations above 65504 overflow fp16)")
    if not x.is_contiguous() or x.data_ptr() % 16:
        x = x.contiguous().clone()
    mean = torch.empty(C, dtype=out_dtype, device=x.device)
    var = torch.empty(C, dtype=out_dtype, device=x.device)
    ws = workspace(_lib.TC_OP_BN_STATS, N * C * HW, HW, x.device)
    _check(_lib.lib.tc_bn_stats(x.data_ptr(), _IN[x.dtype], N, C, HW, mean.data_ptr(),
                                var.data_ptr(), _DT[out_dtype], ws.data_ptr(), ws.numel(),
                                _stream_ptr(x.device)))
    return mean, var


MODES = ("LOCAL", "ROWS", "TILES", "GENERAL", "CHUNK", "IRREG", "GSCR", "ROWSEG", "SPLIT", "SPLITM")


def plan_info(op: str, n: int, seg: int, out_dtype=torch.float16, carry_in: bool = False,
              total_out: bool = False) -> tuple[str, int]:
    """(kernel mode, MMA row length in elements) a seg_reduce / seg_scan
    call would use (tc_plan_info; host-only, no device work)."""
    import ctypes

    mode = ctypes.c_int(0)
    row = ctypes.c_int64(0)
    _check(_lib.lib.tc_plan_info(_lib.TC_OP_REDUCE if op == "reduce" else _lib.TC_OP_SCAN, n, seg,
                                 _DT[out_dtype], int(carry_in), int(total_out),
                                 ctypes.byref(mode), ctypes.byref(row)))
    return MODES[mode.value], int(row.value)
