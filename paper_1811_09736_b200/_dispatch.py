"""Host <-> device plumbing shared by the reduce/scan front ends.

Inputs may be numpy arrays (reference behaviour: result is a numpy array),
torch CPU tensors (pinned ones are copied asynchronously; result is a CPU
tensor) or torch CUDA tensors (no copy, stream-ordered, result stays on the
device).  Validation happens before any device work so argument errors
raise the reference's exceptions even on a machine without a GPU; there is
no CPU compute path -- without CUDA the call fails loudly.
"""

from __future__ import annotations

import numpy as np

from .errors import BadLengthError

HALF = np.float16


def flat_half(values):
    """Coerce like reduce._as_flat_half (reduce.py:69-73).

    Returns ``(host_or_device_array, kind)`` with kind in
    {"numpy", "torch_cpu", "torch_cuda"}; raises BadLengthError for
    non-flat input."""
    try:
        import torch
    except ImportError:  # pragma: no cover - torch is a hard dependency at run time
        torch = None
    if torch is not None and isinstance(values, torch.Tensor):
        if values.dim() != 1:
            raise BadLengthError("collectives operate on flat vectors")
        kind = "torch_cuda" if values.is_cuda else "torch_cpu"
        return values, kind
    arr = np.ascontiguousarray(values, dtype=HALF)
    if arr.ndim != 1:
        raise BadLengthError("collectives operate on flat vectors")
    return arr, "numpy"


def size_of(x) -> int:
    return int(x.numel()) if hasattr(x, "numel") else int(x.size)


# ---------------------------------------------------------------------------
# Host <-> device copies for host inputs (numpy arrays, torch CPU tensors).
#
# A pageable ``torch.from_numpy(x).to(dev)`` runs at ~11 GB/s (the driver
# stages it through its own small pinned buffer, synchronously).  Large
# host buffers go through the library's native stager instead
# (tc_h2d_pageable / tc_d2h_pageable, csrc/host_stager.cpp): a pinned ring
# filled by a pool of host threads with non-temporal stores, overlapped with
# the copy engine.  Stream order: the H2D is enqueued on the current stream
# (no host sync on the way in); the D2H returns when the array holds the data.

_SMALL = 4 << 20           # below this, one direct copy is cheaper


def _stream_handle(device):
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def _h2d(src: np.ndarray, dst) -> None:
    from . import _lib

    rc = _lib.lib.tc_h2d_pageable(dst.data_ptr(), src.ctypes.data, src.nbytes,
                                  _stream_handle(dst.device))
    if rc != _lib.TC_OK:
        raise RuntimeError(f"host -> device copy failed: {_lib.status_string(rc)}")


def _d2h(src, dst: np.ndarray) -> None:
    from . import _lib

    rc = _lib.lib.tc_d2h_pageable(dst.ctypes.data, src.data_ptr(), dst.nbytes,
                                  _stream_handle(src.device))
    if rc != _lib.TC_OK:
        raise RuntimeError(f"device -> host copy failed: {_lib.status_string(rc)}")


def to_device(x, kind):
    import torch

    if kind == "torch_cuda":
        t = x
        if t.dtype != torch.float16:
            t = t.to(torch.float16)
        return t.contiguous()
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1811_09736_b200 runs on an sm_100 GPU only (no CPU fallback); "
            "no CUDA device is visible")
    dev = torch.device("cuda", torch.cuda.current_device())
    if kind == "torch_cpu":
        t = x if x.dtype == torch.float16 else x.to(torch.float16)
        t = t.contiguous()
        if t.is_pinned() or t.numel() * 2 < _SMALL:
            return t.to(dev, non_blocking=t.is_pinned())
        x = t.numpy()
    elif x.nbytes < _SMALL:
        return torch.from_numpy(x).to(dev)
    x = np.ascontiguousarray(x)
    out = torch.empty(x.size, dtype=torch.float16, device=dev)
    _h2d(x, out)
    return out


def from_device(t, kind, np_dtype):
    """Return results in the caller's domain (numpy / CPU tensor / CUDA tensor)."""
    import torch

    if kind == "torch_cuda":
        return t
    if kind == "torch_cpu":
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t, non_blocking=True)
        torch.cuda.current_stream(t.device).synchronize()
        return out
    t = t.contiguous()
    if t.numel() * t.element_size() < _SMALL:
        return t.cpu().numpy().astype(np_dtype, copy=False)
    host = np.empty(tuple(t.shape), dtype=_NP_OF[t.dtype])
    _d2h(t, host)
    return host.astype(np_dtype, copy=False)


def _np_of():
    import torch

    return {torch.float16: np.float16, torch.float32: np.float32, torch.float64: np.float64}


class _NpOf(dict):
    def __missing__(self, k):
        self.update(_np_of())
        return dict.__getitem__(self, k)


_NP_OF = _NpOf()


def torch_dtype(np_dtype):
    import torch

    return torch.float32 if np.dtype(np_dtype) == np.float32 else torch.float16
