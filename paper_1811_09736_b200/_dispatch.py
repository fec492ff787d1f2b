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
        return t.to(dev, non_blocking=t.is_pinned())
    return torch.from_numpy(x).to(dev)


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
    return t.cpu().numpy().astype(np_dtype, copy=False)


def torch_dtype(np_dtype):
    import torch

    return torch.float32 if np.dtype(np_dtype) == np.float32 else torch.float16
