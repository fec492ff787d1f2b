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
# A pageable ``torch.from_numpy(x).to(dev)`` runs at a fraction of PCIe speed
# (the driver stages through its own small pinned buffer, synchronously).
# The stager instead streams the bytes through a ring of pinned chunks: host
# threads copy chunk c into pinned memory (numpy's copy releases the GIL)
# while the copy engine moves chunk c-1 to the device on a side stream, so
# the whole transfer runs at the slower of PCIe and the parallel host copy.
# Device -> host is the mirror image.  Stream order: the compute stream
# waits on the copy stream's last event (no host sync on the way in).

_CHUNK = 32 << 20          # bytes per pinned chunk
_RING = 4                  # pinned chunks in flight
_SMALL = 4 << 20           # below this, one direct copy is cheaper
_stagers: dict = {}


def _host_threads() -> int:
    import os

    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        n = os.cpu_count() or 1
    return max(1, min(8, n))


class _Stager:
    """Pinned ring buffer + copy stream + host thread pool, one per device."""

    def __init__(self, device):
        import concurrent.futures as cf

        import torch

        self.device = device
        self.ring = [torch.empty(_CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(_RING)]
        self.ring_np = [b.numpy() for b in self.ring]
        self.busy = [None] * _RING  # event of the last DMA that used the chunk
        self.stream = torch.cuda.Stream(device)
        self.threads = _host_threads()
        self.pool = cf.ThreadPoolExecutor(self.threads) if self.threads > 1 else None

    def _par_copy(self, dst: np.ndarray, src: np.ndarray) -> None:
        """dst[:] = src (flat uint8 views) with the host thread pool."""
        nb = src.size
        if self.pool is None or nb < (4 << 20):
            np.copyto(dst, src)
            return
        k = self.threads
        cuts = [nb * t // k for t in range(k + 1)]
        futs = [self.pool.submit(np.copyto, dst[cuts[t]:cuts[t + 1]], src[cuts[t]:cuts[t + 1]])
                for t in range(k)]
        for f in futs:
            f.result()

    def _slot(self, i: int):
        ev = self.busy[i]
        if ev is not None:
            ev.synchronize()  # the chunk's previous DMA has finished reading / writing it
        return self.ring[i], self.ring_np[i]

    def h2d(self, src: np.ndarray, dst) -> None:
        """Copy the bytes of a contiguous host array into the device tensor
        ``dst`` (same byte size); ordered before later work on the current
        stream."""
        import torch

        sb = src.reshape(-1).view(np.uint8)
        db = dst.view(-1).view(torch.uint8)
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)  # dst may still be in use by earlier work
        for c, lo in enumerate(range(0, sb.size, _CHUNK)):
            hi = min(lo + _CHUNK, sb.size)
            i = c % _RING
            pin, pin_np = self._slot(i)
            self._par_copy(pin_np[: hi - lo], sb[lo:hi])
            with torch.cuda.stream(self.stream):
                db[lo:hi].copy_(pin[: hi - lo], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.stream)
            self.busy[i] = ev
        cur.wait_stream(self.stream)

    def d2h(self, src, dst: np.ndarray) -> None:
        """Copy a device tensor's bytes into a contiguous host array
        (synchronous: returns when ``dst`` holds the data)."""
        import torch

        sb = src.reshape(-1).view(torch.uint8)
        db = dst.reshape(-1).view(np.uint8)
        cur = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(cur)  # the producing kernels
        pending = []  # (slot, event, lo, hi) issued but not yet drained
        for c, lo in enumerate(range(0, sb.numel(), _CHUNK)):
            hi = min(lo + _CHUNK, sb.numel())
            i = c % _RING
            if len(pending) == _RING:
                self._drain(pending.pop(0), db)
            pin = self.ring[i]
            with torch.cuda.stream(self.stream):
                pin[: hi - lo].copy_(sb[lo:hi], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.stream)
            self.busy[i] = ev
            pending.append((i, ev, lo, hi))
        for p in pending:
            self._drain(p, db)

    def _drain(self, p, db: np.ndarray) -> None:
        i, ev, lo, hi = p
        ev.synchronize()
        self._par_copy(db[lo:hi], self.ring_np[i][: hi - lo])


def _stager(device):
    key = device.index
    st = _stagers.get(key)
    if st is None:
        st = _stagers[key] = _Stager(device)
    return st


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
    out = torch.empty(x.size, dtype=torch.float16, device=dev)
    _stager(dev).h2d(np.ascontiguousarray(x), out)
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
    _stager(t.device).d2h(t, host)
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
