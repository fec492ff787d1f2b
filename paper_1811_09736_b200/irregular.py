"""Irregular (offset-array) segmented reduction and scan -- the extension
SURVEY.md section 8(f)4 lists after the reference's regular path.

The paper elides irregular segments ("implemented in terms of regular
segmented reduction") and the reference package has no entry
point for them, so this module defines one in the reference's style: the
same value / engine / error conventions as ``segmented_reduce`` and
``segmented_scan`` (reduce.py:379-446, scan.py:316-388), with segments given
as CSR offsets (segment k = values[offsets[k]:offsets[k+1]], empty segments
allowed).

B200 path: ``tc_irreg_reduce`` / ``tc_irreg_scan`` (include/tc_collectives.h)
-- the regular kernels' TMA -> tcgen05.mma -> TMEM tile pipeline with the
full in-row prefix X.U as the tile product; each row's segment starts come
from ``offsets`` (counted per tile in shared memory), and a segment's value
is the difference of two in-row prefixes plus the same (value, has-start)
carry chain across rows, tiles and CTAs as the regular GENERAL mode.

Numerics: fp32 tensor-core accumulation within a row, fp32 / fp64 carries,
one rounding to the output dtype.  Exact-integer inputs are bit-exact; for
general data a segment sum carries the rounding of (at most two) in-row
fp32 prefixes, |error| <= 2^-22 * (sum of |x| over the rows the segment
touches), stated and tested in tests/test_irregular_gpu.py.
"""

from __future__ import annotations

import numpy as np

from . import _dispatch as _d
from .engine import TileEngine
from .errors import BadConfigError, BadLengthError


def _host_offsets(offsets, n: int):
    """Validate offsets; returns (offsets as numpy int64 or torch tensor, nseg)."""
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(offsets, torch.Tensor):
        if offsets.dim() != 1 or offsets.numel() < 2:
            raise BadLengthError("offsets must be a flat vector of nseg + 1 >= 2 entries")
        if not offsets.is_cuda:
            _check_host_offsets(offsets.to(torch.int64).numpy(), n)
        return offsets, offsets.numel() - 1
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    if off.ndim != 1 or off.size < 2:
        raise BadLengthError("offsets must be a flat vector of nseg + 1 >= 2 entries")
    _check_host_offsets(off, n)
    return off, off.size - 1


def _check_host_offsets(off: np.ndarray, n: int) -> None:
    if off[0] != 0 or off[-1] != n:
        raise BadConfigError(
            f"offsets must start at 0 and end at len(values) = {n}, got {off[0]} .. {off[-1]}")
    if np.any(off[1:] < off[:-1]):
        raise BadConfigError("offsets must be non-decreasing")


def _device_offsets(off, dev_values):
    import torch

    if isinstance(off, torch.Tensor):
        return off.to(device=dev_values.device, dtype=torch.int64)
    return torch.from_numpy(off).to(dev_values.device)


def irregular_segmented_reduce(values, offsets, engine: TileEngine | None = None):
    """One sum per segment values[offsets[k]:offsets[k+1]] (0 for an empty
    segment), in ``engine.acc_dtype``; numpy in -> numpy out, torch CUDA in ->
    torch CUDA out (stream-ordered)."""
    from . import _device

    engine = engine or TileEngine()
    x, kind = _d.flat_half(values)
    n = _d.size_of(x)
    if n == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    off, nseg = _host_offsets(offsets, n)
    dev = _d.to_device(x, kind)
    doff = _device_offsets(off, dev)
    out = _device.irreg_reduce(dev, doff, _d.torch_dtype(engine.acc_dtype),
                               validate=(kind == "torch_cuda"))
    engine._account(n, nseg, scan=False)
    return _d.from_device(out, kind, engine.acc_dtype)


def irregular_segmented_scan(values, offsets, engine: TileEngine | None = None,
                             inclusive: bool = True):
    """Prefix sums restarted at every segment start; ``inclusive=False``
    gives the exclusive form (0 at each segment start, like the reference's
    shift-right, scan.py:332-341)."""
    from . import _device

    engine = engine or TileEngine()
    x, kind = _d.flat_half(values)
    n = _d.size_of(x)
    if n == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    off, _ = _host_offsets(offsets, n)
    dev = _d.to_device(x, kind)
    doff = _device_offsets(off, dev)
    out = _device.irreg_scan(dev, doff, _d.torch_dtype(engine.acc_dtype), exclusive=not inclusive,
                             validate=(kind == "torch_cuda"))
    engine._account(n, n, scan=True)
    return _d.from_device(out, kind, engine.acc_dtype)
