"""Segmented inclusive/exclusive scan on B200 tensor cores -- drop-in for
pkg/src/halftile/scan.py.

The reference builds each scan from three tile identities (A.U row scans,
L.A column carries, an all-ones broadcast; scan.py:1-31).  The sm_100a
kernel behind ``tc_seg_scan`` (include/tc_collectives.h) keeps the A.U
product on the tensor core (block-diagonal upper-triangular U in shared
memory, fp32 accumulators in TMEM) and carries across rows, tiles and CTAs
in fp32/fp64 registers (warp shuffles + shared memory + a decoupled
look-back for huge segments), so the fp16 narrowing of the L.A carry
(engine.py:450) disappears.  Exclusive outputs are the reference's
shift-right-inject-zero (scan.py:332-341), computed in the same pass.
"""

from __future__ import annotations

import numpy as np

from . import _dispatch as _d
from .engine import TileEngine
from .errors import BadConfigError, BadLengthError
from .reduce import BlockConfig, _as_flat_half, clamp_block_config  # noqa: F401

GRID_SCAN_PASSES = 3  # reference constant (scan.py:43); B200 does it in ONE launch

SCAN_VARIANTS = (
    "warp16",
    "warp256",
    "strided16n",
    "warp256n",
    "block256n",
    "grid",
)


def _device_scan(x, kind, seg: int, engine: TileEngine, inclusive: bool = True,
                 carry: float | None = None):
    from . import _device

    import torch

    n = _d.size_of(x)
    dev = _d.to_device(x, kind)
    cin = None
    if carry is not None:
        cin = torch.tensor([float(carry)], dtype=torch.float64, device=dev.device)
    out = _device.seg_scan(dev, seg, _d.torch_dtype(engine.acc_dtype), exclusive=not inclusive,
                           carry_in=cin)
    engine._account(n, n, scan=True)
    return _d.from_device(out, kind, engine.acc_dtype)


# -- warp level ----------------------------------------------------------------


def scan_16(values, engine: TileEngine):
    """Inclusive prefix sums of 16 consecutive segments of 16 (scan.py:58-71)."""
    x, kind = _as_flat_half(values)
    if _d.size_of(x) != 256:
        raise BadLengthError(f"scan_16 takes exactly 256 elements, got {_d.size_of(x)}")
    return _device_scan(x, kind, 16, engine)


def scan_256(values, engine: TileEngine):
    """Inclusive scan of one 256-element segment (scan.py:94-99)."""
    return scan_256n(values, 1, engine)


def scan_256n(values, n: int, engine: TileEngine):
    """Inclusive scan of one 256n segment (scan.py:102-119)."""
    x, kind = _as_flat_half(values)
    if n < 1 or _d.size_of(x) != 256 * n:
        raise BadLengthError(f"need exactly 256*{n} elements, got {_d.size_of(x)}")
    return _device_scan(x, kind, 256 * n, engine)


def scan_16n(values, seg_size: int, engine: TileEngine):
    """Inclusive scans of 16 segments of 16n per group (scan.py:122-152)."""
    x, kind = _as_flat_half(values)
    if seg_size < 16 or seg_size % 16:
        raise BadLengthError(f"segment size must be a positive multiple of 16, got {seg_size}")
    group = 256 * (seg_size // 16)
    size = _d.size_of(x)
    if size == 0 or size % group:
        raise BadLengthError(
            f"input length {size} is not a multiple of the {group}-element warp group")
    return _device_scan(x, kind, seg_size, engine)


def last_column_scan_16(frag, engine: TileEngine, carry: float = 0.0):
    """Exclusive scan of a tile's last column seeded with ``carry``
    (scan.py:155-172).  ``frag`` is a 16x16 tile: a reference ``Fragment``
    (its ``matrix``), or any array-like.  The column is narrowed to fp16 and
    the seed rounded to the accumulator dtype exactly as the reference does
    (scan.py:163-168, engine.py:313-324)."""
    tile = np.asarray(getattr(frag, "matrix", frag), dtype=np.float64)
    if tile.shape != (16, 16):
        raise BadLengthError(f"last_column_scan_16 needs a 16x16 tile, got {tile.shape}")
    col = tile[:, -1].astype(np.float16)
    seed = float(engine.acc_dtype.type(carry))
    return _device_scan(col, "numpy", 16, engine, inclusive=False, carry=seed)


# -- block level ---------------------------------------------------------------


def block_scan_256n(values, cfg: BlockConfig, engine: TileEngine, workers: int = 1,
                    reverse: bool = False, debug_capture: dict | None = None):
    """Inclusive scan of one 256n segment (scan.py:178-243)."""
    x, kind = _as_flat_half(values)
    size = _d.size_of(x)
    if size % 256:
        raise BadLengthError(f"segment length {size} is not a multiple of 256")
    n = size // 256
    if n % cfg.wpb:
        raise BadConfigError(f"{n} tiles do not divide across {cfg.wpb} warps")
    if debug_capture is not None:
        _capture_first_super_iteration(x, kind, cfg.wpb, engine, debug_capture)
    return _device_scan(x, kind, size, engine)


def _capture_first_super_iteration(x, kind, wpb: int, engine: TileEngine, cap: dict) -> None:
    """The reference's block-scan introspection (scan.py:224-227): the
    scratch of the first super-iteration (``first_sout``: the wpb unseeded
    256-element tile scans, zeros after) and its partials (``first_prtls``:
    last_column_scan_16 of the tiles' totals, seeded with 0).  Recomputed on
    the GPU from the same tile scans / totals (extra launches, only when
    requested) -- the B200 kernel itself has no such scratch."""
    head = x[: 256 * wpb]
    eng = TileEngine(accumulate=engine.accumulate)
    sout = np.zeros(256 * 16, dtype=engine.acc_dtype)
    sout[: 256 * wpb] = _as_numpy(_device_scan(head, kind, 256, eng))
    tile = np.zeros((16, 16), np.float64)
    tile[:wpb, 15] = sout[255: 256 * wpb: 256]
    cap["first_prtls"] = last_column_scan_16(tile, eng, carry=0.0)
    cap["first_sout"] = sout


def _as_numpy(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


# -- grid level ----------------------------------------------------------------


def grid_scan(values, engine: TileEngine, cfg: BlockConfig = BlockConfig(),
              block_elems: int = 4096, workers: int = 1, reverse: bool = False,
              debug_capture: dict | None = None):
    """Inclusive scan of the whole vector (scan.py:249-310) in ONE launch:
    the CHUNK kernel fuses the reference's three passes (block totals, their
    scan, the uniform add) -- unit aggregates, their fixed-order fp64
    composition and the carry-seeded output pass run concurrently in one
    kernel.  ``debug_capture`` receives the reference's keys: ``passes`` =
    GRID_SCAN_PASSES (the logical passes; ``launches`` = 1 says they are
    fused) and ``block_totals``, the ``block_elems`` block sums in the
    accumulator dtype (one extra launch, only when requested)."""
    x, kind = _as_flat_half(values)
    _check_grid_cfg(cfg, block_elems)
    size = _d.size_of(x)
    if size == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    out = _device_scan(x, kind, size, engine)
    if debug_capture is not None:
        from .reduce import _device_reduce

        debug_capture["passes"] = GRID_SCAN_PASSES
        debug_capture["launches"] = 1
        debug_capture["block_totals"] = _as_numpy(_device_reduce(
            x, kind, block_elems, TileEngine(accumulate=engine.accumulate)))
    return out


def _check_grid_cfg(cfg: BlockConfig, block_elems: int = 4096) -> None:
    if block_elems % (256 * cfg.wpb):
        raise BadConfigError(
            f"block capacity {block_elems} is not a multiple of 256*wpb ({256 * cfg.wpb})")


# -- segmented driver -----------------------------------------------------------


def segmented_scan(values, seg_size: int, variant: str, engine: TileEngine,
                   cfg: BlockConfig = BlockConfig(), workers: int = 1, reverse: bool = False,
                   inclusive: bool = True):
    """Per-segment prefix sums at the logical length (scan.py:316-342).

    ``inclusive=False`` returns the exclusive scan; like the reference it
    requires the length to be a segment multiple."""
    x, kind = _as_flat_half(values)
    size = _d.size_of(x)
    if variant == "grid":
        if seg_size < size:
            raise BadConfigError("the grid variant scans the whole input as one segment")
        _check_grid_cfg(cfg)  # as grid_scan (scan.py:345-348 -> :262-265)
        if size == 0:
            raise BadLengthError("input must be a non-empty flat vector")
        if not inclusive and size % seg_size:
            raise BadLengthError("exclusive output needs the logical length to be a segment multiple")
        return _device_scan(x, kind, size, engine, inclusive=inclusive)
    if variant == "warp16" and seg_size != 16:
        raise BadConfigError("warp16 scans segments of exactly 16")
    if variant == "warp256" and seg_size != 256:
        raise BadConfigError("warp256 scans segments of exactly 256")
    if variant not in SCAN_VARIANTS:
        raise BadConfigError(f"unknown scan variant {variant!r}; pick from {SCAN_VARIANTS}")
    if size == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    if seg_size < 1:
        raise BadLengthError(f"segment size must be positive, got {seg_size}")
    if not inclusive and size % seg_size:
        raise BadLengthError("exclusive output needs the logical length to be a segment multiple")
    return _device_scan(x, kind, seg_size, engine, inclusive=inclusive)
