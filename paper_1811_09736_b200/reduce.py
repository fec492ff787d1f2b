"""Segmented reduction on B200 tensor cores -- drop-in for
pkg/src/halftile/reduce.py.

Every public function keeps the reference signature, argument validation,
exception types and result shape/dtype; the arithmetic runs in the sm_100a
kernels behind ``tc_seg_reduce`` / ``tc_full_reduce``
(include/tc_collectives.h).  The reference's warp / block / grid variants
are different *schedules* of the same P.A.Q tile product (reduce.py:1-27);
on B200 one persistent TMA -> tcgen05.mma -> TMEM pipeline serves all of
them, so every variant name maps to that kernel family and the values agree
(they are bit-identical to the reference on exact-integer data, and at
least as accurate on general data: one rounding instead of one per MMA).

Scheduling knobs (``cfg``, ``workers``, ``reverse``) are validated exactly
like the reference and do not change results (the kernels are
deterministic: no float atomics, fixed combine order).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _dispatch as _d
from .engine import TileEngine
from .errors import BadConfigError, BadLengthError

GRID_REDUCE_PASSES = 2  # reference constant (reduce.py:41); B200 does it in ONE launch

REDUCE_VARIANTS = (
    "warp16",
    "warp256",
    "strided16n",
    "coalesced16n",
    "efficient256n",
    "inefficient256n",
    "block256n",
    "grid",
)


@dataclass(frozen=True)
class BlockConfig:
    """Block-level execution shape (reduce.py:55-66): validated, and used
    only for the reference's divisibility contracts."""

    wpb: int = 4
    coarsening: int = 1

    def __post_init__(self):
        if not 1 <= self.wpb <= 16:
            raise BadConfigError(f"warps per block must be in [1, 16], got {self.wpb}")
        if self.coarsening < 1:
            raise BadConfigError(f"coarsening must be positive, got {self.coarsening}")


def _as_flat_half(values):
    """reduce.py:69-73 (non-flat -> BadLengthError)."""
    return _d.flat_half(values)


def clamp_block_config(cfg: BlockConfig, n_tiles: int) -> BlockConfig:
    """Largest warp count <= cfg.wpb dividing the tile count (reduce.py:267-272)."""
    wpb = min(cfg.wpb, n_tiles)
    while n_tiles % wpb:
        wpb -= 1
    return cfg if wpb == cfg.wpb else BlockConfig(wpb=wpb, coarsening=cfg.coarsening)


def coalesced_group_mma_count(seg_size: int) -> int:
    """Closed-form MMA count of the reference's coalesced group (reduce.py:259-264)."""
    n = seg_size // 16
    if n < 16:
        return n
    return 16 * (n // 16 + 1) + n % 16


# -- device dispatch -----------------------------------------------------------


def _device_reduce(x, kind, seg: int, engine: TileEngine):
    """ceil(n/seg) sums of x on the GPU, returned in the caller's domain."""
    from . import _device

    n = _d.size_of(x)
    dev = _d.to_device(x, kind)
    out = _device.seg_reduce(dev, seg, _d.torch_dtype(engine.acc_dtype))
    engine._account(n, -(-n // seg), scan=False)
    return _d.from_device(out, kind, engine.acc_dtype)


def _scalar(res, engine):
    if hasattr(res, "numel"):  # torch result: 0-d view stays on its device
        return res[0]
    return engine.acc_dtype.type(res[0])


# -- warp level ----------------------------------------------------------------


def reduce_16(values, engine: TileEngine):
    """Sums of 16 consecutive segments of 16 (reduce.py:92-106)."""
    x, kind = _as_flat_half(values)
    if _d.size_of(x) != 256:
        raise BadLengthError(f"reduce_16 takes exactly 256 elements, got {_d.size_of(x)}")
    return _device_reduce(x, kind, 16, engine)


def reduce_256(values, engine: TileEngine):
    """Total of one 256-element segment (reduce.py:109-120)."""
    x, kind = _as_flat_half(values)
    if _d.size_of(x) != 256:
        raise BadLengthError(f"reduce_256 takes exactly 256 elements, got {_d.size_of(x)}")
    return _scalar(_device_reduce(x, kind, 256, engine), engine)


def reduce_256n_efficient(values, n: int, engine: TileEngine):
    """Total of a 256n segment (reduce.py:123-141)."""
    x, kind = _as_flat_half(values)
    if n < 1 or _d.size_of(x) != 256 * n:
        raise BadLengthError(f"need exactly 256*{n} elements, got {_d.size_of(x)}")
    return _scalar(_device_reduce(x, kind, 256 * n, engine), engine)


def reduce_256n_inefficient(values, n: int, engine: TileEngine):
    """Same value as the efficient variant (reduce.py:144-168)."""
    x, kind = _as_flat_half(values)
    if n < 1 or _d.size_of(x) != 256 * n:
        raise BadLengthError(f"need exactly 256*{n} elements, got {_d.size_of(x)}")
    return _scalar(_device_reduce(x, kind, 256 * n, engine), engine)


def _check_16n(x, seg_size, group):
    if seg_size < 16 or seg_size % 16:
        raise BadLengthError(f"segment size must be a positive multiple of 16, got {seg_size}")
    size = _d.size_of(x)
    if size == 0 or size % group:
        raise BadLengthError(
            f"input length {size} is not a multiple of the {group}-element warp group")


def reduce_16n_strided(values, seg_size: int, engine: TileEngine):
    """Per-segment sums, 16 segments of 16n per warp group (reduce.py:171-198)."""
    x, kind = _as_flat_half(values)
    _check_16n(x, seg_size, 256 * (seg_size // 16))
    return _device_reduce(x, kind, seg_size, engine)


def reduce_16n_coalesced(values, seg_size: int, engine: TileEngine):
    """Per-segment sums, contiguous-chunk schedule (reduce.py:201-256)."""
    x, kind = _as_flat_half(values)
    _check_16n(x, seg_size, 16 * seg_size)
    return _device_reduce(x, kind, seg_size, engine)


# -- block level ---------------------------------------------------------------


def block_reduce_256n(values, cfg: BlockConfig, engine: TileEngine, workers: int = 1,
                      reverse: bool = False, debug_capture: dict | None = None):
    """Total of one 256n segment (reduce.py:278-326).  ``debug_capture``
    receives the per-warp-slice partials (computed on the GPU with one extra
    launch, only when requested)."""
    x, kind = _as_flat_half(values)
    size = _d.size_of(x)
    if size % 256:
        raise BadLengthError(f"segment length {size} is not a multiple of 256")
    n = size // 256
    if n % cfg.wpb:
        raise BadConfigError(f"{n} tiles do not divide across {cfg.wpb} warps")
    if debug_capture is not None:
        debug_capture["partials"] = _device_reduce(x, kind, size // cfg.wpb, TileEngine(
            accumulate=engine.accumulate))
    return _scalar(_device_reduce(x, kind, size, engine), engine)


# -- grid level ----------------------------------------------------------------


def grid_reduce(values, engine: TileEngine, cfg: BlockConfig = BlockConfig(),
                block_elems: int = 4096, workers: int = 1, reverse: bool = False,
                debug_capture: dict | None = None):
    """Full reduction (reduce.py:332-373) in ONE kernel launch: per-CTA fp64
    partials combined in CTA order by the last CTA.  ``debug_capture``
    receives the reference's keys: ``passes`` = GRID_REDUCE_PASSES, the
    reference algorithm's two logical passes (block partials, then their
    reduction), which the B200 kernel fuses -- ``launches`` = 1 says so --
    and ``partials``, the ``block_elems`` block sums in the accumulator dtype
    (one extra launch, only when requested)."""
    x, kind = _as_flat_half(values)
    if block_elems % (256 * cfg.wpb):
        raise BadConfigError(
            f"block capacity {block_elems} is not a multiple of 256*wpb ({256 * cfg.wpb})")
    size = _d.size_of(x)
    if size == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    total = _scalar(_device_reduce(x, kind, size, engine), engine)
    if debug_capture is not None:
        debug_capture["passes"] = GRID_REDUCE_PASSES
        debug_capture["launches"] = 1
        debug_capture["partials"] = _device_reduce(x, kind, block_elems, TileEngine(
            accumulate=engine.accumulate))
    return total


# -- segmented driver -----------------------------------------------------------


def segmented_reduce(values, seg_size: int, variant: str, engine: TileEngine,
                     cfg: BlockConfig = BlockConfig(), workers: int = 1,
                     reverse: bool = False):
    """One sum per logical segment (reduce.py:379-446); same validation order
    and errors as the reference, one B200 kernel for every variant."""
    x, kind = _as_flat_half(values)
    size = _d.size_of(x)
    if variant == "grid":
        total = grid_reduce(x, engine, cfg=cfg, workers=workers, reverse=reverse)
        if kind == "numpy":
            return np.array([total], dtype=engine.acc_dtype)
        return total.reshape(1)
    if variant == "warp16" and seg_size != 16:
        raise BadConfigError("warp16 reduces segments of exactly 16")
    if variant == "warp256" and seg_size != 256:
        raise BadConfigError("warp256 reduces segments of exactly 256")
    if variant not in REDUCE_VARIANTS:
        raise BadConfigError(f"unknown reduce variant {variant!r}; pick from {REDUCE_VARIANTS}")
    # pad_segmented's contract (segmented.py:57-89)
    if size == 0:
        raise BadLengthError("input must be a non-empty flat vector")
    if seg_size < 1:
        raise BadLengthError(f"segment size must be positive, got {seg_size}")
    return _device_reduce(x, kind, seg_size, engine)
