"""``TileEngine`` of the drop-in: precision mode + cost counters.

The reference ``TileEngine`` (pkg/src/halftile/engine.py:221-529) is a CPU
simulation of WMMA fragments.  On B200 the tiles live in shared memory and
TMEM inside the kernels, so this class keeps only what callers of the
collectives use:

* ``accumulate`` ("half" | "single") selects the output dtype,
  ``acc_dtype`` (engine.py:244-246): fp16 or fp32 results.  On B200 every
  result is accumulated in fp32/fp64 and rounded ONCE to ``acc_dtype``
  (never less precise than the reference's per-MMA rounding, engine.py:
  326-348).
* ``counters`` (``CostCounters``, engine.py:95-126) tallies the work the
  B200 kernels actually issue: 4 ``tcgen05.mma`` (K = 4 x 16) per
  8192-element tile, one TMA tile load per tile, one TMA tile store per
  scan tile.  ``cycle_estimate`` keeps the reference's 32-cycles-per-MMA
  formula for API compatibility only.
* ``relaxed`` / ``trace`` are accepted and stored (the strict-WMMA traffic
  model and the load trace are simulator-only).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, fields

import numpy as np

HALF = np.float16

#: elements per kernel tile (128 rows x 64) and tcgen05.mma per tile
TILE_ELEMS = 8192
MMA_PER_TILE = 4


class FragmentKind(enum.Enum):
    """Operand roles of an MMA (engine.py:55-58), kept for API compatibility."""

    MATRIX_A = "matrix_a"
    MATRIX_B = "matrix_b"
    ACCUMULATOR = "accumulator"


class Layout(enum.Enum):
    """Tile layouts (engine.py:61-63), kept for API compatibility."""

    ROW_MAJOR = "row_major"
    COL_MAJOR = "col_major"


@dataclass
class CostCounters:
    """Operation tallies (same fields as engine.py:95-126)."""

    mma_count: int = 0
    tile_loads: int = 0
    tile_stores: int = 0
    fill_count: int = 0
    elements_loaded: int = 0
    elements_stored: int = 0

    CYCLES_PER_MMA = 32

    @property
    def cycle_estimate(self) -> int:
        return self.CYCLES_PER_MMA * self.mma_count

    def merge(self, other: "CostCounters") -> None:
        for f in fields(self):
            setattr(self, f.name, getattr(self, f.name) + getattr(other, f.name))

    def snapshot(self) -> "CostCounters":
        return CostCounters(**{f.name: getattr(self, f.name) for f in fields(self)})

    def delta(self, since: "CostCounters") -> "CostCounters":
        return CostCounters(
            **{f.name: getattr(self, f.name) - getattr(since, f.name) for f in fields(self)}
        )


class TileEngine:
    """Precision mode and counters of one caller (engine.py:233-240 signature)."""

    def __init__(self, relaxed: bool = True, accumulate: str = "half", trace: bool = False):
        if accumulate not in ("half", "single"):
            raise ValueError("accumulate must be 'half' or 'single'")
        self.relaxed = relaxed
        self.accumulate = accumulate
        self.counters = CostCounters()
        self.load_trace = [] if trace else None
        self._trace = trace

    @property
    def acc_dtype(self) -> np.dtype:
        return np.dtype(np.float32) if self.accumulate == "single" else np.dtype(HALF)

    def spawn(self) -> "TileEngine":
        return TileEngine(relaxed=self.relaxed, accumulate=self.accumulate, trace=self._trace)

    def absorb(self, other: "TileEngine") -> None:
        self.counters.merge(other.counters)
        if self._trace and other.load_trace:
            self.load_trace.extend(other.load_trace)

    # -- B200 accounting ---------------------------------------------------
    def _account(self, n: int, n_out: int, scan: bool) -> None:
        tiles = -(-n // TILE_ELEMS)
        c = self.counters
        c.mma_count += MMA_PER_TILE * tiles
        c.tile_loads += tiles
        c.tile_stores += tiles if scan else 0
        c.elements_loaded += n
        c.elements_stored += n_out
