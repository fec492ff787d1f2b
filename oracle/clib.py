"""TEST INFRASTRUCTURE -- ctypes binding of oracle/oracle.c (the threaded C
restatement of halftile's exact oracle, pkg/src/halftile/oracle.py:47-75).

Used by tests/ and by bench.py's CPU-baseline leg only; the product never
imports anything under oracle/.  The tolerance checkers compare a GPU result
with the exact binary64 oracle element by element without materialising the
reference, which is what makes element-wise checks at 2^30 / 2^33 elements
feasible (tests/test_parity_full_gpu.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
SO = ROOT / "build" / "liboracle.so"

_lib = None

# dtype codes of the checkers
DT = {np.dtype(np.float16): 0, np.dtype(np.float32): 1, np.dtype(np.float64): 2}


def threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


def lib():
    global _lib
    if _lib is None:
        if not SO.exists():
            subprocess.run(["make", "-s", "-C", str(ROOT)], check=True)
        L = ctypes.CDLL(str(SO))
        P, I64, I, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.or_seg_reduce.argtypes = [P, I64, I64, P, I]
        L.or_seg_scan.argtypes = [P, I64, I64, I, D, I, P, I]
        L.or_check_seg_reduce.argtypes = [P, I64, I64, P, I, D, D, I, P]
        L.or_check_seg_reduce.restype = I64
        L.or_check_seg_scan.argtypes = [P, I64, I64, I64, I, I, P, P, P, I, D, D, I, P]
        L.or_check_seg_scan.restype = I64
        _lib = L
    return _lib


def _bits(x) -> np.ndarray:
    x = np.ascontiguousarray(x)
    assert x.dtype == np.float16
    return x


def seg_reduce(x, s: int) -> np.ndarray:
    """Exact (binary64) segment sums, ceil(n/s) outputs."""
    x = _bits(x)
    out = np.empty(-(-x.size // s), np.float64)
    lib().or_seg_reduce(x.ctypes.data, x.size, s, out.ctypes.data, threads())
    return out


class Check:
    """Result of a checker call: violations, worst error / bound ratio, worst
    absolute error, first violating index, worst relative error (|v| >= 1)."""

    def __init__(self, bad, stats):
        self.bad = int(bad)
        self.max_ratio, self.max_abs, first, self.max_rel = (float(v) for v in stats)
        self.first_bad = int(first)

    def __repr__(self):
        return (f"Check(bad={self.bad}, first_bad={self.first_bad}, max_ratio={self.max_ratio:.3g}, "
                f"max_abs={self.max_abs:.3g}, max_rel={self.max_rel:.3g})")


def check_seg_reduce(x, s: int, got, ulps: float, gamma: float) -> Check:
    """|got[k] - exact_k| <= ulps * ulp(exact_k) + gamma * sum|x| over segment k."""
    x = _bits(x)
    got = np.ascontiguousarray(got)
    assert got.size == -(-x.size // s)
    st = np.zeros(4)
    bad = lib().or_check_seg_reduce(x.ctypes.data, x.size, s, got.ctypes.data, DT[got.dtype],
                                    ulps, gamma, threads(), st.ctypes.data)
    return Check(bad, st)


class ScanChecker:
    """Chunk-by-chunk check of a segmented scan of x (global segment starts
    at multiples of s): feed consecutive output chunks with ``check(lo, got)``;
    the exact running state is carried between chunks."""

    def __init__(self, x, s: int, inclusive: bool = True, carry: float | None = None):
        self.x = _bits(x)
        self.s = int(s)
        self.inclusive = 1 if inclusive else 0
        self.cont0 = 1 if carry is not None else 0
        self.run = ctypes.c_double(float(carry) if carry is not None else 0.0)
        self.arun = ctypes.c_double(0.0)
        self.next = 0
        self.bad = 0
        self.max_ratio = self.max_abs = self.max_rel = 0.0
        self.first_bad = -1

    def check(self, lo: int, got, ulps: float, gamma: float) -> "ScanChecker":
        assert lo == self.next, "chunks must be consecutive"
        got = np.ascontiguousarray(got)
        hi = lo + got.size
        st = np.zeros(4)
        bad = lib().or_check_seg_scan(self.x.ctypes.data, lo, hi, self.s, self.inclusive,
                                      self.cont0, ctypes.byref(self.run), ctypes.byref(self.arun),
                                      got.ctypes.data, DT[got.dtype], ulps, gamma, threads(),
                                      st.ctypes.data)
        c = Check(bad, st)
        if c.bad and self.first_bad < 0:
            self.first_bad = c.first_bad
        self.bad += c.bad
        self.max_ratio = max(self.max_ratio, c.max_ratio)
        self.max_abs = max(self.max_abs, c.max_abs)
        self.max_rel = max(self.max_rel, c.max_rel)
        self.next = hi
        return self

    @property
    def exact_total(self) -> float:
        """Exact running sum after the last checked element."""
        return self.run.value

    def __repr__(self):
        return (f"ScanChecker(bad={self.bad}, first_bad={self.first_bad}, "
                f"max_ratio={self.max_ratio:.3g}, max_abs={self.max_abs:.3g}, "
                f"max_rel={self.max_rel:.3g})")
