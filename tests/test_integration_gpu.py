"""The torch-free reference-side binding (integration/halftile_b200.py, the
stub INTEGRATION.md tells a halftile maintainer to add) against the oracle,
on the GPU, through nothing but ctypes + the CUDA runtime."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("s", [16, 48, 256, 4096, 65536])
def test_binding_reduce_and_scan_exact(s, cuda):
    from integration import halftile_b200 as B

    assert B.available()
    rng = np.random.default_rng(20260810)
    n = 1 << 20
    x = O.exact_int_segments(rng, (n // s) * s, s)
    sums = B.seg_reduce(x, s, np.float16)
    assert np.array_equal(sums, O.ref_seg_reduce(x, s).astype(np.float16))
    scans = B.seg_scan(x, s, np.float32)
    assert np.array_equal(scans, O.ref_seg_scan(x, s).astype(np.float32))
    ex = B.seg_scan(x, s, np.float32, inclusive=False)
    assert np.array_equal(ex, O.ref_seg_scan(x, s, inclusive=False).astype(np.float32))


def test_binding_irregular_reduce(cuda):
    from integration import halftile_b200 as B

    rng = np.random.default_rng(5)
    n = (1 << 20) + 77
    x = rng.integers(0, 4, n).astype(np.float16)
    off = O.random_offsets(rng, n, 100, empty_frac=0.2)
    got = B.irregular_reduce(x, off, np.float32)
    assert np.array_equal(got, O.ref_irreg_reduce(x, off).astype(np.float32))
