"""GPU parity of the irregular (CSR-offset) segmented reduce / scan
(tc_irreg_reduce / tc_irreg_scan) against the exact oracle
(oracle.ref_irreg_reduce / ref_irreg_scan, binary64 per segment).

Tolerances (stated here and in paper_1811_09736_b200/irregular.py):
* exact-integer inputs (every partial sum < 2^24): BIT-EXACT against
  fp16(exact) / fp32(exact) / fp64(exact);
* uniform [0, 1) inputs, fp32 output: |got - exact| <= 1e-5 * |exact| +
  2^-16 -- a segment value is built from at most two in-row fp32 prefixes
  (each <= 64 here, so a few fp32 ulps of 64 = 2^-16 absolute) plus the
  same fp32/fp64 carry chain as the regular path (relative 1e-5);
* fp16 output: |got - exact| <= 1 fp16 ulp(exact) + 2^-16;
* output counts and positions: identical (empty segments give 0).
"""

import numpy as np
import pytest
import torch

import paper_1811_09736_b200 as ht
from paper_1811_09736_b200 import _device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

ATOL = 2.0 ** -16


def ulp16(v):
    a = np.abs(np.asarray(v, np.float64)).astype(np.float16)
    return np.spacing(a).astype(np.float64)


def assert_bits(got, exp64):
    got = np.asarray(got)
    exp = np.asarray(exp64, np.float64).astype(got.dtype)
    assert got.shape == exp.shape, (got.shape, exp.shape)
    ui = {2: np.uint16, 4: np.uint32, 8: np.uint64}[got.dtype.itemsize]
    bad = np.nonzero(got.view(ui) != exp.view(ui))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[:5]}: {got[bad[:3]]} vs {exp[bad[:3]]}"


def assert_close(got, exact):
    got = np.asarray(got)
    exact = np.asarray(exact, np.float64)
    assert got.shape == exact.shape
    err = np.abs(got.astype(np.float64) - exact)
    if got.dtype == np.float16:
        tol = ulp16(exact) + ATOL
    else:
        tol = 1e-5 * np.abs(exact) + ATOL
    bad = np.nonzero(err > tol)[0]
    assert bad.size == 0, f"{bad.size} out of tolerance, first {bad[:5]}: {got[bad[:3]]} vs {exact[bad[:3]]}"


def int_data(rng, n):
    return rng.integers(0, 4, n).astype(np.float16)  # sums <= 3n < 2^24 for n <= 2^22


# sizes around the row (64), tile (8192) and CTA-range boundaries
SIZES = [1, 63, 64, 65, 8191, 8192, 8193, 3 * 8192 + 100, (1 << 20) + 37, 1 << 21]
MEANS = [1, 3, 17, 64, 300, 5000]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("mean", MEANS)
def test_irreg_reduce_exact_int(cuda, rng, n, mean):
    x = int_data(rng, n)
    off = O.random_offsets(rng, n, mean, empty_frac=0.2)
    exp = O.ref_irreg_reduce(x, off)
    for acc in ("half", "single"):
        got = ht.irregular_segmented_reduce(x, off, ht.TileEngine(accumulate=acc))
        assert_bits(got, exp)
    xd = torch.from_numpy(x).to(cuda)
    od = torch.from_numpy(off).to(cuda)
    assert_bits(D.irreg_reduce(xd, od, torch.float64).cpu().numpy(), exp)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("mean", MEANS)
def test_irreg_scan_exact_int(cuda, rng, n, mean):
    x = int_data(rng, n)
    off = O.random_offsets(rng, n, mean, empty_frac=0.2)
    for inclusive in (True, False):
        exp = O.ref_irreg_scan(x, off, inclusive)
        got = ht.irregular_segmented_scan(x, off, ht.TileEngine(accumulate="single"), inclusive=inclusive)
        assert_bits(got, exp)
    # fp16 out on data whose prefix sums stay exact in fp16 (<= 2048)
    x16 = (rng.random(n) < 0.05).astype(np.float16)
    off16 = O.random_offsets(rng, n, min(mean, 2000), empty_frac=0.1)
    got = ht.irregular_segmented_scan(x16, off16, ht.TileEngine())
    assert_bits(got, O.ref_irreg_scan(x16, off16))


def special_offsets(n):
    cases = {
        "one_segment": [0, n],
        "leading_empties": [0, 0, 0, n],
        "trailing_empties": [0, n, n, n],
        "all_singletons": list(range(n + 1)),
        "row_aligned": sorted(set(list(range(0, n, 64)) + [n])),
        "tile_aligned": sorted(set(list(range(0, n, 8192)) + [n])),
        "mid_and_dups": [0] + [n // 3] * 5 + [n // 2, n // 2] + [n],
    }
    return {k: np.asarray(v, np.int64) for k, v in cases.items()}


@pytest.mark.parametrize("n", [64, 8192, 5 * 8192, 5 * 8192 + 1, (1 << 21) + 64 * 5, 1 << 21])
def test_irreg_special_offsets(cuda, rng, n):
    x = int_data(rng, n)
    for name, off in special_offsets(n).items():
        if name == "all_singletons" and n > 1 << 16:
            continue
        er = O.ref_irreg_reduce(x, off)
        assert_bits(ht.irregular_segmented_reduce(x, off, ht.TileEngine(accumulate="single")), er)
        for inclusive in (True, False):
            es = O.ref_irreg_scan(x, off, inclusive)
            got = ht.irregular_segmented_scan(x, off, ht.TileEngine(accumulate="single"),
                                              inclusive=inclusive)
            assert_bits(got, es)


@pytest.mark.parametrize("mean", [1, 17, 300, 5000, 1 << 20])
def test_irreg_uniform_tolerance(cuda, mean):
    g = np.random.default_rng(7)
    n = (1 << 22) + 123
    x = g.random(n).astype(np.float16)
    off = O.random_offsets(g, n, mean, empty_frac=0.1)
    er = O.ref_irreg_reduce(x, off)
    for acc in ("single", "half"):
        assert_close(ht.irregular_segmented_reduce(x, off, ht.TileEngine(accumulate=acc)), er)
    es = O.ref_irreg_scan(x, off)
    assert_close(ht.irregular_segmented_scan(x, off, ht.TileEngine(accumulate="single")), es)
    ee = O.ref_irreg_scan(x, off, inclusive=False)
    assert_close(ht.irregular_segmented_scan(x, off, ht.TileEngine(accumulate="single"),
                                             inclusive=False), ee)


def test_irreg_matches_regular_path(cuda, rng):
    """Uniform offsets k*s: the irregular kernels equal the regular ones."""
    n = (1 << 20) + 300
    x = int_data(rng, n)
    xd = torch.from_numpy(x).to(cuda)
    for s in (16, 300, 4096, 100000):
        off = torch.from_numpy(np.minimum(np.arange(0, n + s, s), n).astype(np.int64)).to(cuda)
        off = torch.unique(off)
        a = D.irreg_reduce(xd, off, torch.float32)
        b = D.seg_reduce(xd, s, torch.float32)
        assert torch.equal(a, b), s
        a = D.irreg_scan(xd, off, torch.float32)
        b = D.seg_scan(xd, s, torch.float32)
        assert torch.equal(a, b), s


def test_irreg_bf16_and_determinism(cuda, rng):
    n = (1 << 21) + 9
    xi = rng.integers(0, 4, n).astype(np.float32)
    off = O.random_offsets(rng, n, 200, empty_frac=0.2)
    xd = torch.from_numpy(xi).to(cuda).to(torch.bfloat16)
    od = torch.from_numpy(off).to(cuda)
    assert_bits(D.irreg_reduce(xd, od, torch.float32).cpu().numpy(), O.ref_irreg_reduce(xi, off))
    assert_bits(D.irreg_scan(xd, od, torch.float32).cpu().numpy(), O.ref_irreg_scan(xi, off))
    xu = torch.rand(n, device=cuda).to(torch.float16)
    r1 = D.irreg_reduce(xu, od, torch.float32)
    s1 = D.irreg_scan(xu, od, torch.float32)
    for _ in range(3):
        assert torch.equal(D.irreg_reduce(xu, od, torch.float32), r1)
        assert torch.equal(D.irreg_scan(xu, od, torch.float32), s1)


def test_irreg_device_offsets_validation(cuda):
    x = torch.ones(1000, device=cuda, dtype=torch.float16)
    for bad in ([0, 500, 400, 1000], [1, 1000], [0, 999]):
        with pytest.raises(ht.BadConfigError):
            ht.irregular_segmented_reduce(x, torch.tensor(bad, device=cuda))
        with pytest.raises(ht.BadConfigError):
            ht.irregular_segmented_scan(x, torch.tensor(bad, device=cuda))
    out = ht.irregular_segmented_reduce(x, torch.tensor([0, 10, 10, 1000], device=cuda))
    assert out.is_cuda and out.tolist() == [10.0, 0.0, 990.0]


def test_irreg_full_size_properties(cuda):
    """2^30 elements, ~2^22 segments: scan tail == reduce (exact ints, fp32),
    and the fp64 sum of the segment sums == the full reduce."""
    n = 1 << 30
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    x = torch.randint(0, 2, (n,), device=cuda, generator=g, dtype=torch.int32).to(torch.float16)
    lens = torch.randint(0, 512, (n // 200,), device=cuda, generator=g, dtype=torch.int64)
    ends = torch.cumsum(lens, 0)
    ends = ends[ends < n]
    off = torch.cat([torch.zeros(1, dtype=torch.int64, device=cuda), ends,
                     torch.tensor([n], device=cuda)])
    red = D.irreg_reduce(x, off, torch.float64)
    assert float(red.sum()) == float(D.full_reduce(x, torch.float64).item())
    scan = D.irreg_scan(x, off, torch.float32)
    nonempty = off[1:] > off[:-1]
    tails = scan[(off[1:] - 1)[nonempty]]
    assert torch.equal(tails.to(torch.float64), red[nonempty])
    del scan
    ex = D.irreg_scan(x, off, torch.float32, exclusive=True)
    assert torch.all(ex[off[:-1][nonempty]] == 0)
