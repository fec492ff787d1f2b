"""GPU parity over the FULL binary16 input domain: signed data, mixed
magnitudes, cancellation and non-finite values, in every carry mode.

Error bound (stated here and in DESIGN.md section 5).  For an output whose
exact (binary64) value is v and whose elements have absolute mass
A = sum |x| (the segment for a reduce, the segment's prefix up to the
output for a scan):

    |got - v| <= 1 ulp_out(v) + GAMMA * A,     GAMMA = 16 * 2^-24

ulp_out is the fp16 / fp32 unit in the last place at |v|: one rounding of
the output (1 ulp covers the double rounding fp32 -> fp16); GAMMA * A bounds
the fp32 accumulation inside the tensor core and the epilogue's fp32 row /
warp combines (at most ~16 dependent fp32 roundings of partial sums of the
output's OWN elements; cross-tile and cross-CTA carries are fp64).  A bound
in A -- rather than in |v| -- is the standard one for floating-point
summation: it stays meaningful under cancellation, and it is violated by any
scheme whose error scales with NEIGHBOURING segments' magnitudes (prefix
differences across segment boundaries), which the mixed-magnitude data below
is built to expose.

Irregular (CSR) segments (an extension with no reference counterpart) are
bounded with A' = sum |x| from the start of the 64-element row holding the
segment's first element: their in-row pieces are differences of in-row
prefixes (IRREG).

Exact-integer signed data is checked bit-for-bit (every partial sum is an
exact integer < 2^24, so fp32 outputs are exact and fp16 outputs are
fp16(exact) -- the reference simulator's own answer on such data).
"""

import numpy as np
import pytest
import torch

from paper_1811_09736_b200 import _device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu

GAMMA = 16 * 2.0 ** -24
N = (1 << 22) + 1234  # ragged: not a multiple of 64, 8192 or any segment size

# segment sizes by kernel mode (tc_collectives.cu make_params):
#   LOCAL s | 64; ROWS 64 * 2^k <= 8192; TILES 8192 * k; GENERAL (incl. the
#   one/two-end select sums: 48, 1000, 127, 129, 4097); GSCR (many ends per
#   row); ROWSEG (gcd(s, 64) <= 8 with whole segments per TMA row: 3, 7, 12,
#   17, 20, 24, 63, 65, 100, 300); SPLIT (s >= 12288, gcd(s, 64) <= 4:
#   16411, 100001, 524292, 1000003)
REDUCE_SEGS = [1, 2, 16, 64, 256, 8192, 16384, 24576, 3, 7, 12, 17, 20, 24, 63, 48, 65, 100,
               127, 129, 4097, 16411, 524292, 1000003, 300, 1000, 100001, N]
#   scans: LOCAL / ROWS / TILES / GENERAL as above; ROWSEG (s < 9, gcd(s, 64)
#   <= 2, fp16 out: 3, 6, 9, 17, 33, 63; fp32 out s <= 9); SPLITM (fp32 out, odd
#   11 <= s < 64: 17, 33, 63); SPLIT (s >= 64, gcd(s, 64) <= 4, up to
#   2^21: 65, 66, 100, 130, 300, 4097, 100001, 524292, 1000003); CHUNK for
#   s > 2^18 with one granule per row ((1 << 18) + 8192), s > 2^21 and full
SCAN_SEGS = [1, 16, 64, 256, 8192, 16384, 3, 6, 9, 10, 12, 17, 33, 48, 63, 65, 66, 100, 130, 300,
             1000, 4097, 100001, (1 << 18) + 8192, 524292, 1000003, (1 << 21) + 1, N]


def _ulp(v, dt):
    a = np.abs(np.asarray(v, np.float64))
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    if dt == np.float16:
        return np.where((a > 0) & (e >= -14), 2.0 ** (e - 10), 2.0 ** -24)
    return np.where((a > 0) & (e >= -126), 2.0 ** (e - 23), 2.0 ** -149)


def assert_bounded(got, exact, mass, dt, what):
    got = np.asarray(got).astype(np.float64)
    assert got.shape == exact.shape, what
    err = np.abs(got - exact)
    bound = _ulp(exact, dt) + GAMMA * mass
    bad = np.nonzero(~np.isfinite(got) | (err > bound))[0]
    assert bad.size == 0, (f"{what}: {bad.size} outputs out of bound, first {bad[:4]}, "
                           f"err {err[bad[:4]]}, bound {bound[bad[:4]]}")


def mixed_magnitude(rng, n, big=16.0, small=2.0 ** -8):
    """Signed values in runs of random length (1..200) whose magnitude
    alternates between ~big and ~small (ratio 2^12): a segment of small
    values sits next to large ones in the same row / tile."""
    x = np.empty(n, np.float64)
    i = 0
    flip = False
    while i < n:
        L = int(rng.integers(1, 201))
        mag = big if flip else small
        x[i:i + L] = (rng.random(min(L, n - i)) * 2 - 1) * mag
        i += L
        flip = not flip
    return x.astype(np.float16)


DATASETS = {
    "int": lambda rng, n: rng.integers(-8, 8, n).astype(np.float16),
    "uniform_pm1": lambda rng, n: (rng.random(n) * 2 - 1).astype(np.float16),
    "mixed_mag": mixed_magnitude,
    # near-cancelling: +a / -a pairs shifted by one element, plus tiny noise
    "cancel": lambda rng, n: (np.repeat(rng.random((n + 1) // 2) * 100, 2)[:n]
                              * np.resize([1.0, -1.0], n) + rng.random(n) * 2.0 ** -6
                              ).astype(np.float16),
}


@pytest.fixture(scope="module")
def data(cuda):
    rng = np.random.default_rng(20260810)
    out = {}
    for k, f in DATASETS.items():
        x = f(rng, N)
        out[k] = (x, torch.from_numpy(x).to(cuda))
    return out


@pytest.mark.parametrize("kind", list(DATASETS))
def test_signed_reduce_every_mode(kind, data):
    x, xd = data[kind]
    ax = np.abs(x)
    for s in REDUCE_SEGS:
        exact = O.ref_seg_reduce(x, s)
        mass = O.ref_seg_reduce(ax, s)
        for dt, npdt in ((torch.float32, np.float32), (torch.float16, np.float16),
                         (torch.float64, np.float64)):
            if npdt == np.float16 and np.abs(exact).max() >= 65504:
                continue  # fp16 overflow is its own test (test_edge_semantics)
            got = D.seg_reduce(xd, s, dt).cpu().numpy()
            if kind == "int":
                assert np.array_equal(got, exact.astype(npdt)), (kind, s, npdt)
            else:
                assert_bounded(got, exact, mass, np.float32 if npdt == np.float64 else npdt,
                               f"reduce {kind} s={s} {npdt.__name__}")


@pytest.mark.parametrize("kind", list(DATASETS))
def test_signed_scan_every_mode(kind, data):
    x, xd = data[kind]
    ax = np.abs(x)
    for s in SCAN_SEGS:
        for exc in (False, True):
            exact = O.ref_seg_scan(x, s, inclusive=not exc)
            # mass of an exclusive output = the elements it sums (those before it)
            mass = O.ref_seg_scan(ax, s, inclusive=not exc)
            for dt, npdt in ((torch.float32, np.float32), (torch.float16, np.float16)):
                if npdt == np.float16 and np.abs(exact).max() >= 65504:
                    continue
                got = D.seg_scan(xd, s, dt, exclusive=exc).cpu().numpy()
                if kind == "int":
                    assert np.array_equal(got, exact.astype(npdt)), (kind, s, exc, npdt)
                else:
                    assert_bounded(got, exact, mass, npdt, f"scan {kind} s={s} exc={exc} {npdt.__name__}")


@pytest.mark.parametrize("kind", ["int", "uniform_pm1", "mixed_mag"])
def test_signed_carry_in_total_out(kind, data, cuda):
    """CHUNK mode with a carry-in (the multi-GPU full-scan building block):
    outputs bounded as above (the carry counts as one more summand); total_out comes
    from the fp64 carry chain, so its only error is the fp32 accumulation of
    the in-row / in-tile pieces: bounded by GAMMA * A with no output
    rounding (and exact on integer data)."""
    x, xd = data[kind]
    carry = -1234.5
    cin = torch.tensor([carry], dtype=torch.float64, device=cuda)
    tot = torch.zeros(1, dtype=torch.float64, device=cuda)
    ax = np.abs(x)
    for exc in (False, True):
        exact = O.ref_seg_scan(x, N, inclusive=not exc, carry=carry)
        # the caller's carry is one more summand of every output (its value
        # enters the kernel's fp64 chain and is rounded with the offset)
        mass = O.ref_seg_scan(ax, N, inclusive=not exc) + abs(carry)
        got = D.seg_scan(xd, N, torch.float32, exclusive=exc, carry_in=cin, total_out=tot)
        got = got.cpu().numpy()
        if kind == "int":
            assert np.array_equal(got, exact.astype(np.float32))
        else:
            assert_bounded(got, exact, mass, np.float32, f"carry scan {kind}")
        etot = carry + x.astype(np.float64).sum()
        A = float(ax.astype(np.float64).sum())
        if kind == "int":
            assert tot.item() == etot
        else:
            assert abs(tot.item() - etot) <= GAMMA * A + 1e-15 * abs(etot), (tot.item(), etot)


def _irreg_mass(ax, off, inclusive_scan=None):
    """A' for irregular segments: |x| mass from the start of the 64-element
    row holding each segment's first element (see module docstring)."""
    c = np.concatenate([[0.0], np.cumsum(ax.astype(np.float64))])
    a = off[:-1]
    rs = (a // 64) * 64
    if inclusive_scan is None:
        return c[off[1:]] - c[rs]
    n = ax.size
    seg = np.repeat(np.arange(off.size - 1), np.diff(off))
    i = np.arange(n)
    end = i + 1 if inclusive_scan else i
    return c[end] - c[rs[seg]]


@pytest.mark.parametrize("kind", ["int", "uniform_pm1", "mixed_mag"])
@pytest.mark.parametrize("mean", [5, 64, 1000, 50000])
def test_signed_irregular(kind, mean, data, cuda):
    x, xd = data[kind]
    rng = np.random.default_rng(mean)
    off = O.random_offsets(rng, N, mean, empty_frac=0.1)
    offd = torch.from_numpy(off).to(cuda)
    ax = np.abs(x)
    exact = O.ref_irreg_reduce(x, off)
    got = D.irreg_reduce(xd, offd, torch.float32).cpu().numpy()
    if kind == "int":
        assert np.array_equal(got, exact.astype(np.float32))
    else:
        assert_bounded(got, exact, _irreg_mass(ax, off), np.float32, f"irreg reduce {kind} {mean}")
    for exc in (False, True):
        exact = O.ref_irreg_scan(x, off, inclusive=not exc)
        got = D.irreg_scan(xd, offd, torch.float32, exclusive=exc).cpu().numpy()
        if kind == "int":
            assert np.array_equal(got, exact.astype(np.float32))
        else:
            assert_bounded(got, exact, _irreg_mass(ax, off, not exc), np.float32,
                           f"irreg scan {kind} {mean} exc={exc}")


def test_neighbour_magnitude_isolation(cuda):
    """The advisor's case: small segments next to segments of
    ~1000s.  Every small segment's sum must be accurate relative to its OWN
    mass, for fp32 and fp16 outputs, in the one-end, two-end and many-end
    GENERAL kernels."""
    rng = np.random.default_rng(5)
    for s in (17, 24, 48, 63, 65, 100, 300, 1000, 4097):
        nseg = 4096
        n = s * nseg
        big = (rng.random(n) * 1000 + 500).astype(np.float16)
        small = (rng.random(n) * 2.0 ** -6).astype(np.float16)
        x = np.where((np.arange(n) // s) % 2 == 0, big, small).astype(np.float16)
        xd = torch.from_numpy(x).to(cuda)
        exact = O.ref_seg_reduce(x, s)
        mass = O.ref_seg_reduce(np.abs(x), s)
        for dt, npdt in ((torch.float32, np.float32), (torch.float16, np.float16)):
            got = D.seg_reduce(xd, s, dt).cpu().numpy()
            idx = np.arange(nseg)
            if npdt == np.float16:
                idx = idx[np.abs(exact) < 65504]  # the large sums overflow fp16
            assert_bounded(got[idx], exact[idx], mass[idx], npdt, f"isolation s={s} {npdt.__name__}")


# ------------------------------------------------------------ non-finite data


def _poison_units(pos, n, s, op):
    """[lo, hi) of the MMA row accumulation each non-finite position feeds
    (tc_plan_info): the 64-element row, or for MODE_ROWSEG (rows of L = k s
    whole segments) the whole L-row (reduce) / its 64-column chunk (scan).
    Positions past the last full row (the ragged tail, CUDA cores) feed none."""
    mode, L = D.plan_info(op, n, s, torch.float32)
    units = set()
    for p in pos:
        r = p // L
        if (r + 1) * L > n:
            continue
        if mode == "ROWSEG" and op == "scan":
            c = (p - r * L) // 64
            units.add((r * L + 64 * c, min(r * L + 64 * c + 64, (r + 1) * L)))
        else:
            units.add((r * L, (r + 1) * L))
    return sorted(units)


def test_nonfinite_contamination_rule(cuda):
    """Documented B200 semantics for NaN / +-Inf inputs (
    the reference: engine.py:344-348 -- NaN*0 and Inf*0 in the tile MMA
    poison the whole 16-wide tile row).  Here a non-finite x[i] poisons the
    MMA row accumulation it feeds (tc_plan_info): its 64-element row, or in
    the whole-segments-per-row kernels (MODE_ROWSEG) the row of k segments
    (reduce) / the row's 64-column chunk (scan):

    * an output whose exact value involves a non-finite element is non-finite;
    * every other output is exact, or -- only inside the poison zone -- non-
      finite.  The zone: for a reduce, the segments that overlap a poisoned
      unit; for a scan, output i when a poisoned unit [lo, hi) overlaps i's
      segment and lo <= i (the unit itself, and the rest of every segment
      running through it; CTAs that re-derive their entry carry from HBM on
      CUDA cores may return the exact value instead).  An exclusive scan's
      segment-start outputs are always 0.

    (The ragged tail past the last full row is summed on CUDA cores and
    follows exact-arithmetic contamination.)"""
    rng = np.random.default_rng(11)
    n = (1 << 20) + 100
    x = rng.integers(-8, 8, n).astype(np.float16)
    bad_at = np.sort(rng.choice(n, 24, replace=False))
    x[bad_at[0::3]] = np.nan
    x[bad_at[1::3]] = np.inf
    x[bad_at[2::3]] = -np.inf
    xd = torch.from_numpy(x).to(cuda)
    nf = ~np.isfinite(x.astype(np.float32))
    clean = np.where(nf, 0, x).astype(np.float16)
    i = np.arange(n)
    nf_count = np.concatenate([[0], np.cumsum(nf)])  # non-finite elements before position j
    for s in (16, 64, 256, 3, 7, 17, 48, 300, 16384, 8192 * 3, 100001, (1 << 18) + 8192, n):
        nseg = -(-n // s)
        starts = np.arange(nseg) * s
        ends = np.minimum(starts + s, n)
        must = (nf_count[ends] - nf_count[starts]) > 0
        zone = must.copy()
        for lo, hi in _poison_units(bad_at, n, s, "reduce"):
            zone |= (starts < hi) & (ends > lo)
        got = D.seg_reduce(xd, s, torch.float32).cpu().numpy()
        exp = O.ref_seg_reduce(clean, s).astype(np.float32)
        fin = np.isfinite(got)
        assert not fin[must].any(), ("reduce: non-finite segment came back finite", s)
        assert np.array_equal(got[fin], exp[fin]), ("reduce: finite outputs exact", s)
        assert zone[~fin].all(), ("reduce: non-finite outside the zone", s)
        seg_start = (i // s) * s
        units = _poison_units(bad_at, n, s, "scan")
        for exc in (False, True):
            got = D.seg_scan(xd, s, torch.float32, exclusive=exc).cpu().numpy()
            exp = O.ref_seg_scan(clean, s, inclusive=not exc).astype(np.float32)
            upto = i + 1 if not exc else i
            must = (nf_count[upto] - nf_count[seg_start]) > 0
            pz = must.copy()
            for lo, hi in units:
                pz |= (i >= lo) & (seg_start < hi)
            fin = np.isfinite(got)
            if exc:
                assert np.all(got[i % s == 0] == 0), ("excl starts", s)
            assert not fin[must].any(), ("scan: non-finite prefix came back finite", s, exc)
            assert np.array_equal(got[fin], exp[fin]), ("scan: finite outputs exact", s, exc)
            assert pz[~fin].all(), ("scan: non-finite outside the zone", s, exc)
