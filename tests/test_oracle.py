"""The oracle is pinned before it is trusted (CPU only).

* The exact oracle restatement reproduces the reference's exact oracle
  outputs (pkg/src/halftile/oracle.py:47-75 through pad_segmented, as
  cli._check_against_oracle does) bit for bit on every golden case.
* The tile-engine restatement (oracle.sim_*) reproduces the reference
  simulator's own outputs bit for bit -- half AND single accumulate,
  integer AND non-integer data, ragged lengths -- on every golden case.
* The reference's known-answer tests hold.
* The multi-threaded C restatement (oracle/oracle.c) agrees with numpy.
Golden fixtures: tests/golden/make_golden.py (imports the real reference).
"""

import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

ROOT = Path(__file__).resolve().parent.parent


def _x(z, k):
    return z[f"x{k}"].view(np.float16)


def test_golden_exact_oracle_bit_exact(golden):
    z, meta = golden
    for case in meta["manifest"]:
        k, op, seg, x = case["id"], case["op"], case["seg"], _x(z, case["id"])
        s = x.size if case["variant"] == "grid" else seg
        if op == "reduce":
            got = O.ref_seg_reduce(x, s)
        else:
            got = O.ref_seg_scan(x, s, inclusive=case["inclusive"])
        exp = z[f"exact{k}"]
        assert got.shape == exp.shape and np.array_equal(got, exp), case


@pytest.mark.parametrize("acc", ["half", "single"])
def test_golden_simulator_restatement_bit_exact(golden, acc):
    z, meta = golden
    for case in meta["manifest"]:
        k, op, seg, v, x = case["id"], case["op"], case["seg"], case["variant"], _x(z, case["id"])
        if op == "reduce":
            got = O.sim_segmented_reduce(x, seg, v, acc)
        else:
            got = O.sim_segmented_scan(x, x.size if v == "grid" else seg, v, acc,
                                       inclusive=case["inclusive"])
        exp = z[f"sim_{acc}{k}"]
        assert got.shape == exp.shape, case
        assert np.array_equal(got, exp, equal_nan=True), case


def test_golden_exact_int_cases_agree_across_oracles(golden):
    """On exact-integer data the simulator equals fp16(exact): the two
    reference legs agree, which is what makes bit-exact GPU parity
    meaningful."""
    z, meta = golden
    for case in meta["manifest"]:
        if "int" not in case["kind"]:
            continue
        k = case["id"]
        e16 = z[f"exact{k}"].astype(np.float16).astype(np.float64)
        assert np.array_equal(z[f"sim_half{k}"], e16), case
        assert np.array_equal(z[f"sim_single{k}"], z[f"exact{k}"]), case


def test_known_answers(golden):
    z, meta = golden
    k = {n: (z[f"kat_x_{n}"].view(np.float16), z[f"kat_y_{n}"]) for n in meta["kats"]}
    x, y = k["reduce_16_arange"]
    assert y[0] == 136.0 and y[1] == 392.0  # pkg/tests/test_reduce.py:40-47
    assert np.array_equal(y, O.ref_seg_reduce(x, 16).astype(np.float16).astype(np.float64))
    assert k["reduce_256_zeros"][1].tolist() == [0.0]
    assert k["reduce_256_ones"][1].tolist() == [256.0]
    assert k["reduce_256_halves"][1].tolist() == [128.0]
    assert k["efficient_1024_ones"][1].tolist() == [1024.0]
    assert k["strided_512_ones_seg32"][1].tolist() == [32.0] * 16
    assert k["coalesced_seg512_ones"][1].tolist() == [512.0] * 16
    assert k["grid_1024_ones"][1].tolist() == [1024.0]
    assert k["grid_100_ones"][1].tolist() == [100.0]
    assert k["scan_256_ones"][1].tolist() == list(range(1, 257))
    assert k["scan_16_ones"][1].reshape(16, 16).tolist() == [list(range(1, 17))] * 16
    assert k["scan_256n_512_ones"][1].tolist() == list(range(1, 513))
    for name, (x, y) in k.items():
        # every KAT equals the exact oracle rounded once to fp16
        if name.startswith("reduce_16") or name.startswith("strided") or name.startswith("coalesced"):
            seg = {"reduce_16_arange": 16, "strided_512_ones_seg32": 32, "coalesced_seg512_ones": 512}[name]
            assert np.array_equal(y, O.ref_seg_reduce(x, seg).astype(np.float16).astype(np.float64))
        if name.startswith("scan") or name.startswith("block_scan") or name.startswith("grid_scan"):
            seg = {"scan_16_ones": 16, "scan_16n_512_ones_seg32": 32}.get(name, x.size)
            assert np.array_equal(y, O.ref_seg_scan(x, seg).astype(np.float16).astype(np.float64)), name
    # last_column_scan_16 (pkg/tests/test_scan.py:183-199)
    assert z["lcs_y_ones"].tolist() == list(range(16))
    assert z["lcs_y_ones_carry5"].tolist() == [5 + i for i in range(16)]
    assert z["lcs_y_seq"].tolist() == np.concatenate([[0], np.arange(1, 16).cumsum()]).tolist()


def test_reference_oracle_closed_forms():
    # pkg/tests/test_oracle.py:34-38: faithful-half loses, exact does not
    x = np.array([2048, 1, 1, 1], np.float16)
    assert O.oracle_segmented_reduce(x, 4)[0] == 2051.0
    assert O.oracle_segmented_reduce(x, 4, "faithful_half")[0] == 2048.0
    with pytest.raises(ValueError):
        O.oracle_segmented_reduce(np.ones(10, np.float16), 4)


def test_exact_int_generator_bounds(rng):
    x = O.exact_int_segments(rng, 1 << 16, 256)
    segs = x.astype(np.float64).reshape(-1, 256)
    assert segs.min() >= 0 and segs.max() < 8
    assert segs.cumsum(axis=1).max() <= 2048


def test_chunked_oracle_matches_direct(rng):
    saved = O._CHUNK
    try:
        O._CHUNK = 64
        for n, s in [(1000, 100), (1000, 16), (999, 1000), (5000, 333), (4096, 4096)]:
            x = rng.integers(0, 8, n).astype(np.float16)
            for inc in (True, False):
                for c in (None, 2.5):
                    assert np.array_equal(O.ref_seg_scan(x, s, inc, c),
                                          O.ref_seg_scan_exact(x, s, inc, c))
            assert np.array_equal(O.ref_seg_reduce(x, s),
                                  O.ref_seg_scan_exact(x, s)[np.minimum(np.arange(s - 1, n + s - 1, s), n - 1)])
    finally:
        O._CHUNK = saved


@pytest.fixture(scope="module")
def liboracle():
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    lib = ctypes.CDLL(str(ROOT / "oracle" / "build" / "liboracle.so"))
    P = ctypes.c_void_p
    lib.or_seg_reduce.argtypes = [P, ctypes.c_int64, ctypes.c_int64, P, ctypes.c_int]
    lib.or_seg_scan.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                ctypes.c_int, P, ctypes.c_int]
    lib.or_f16_to_f64.restype = ctypes.c_double
    lib.or_f16_to_f64.argtypes = [ctypes.c_uint16]
    return lib


def test_c_oracle_binary16_decode_exhaustive(liboracle):
    bits = np.arange(1 << 16, dtype=np.uint16)
    ref = bits.view(np.float16).astype(np.float64)
    got = np.array([liboracle.or_f16_to_f64(int(b)) for b in bits[::97]])
    assert np.array_equal(got, ref[::97], equal_nan=True)


@pytest.mark.parametrize("n,s", [(100000, 16), (100000, 300), (1 << 20, 1 << 20), (123457, 4096),
                                 (1 << 20, 1000), (5000, 100000)])
def test_c_oracle_matches_numpy(liboracle, rng, n, s):
    for kind in ("int", "uniform"):
        x = (rng.integers(0, 8, n) if kind == "int" else rng.random(n)).astype(np.float16)
        o = np.empty(-(-n // s))
        liboracle.or_seg_reduce(x.ctypes.data, n, s, o.ctypes.data, 8)
        r = O.ref_seg_reduce(x, s)
        assert np.array_equal(o, r) if kind == "int" else np.allclose(o, r, rtol=1e-14, atol=0)
        for inc in (1, 0):
            for hc, c in ((0, 0.0), (1, 3.5)):
                o = np.empty(n)
                liboracle.or_seg_scan(x.ctypes.data, n, s, inc, c, hc, o.ctypes.data, 8)
                r = O.ref_seg_scan(x, s, bool(inc), c if hc else None)
                assert np.array_equal(o, r) if kind == "int" else np.allclose(o, r, rtol=1e-13)


def test_irregular_oracle_against_direct_loops():
    """The irregular oracle (extension, no reference fixture exists: the
    paper elides irregular segments) against per-segment
    binary64 loops -- the definition restated directly."""
    rng = np.random.default_rng(3)
    for n, mean, ef in ((1, 1, 0.0), (1000, 1, 0.5), (5000, 37, 0.2), (20000, 3000, 0.0)):
        x = rng.random(n).astype(np.float16)
        off = O.random_offsets(rng, n, mean, ef)
        assert off[0] == 0 and off[-1] == n and np.all(np.diff(off) >= 0)
        xs = x.astype(np.float64)
        r = O.ref_irreg_reduce(x, off)
        s = O.ref_irreg_scan(x, off)
        e = O.ref_irreg_scan(x, off, inclusive=False)
        for k in range(off.size - 1):
            a, b = off[k], off[k + 1]
            assert r[k] == pytest.approx(xs[a:b].sum(), rel=1e-15, abs=0)
            c = np.cumsum(xs[a:b])
            assert np.allclose(s[a:b], c, rtol=1e-14, atol=0)
            if b > a:
                assert e[a] == 0 and np.allclose(e[a + 1:b], c[:-1], rtol=1e-14, atol=0)


def test_bn_oracle_definition():
    """ref_bn_stats restates PAPER.md:2195-2203 (mu_B, sigma_B^2 per channel)."""
    rng = np.random.default_rng(0)
    x = rng.random((3, 4, 5, 6))
    m, v = O.ref_bn_stats(x)
    for c in range(4):
        vals = x[:, c].reshape(-1)
        assert m[c] == pytest.approx(vals.mean(), rel=1e-14)
        assert v[c] == pytest.approx(((vals - vals.mean()) ** 2).mean(), rel=1e-12)


# ------------------------------------------- tolerance checkers (oracle/clib)


def _np_bound(exact, A, dt, ulps, gamma):
    a = np.abs(exact)
    if dt == np.float16:
        e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
        ulp = np.where((a > 0) & (e >= -14), 2.0 ** (e - 10), 2.0 ** -24)
    else:
        e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
        ulp = np.where((a > 0) & (e >= -126), 2.0 ** (e - 23), 2.0 ** -149)
    return ulps * ulp + gamma * A


@pytest.mark.parametrize("s", [1, 7, 64, 300, 5000, 100000])
def test_clib_reduce_checker_matches_numpy(s):
    from oracle import clib

    rng = np.random.default_rng(s)
    n = 50000
    x = (rng.random(n) * 2 - 1).astype(np.float16)
    exact = O.ref_seg_reduce(x, s)
    A = O.ref_seg_reduce(np.abs(x), s)
    assert np.allclose(clib.seg_reduce(x, s), exact, rtol=1e-14, atol=1e-300)
    for dt in (np.float16, np.float32):
        got = exact.astype(dt)
        c = clib.check_seg_reduce(x, s, got, 1.0, 0.0)
        assert c.bad == 0 and c.max_ratio <= 1.0, c
        # a perturbation of 2 bounds is caught at the right place
        bad = got.copy()
        k = bad.size // 2
        b = _np_bound(exact, A, dt, 1.0, 1e-6)
        bad[k] = dt(exact[k] + 4 * b[k] + (2.0 ** -10 if dt == np.float16 else 1e-5) * abs(exact[k]))
        c = clib.check_seg_reduce(x, s, bad, 1.0, 1e-6)
        assert c.bad == 1 and c.first_bad == k, c
        nan = got.copy()
        nan[0] = np.nan
        assert clib.check_seg_reduce(x, s, nan, 1.0, 1e-6).first_bad == 0


@pytest.mark.parametrize("s,carry", [(16, None), (300, None), (100000, None), (100000, 2.5)])
def test_clib_scan_checker_chunked(s, carry):
    from oracle import clib

    rng = np.random.default_rng(1)
    n = 123457
    x = (rng.random(n) * 2 - 1).astype(np.float16)
    for inc in (True, False):
        exact = O.ref_seg_scan(x, s, inc, carry)
        got = exact.astype(np.float32)
        ch = clib.ScanChecker(x, s, inc, carry)
        for lo in range(0, n, 40000):
            ch.check(lo, got[lo:lo + 40000], 1.0, 0.0)
        assert ch.bad == 0 and ch.max_ratio <= 1.0, ch
        if inc:
            assert ch.exact_total == pytest.approx(exact[-1], rel=1e-13, abs=1e-13)
        bad = got.copy()
        bad[77777] += 1.0
        ch = clib.ScanChecker(x, s, inc, carry)
        ch.check(0, bad, 1.0, 1e-7)
        assert ch.bad == 1 and ch.first_bad == 77777, ch
