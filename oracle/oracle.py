"""TEST INFRASTRUCTURE: CPU restatement of the reference's reduction/scan.

Never imported by the product.  Three layers, each citing the reference
(/root/reference/pkg/...) it restates:

1. Generators: ``exact_int_segments`` (pkg/tests/conftest.py:7-19).
2. The exact oracle: ``oracle_segmented_reduce`` / ``oracle_segmented_scan``
   (pkg/src/halftile/oracle.py:38-75) plus the padded / ragged-segment and
   memory-chunked forms the GPU parity tests need (``ref_seg_reduce``,
   ``ref_seg_scan``; padding semantics of segmented.py:57-89).
3. ``sim_*``: the reference's tile-MMA arithmetic (engine.py:326-348: exact
   binary64 dot + accumulator, ONE rounding to fp16 "half" or fp32
   "single" per MMA; fp16 narrowing in cast_kind, engine.py:430-450) for the
   reduction variants of reduce.py and the scan variants of scan.py,
   vectorised over tiles.  These reproduce halftile's outputs bit for bit
   (pinned in tests/test_oracle.py against fixtures generated from the real
   package by tests/golden/make_golden.py).
"""

from __future__ import annotations

import numpy as np

HALF = np.float16

# ---------------------------------------------------------------- generators


def exact_int_segments(rng, total_len, seg_size, cap=2048, hi=8):
    """Integers in [0, hi) with every per-segment running total <= cap
    (pkg/tests/conftest.py:7-19): all intermediates exact in binary16."""
    assert total_len % seg_size == 0
    x = rng.integers(0, hi, total_len).astype(np.float64)
    segs = x.reshape(-1, seg_size)
    running = segs.cumsum(axis=1)
    segs[running > cap] = 0
    return segs.reshape(-1).astype(np.float16)


# --------------------------------------------------------------- exact oracle


def _segments(values, seg_size):
    """oracle.py:38-44: length must be a segment multiple."""
    values = np.asarray(values)
    if seg_size < 1 or values.size % seg_size:
        raise ValueError(f"length {values.size} is not a multiple of segment size {seg_size}")
    return values.reshape(-1, seg_size)


def oracle_segmented_reduce(values, seg_size, mode="exact"):
    """oracle.py:47-57: binary64 sums ("exact") or strict left-to-right
    binary16 sums ("faithful_half")."""
    segs = _segments(values, seg_size)
    if mode == "exact":
        return segs.astype(np.float64).sum(axis=1)
    if mode == "faithful_half":
        return np.cumsum(segs.astype(HALF), axis=1)[:, -1]
    raise ValueError(f"unknown oracle mode {mode!r}")


def oracle_segmented_scan(values, seg_size, mode="exact", inclusive=True):
    """oracle.py:60-75: per-segment prefix sums; exclusive = shift right
    within each segment with a leading zero."""
    segs = _segments(values, seg_size)
    if mode == "exact":
        out = np.cumsum(segs.astype(np.float64), axis=1)
    elif mode == "faithful_half":
        out = np.cumsum(segs.astype(HALF), axis=1)
    else:
        raise ValueError(f"unknown oracle mode {mode!r}")
    if not inclusive:
        shifted = np.zeros_like(out)
        shifted[:, 1:] = out[:, :-1]
        out = shifted
    return out.reshape(-1)


_CHUNK = 1 << 24  # elements per chunk for memory-bounded oracle runs


def ref_seg_reduce(values, seg_size):
    """Exact binary64 sums of ceil(n/s) segments, the last one ragged
    (pad_segmented zero padding, segmented.py:57-89 + unpad_sums :53-54).
    Chunked by whole segments so 2^30-element inputs stay memory-bounded."""
    x = np.asarray(values)
    n = x.size
    s = int(seg_size)
    nseg = -(-n // s)
    out = np.empty(nseg, dtype=np.float64)
    if s >= _CHUNK:
        for k in range(nseg):
            lo, hi = k * s, min((k + 1) * s, n)
            acc = 0.0
            for c in range(lo, hi, _CHUNK):
                acc += x[c:min(c + _CHUNK, hi)].astype(np.float64).sum()
            out[k] = acc
        return out
    per = max(1, _CHUNK // s)
    full = n // s
    for k0 in range(0, full, per):
        k1 = min(full, k0 + per)
        out[k0:k1] = x[k0 * s:k1 * s].astype(np.float64).reshape(k1 - k0, s).sum(axis=1)
    if full < nseg:
        out[full] = x[full * s:].astype(np.float64).sum()
    return out


def ref_seg_scan(values, seg_size, inclusive=True, carry=None):
    """Exact binary64 segmented prefix sums, n outputs (ragged last segment
    allowed), memory-bounded.  ``carry`` continues segment 0 from an earlier
    shard.  Exclusive = the reference's shift-right-inject-zero
    (scan.py:332-341); with a carry the first output is the carry.

    Small segments: whole segments per chunk.  Large segments: carry-first
    ``np.cumsum(np.r_[run, chunk])`` per chunk, which is bit-identical to one
    sequential cumsum (np.add.accumulate runs left to right)."""
    x = np.asarray(values)
    n = x.size
    s = int(seg_size)
    out = np.empty(n, dtype=np.float64)
    if s < _CHUNK:
        per = max(1, _CHUNK // s)
        nseg = -(-n // s)
        for k0 in range(0, nseg, per):
            k1 = min(nseg, k0 + per)
            lo, hi = k0 * s, min(k1 * s, n)
            out[lo:hi] = ref_seg_scan_exact(x[lo:hi], s, inclusive, carry if k0 == 0 else None)
        return out
    run = 0.0 if carry is None else float(carry)
    lo = 0
    while lo < n:
        hi = min(n, lo + _CHUNK)
        nb = ((lo // s) + 1) * s  # next segment boundary
        if nb < hi:
            hi = nb
        if lo % s == 0 and not (lo == 0 and carry is not None):
            run = 0.0
        chunk = x[lo:hi].astype(np.float64)
        incl = np.cumsum(np.concatenate([[run], chunk]))[1:]
        if inclusive:
            out[lo:hi] = incl
        else:
            out[lo:hi] = np.concatenate([[run], incl[:-1]])
        run = incl[-1]
        lo = hi
    return out


def ref_seg_scan_exact(values, seg_size, inclusive=True, carry=None):
    """Per-segment np.cumsum (no subtraction anywhere): the direct
    restatement of oracle.py:60-75 for ragged inputs; use for modest n."""
    x = np.asarray(values).astype(np.float64)
    n = x.size
    s = int(seg_size)
    nseg = -(-n // s)
    pad = np.zeros(nseg * s)
    pad[:n] = x
    segs = pad.reshape(nseg, s)
    if carry is not None:
        segs = segs.copy()
        segs[0, 0] += float(carry)
    c = np.cumsum(segs, axis=1)
    if not inclusive:
        e = np.zeros_like(c)
        e[:, 1:] = c[:, :-1]
        if carry is not None:
            e[0, 0] = float(carry)
        c = e
    return c.reshape(-1)[:n]


# ----------------------------------------- irregular (CSR-offset) segments
# Extension: the reference has no irregular entry
# point (the paper elides it), so these restate the exact
# oracle (oracle.py:47-75: binary64 per-segment sums / prefix sums) for
# segments values[offsets[k]:offsets[k+1]].


def random_offsets(rng, n, mean_len, empty_frac=0.0):
    """nseg + 1 non-decreasing offsets over [0, n]: segment lengths
    geometric with the given mean, a fraction of them forced empty."""
    lens = rng.geometric(1.0 / max(1.0, float(mean_len)), size=max(4, 2 * n // max(1, int(mean_len)) + 8))
    if empty_frac > 0:
        lens[rng.random(lens.size) < empty_frac] = 0
    ends = np.cumsum(lens)
    ends = ends[ends < n]
    off = np.concatenate([[0], ends, [n]]).astype(np.int64)
    return off


def ref_irreg_reduce(values, offsets):
    """Exact binary64 sums of values[offsets[k]:offsets[k+1]] (0 if empty)."""
    x = np.asarray(values).astype(np.float64)
    off = np.asarray(offsets, dtype=np.int64)
    out = np.zeros(off.size - 1, dtype=np.float64)
    ne = off[1:] > off[:-1]
    if ne.any():
        out[ne] = np.add.reduceat(x, off[:-1][ne])
    return out


def ref_irreg_scan(values, offsets, inclusive=True):
    """Per-segment prefix sums (exclusive: 0 at each segment start), from an
    extended-precision running sum (np.longdouble: the subtraction of the
    segment base costs < 2^-60 relative, far below any tolerance used)."""
    x = np.asarray(values).astype(np.longdouble)
    off = np.asarray(offsets, dtype=np.int64)
    n = x.size
    c = np.cumsum(x)
    seg = np.searchsorted(off, np.arange(n), side="right") - 1
    st = off[seg]
    base = np.where(st > 0, c[np.maximum(st - 1, 0)], 0)
    incl = c - base
    if inclusive:
        return incl.astype(np.float64)
    ex = np.empty_like(incl)
    ex[1:] = incl[:-1]
    ex[0] = 0
    ex[np.arange(n) == st] = 0
    return ex.astype(np.float64)


# ------------------------------------------------ batch-norm statistics
# Extension: the paper's TCU-reduction consumer
# (mu_B = mean of the mini-batch per channel, sigma_B^2 =
# mean of (x - mu_B)^2), restated in binary64 for an (N, C, *spatial) array.


def ref_bn_stats(x):
    a = np.asarray(x).astype(np.float64)
    a = a.reshape(a.shape[0], a.shape[1], -1)
    mean = a.mean(axis=(0, 2))
    var = ((a - mean[None, :, None]) ** 2).mean(axis=(0, 2))
    return mean, var


# ------------------------------------------------ tile-engine arithmetic (sim)


def _adt(acc):
    return np.float16 if acc == "half" else np.float32


def _R(x, acc):
    """One rounding of a binary64 value to the accumulator dtype (engine.py:347-348)."""
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float64).astype(_adt(acc)).astype(np.float64)


def _h(x):
    """fp16 narrowing (cast_kind / matrix load, engine.py:281-283, :450)."""
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float64).astype(HALF).astype(np.float64)


def _pad(values, seg_size, seg_multiple=16, count_multiple=1):
    """pad_segmented (segmented.py:57-89) -> (data float64, padded seg, n_logical_segs)."""
    v = np.ascontiguousarray(values, dtype=HALF)
    padded_seg = -(-seg_size // seg_multiple) * seg_multiple
    n_logical = -(-v.size // seg_size)
    n_segs = -(-n_logical // count_multiple) * count_multiple
    out = np.zeros((n_segs, padded_seg), dtype=HALF)
    full = v.size // seg_size
    if full:
        out[:full, :seg_size] = v[: full * seg_size].reshape(full, seg_size)
    rem = v.size - full * seg_size
    if rem:
        out[full, :rem] = v[full * seg_size:]
    return out.reshape(-1).astype(np.float64), padded_seg, n_logical


def _colsums(chunks):
    """Column sums of col-major 16x16 tiles: (..., 256) -> (..., 16) exact."""
    return chunks.reshape(chunks.shape[:-1] + (16, 16)).sum(axis=-1)


def sim_reduce_16(x, acc="half"):
    """reduce.py:92-106: one MMA, column sums of a col-major tile."""
    return _R(np.asarray(x, np.float64).reshape(-1, 16).sum(axis=1), acc)


def sim_reduce_256n_efficient(x, acc="half"):
    """reduce.py:123-141 over a batch of segments (rows of x, length 256n)."""
    x = np.atleast_2d(np.asarray(x, np.float64))
    n = x.shape[1] // 256
    cs = _colsums(x.reshape(x.shape[0], n, 256))  # (S, n, 16)
    v = np.zeros((x.shape[0], 16))
    for i in range(n):
        v = _R(v + cs[:, i], acc)
    row = _h(v)
    return _R(row.sum(axis=1), acc)


def sim_reduce_256n_inefficient(x, acc="half"):
    """reduce.py:144-168."""
    x = np.atleast_2d(np.asarray(x, np.float64))
    n = x.shape[1] // 256
    cs = _colsums(x.reshape(x.shape[0], n, 256))
    carry = np.zeros(x.shape[0])
    r = carry
    for i in range(n):
        v = _R(cs[:, i], acc)
        row = _h(v)
        r = _R(row.sum(axis=1) + carry, acc)
        carry = r
    return r


def sim_reduce_256(x, acc="half"):
    """reduce.py:109-120 (two MMAs)."""
    return sim_reduce_256n_efficient(np.asarray(x, np.float64).reshape(-1, 256), acc)


def sim_reduce_16n_strided(data, seg, acc="half"):
    """reduce.py:171-198: per segment, n accumulating MMAs over 16-blocks."""
    segs = np.asarray(data, np.float64).reshape(-1, seg // 16, 16).sum(axis=2)  # (S, n)
    v = np.zeros(segs.shape[0])
    for i in range(segs.shape[1]):
        v = _R(v + segs[:, i], acc)
    return v


def sim_reduce_16n_coalesced(data, seg, acc="half"):
    """reduce.py:201-256."""
    segs = np.asarray(data, np.float64).reshape(-1, seg)
    n = seg // 16
    num_full, tail16 = n // 16, n % 16
    tails = None
    if tail16:
        t = segs[:, 256 * num_full:].reshape(segs.shape[0], tail16, 16).sum(axis=2)
        tails = np.zeros(segs.shape[0])
        for i in range(tail16):
            tails = _R(tails + t[:, i], acc)
    if not num_full:
        return tails
    cs = _colsums(segs[:, : 256 * num_full].reshape(segs.shape[0], num_full, 256))
    v = np.zeros((segs.shape[0], 16))
    for i in range(num_full):
        v = _R(v + cs[:, i], acc)
    row = _h(v)
    seed = tails if tails is not None else 0.0
    return _R(row.sum(axis=1) + seed, acc)


def clamp_wpb(wpb, n_tiles):
    """clamp_block_config (reduce.py:267-272)."""
    w = min(wpb, n_tiles)
    while n_tiles % w:
        w -= 1
    return w


def sim_block_reduce_256n(x, wpb, acc="half"):
    """reduce.py:278-326 over a batch of segments (rows)."""
    x = np.atleast_2d(np.asarray(x, np.float64))
    S, L = x.shape
    per = L // wpb
    parts = sim_reduce_256n_efficient(x.reshape(S * wpb, per), acc).reshape(S, wpb)
    return _R(_h(parts).sum(axis=1), acc)


def sim_grid_reduce(values, acc="half", wpb=4, block_elems=4096):
    """reduce.py:332-373: blocks of block_elems -> partials -> fp16 ->
    work-efficient pass 2."""
    data, _, _ = _pad(values, block_elems, seg_multiple=block_elems)
    blocks = data.reshape(-1, block_elems)
    partials = sim_block_reduce_256n(blocks, wpb, acc)
    pp, _, _ = _pad(_h(partials).astype(HALF), partials.size, seg_multiple=256)
    return sim_reduce_256n_efficient(pp.reshape(1, -1), acc)[0]


def sim_segmented_reduce(values, seg, variant, acc="half", wpb=4):
    """reduce.py:379-446 (values as the reference returns them, float64)."""
    v = np.ascontiguousarray(values, dtype=HALF)
    if variant == "grid":
        return np.array([sim_grid_reduce(v, acc, wpb)])
    if variant == "warp16":
        d, _, nl = _pad(v, 16, 16, 16)
        return sim_reduce_16(d, acc)[:nl]
    if variant == "warp256":
        d, _, nl = _pad(v, 256, 256)
        return sim_reduce_256(d, acc)[:nl]
    if variant in ("strided16n", "coalesced16n"):
        d, ps, nl = _pad(v, seg, 16, 16)
        fn = sim_reduce_16n_strided if variant == "strided16n" else sim_reduce_16n_coalesced
        return fn(d, ps, acc)[:nl]
    if variant in ("efficient256n", "inefficient256n"):
        d, ps, nl = _pad(v, seg, 256)
        fn = sim_reduce_256n_efficient if variant == "efficient256n" else sim_reduce_256n_inefficient
        return fn(d.reshape(-1, ps), acc)[:nl]
    if variant == "block256n":
        d, ps, nl = _pad(v, seg, 256)
        w = clamp_wpb(wpb, ps // 256)
        return sim_block_reduce_256n(d.reshape(-1, ps), w, acc)[:nl]
    raise ValueError(variant)


# -------------------------------------------------------------- scans (sim)


def _scan_tiles(t, carry, acc):
    """_ScanTiles.scan_tile (scan.py:83-91) on a batch of row-major tiles
    t[..., 16, 16] with per-tile scalar carries."""
    row_scans = _R(np.cumsum(t, axis=-1) + carry[..., None, None], acc)
    col_excl = np.zeros_like(t)
    col_excl[..., 1:, :] = np.cumsum(t, axis=-2)[..., :-1, :]
    rows_before = _h(_R(col_excl, acc))
    return _R(rows_before.sum(axis=-1, keepdims=True) + row_scans, acc)


def sim_scan_16(x, acc="half"):
    """scan.py:58-71: one MMA per row of 16."""
    return _R(np.cumsum(np.asarray(x, np.float64).reshape(-1, 16), axis=1), acc).reshape(-1)


def sim_scan_256n(x, acc="half"):
    """scan.py:102-119 over a batch of segments (rows of length 256n)."""
    x = np.atleast_2d(np.asarray(x, np.float64))
    S, L = x.shape
    n = L // 256
    tiles = x.reshape(S, n, 16, 16)
    out = np.empty_like(tiles)
    carry = np.zeros(S)
    for i in range(n):
        r = _scan_tiles(tiles[:, i], carry, acc)
        out[:, i] = r
        carry = r[:, 15, 15]
    return out.reshape(S, L)


def sim_scan_16n(data, seg, acc="half"):
    """scan.py:122-152: strided row scans, carry = last column."""
    segs = np.asarray(data, np.float64).reshape(-1, seg // 16, 16)  # (S, n, 16)
    out = np.empty_like(segs)
    carry = np.zeros(segs.shape[0])
    for i in range(segs.shape[1]):
        r = _R(np.cumsum(segs[:, i], axis=1) + carry[:, None], acc)
        out[:, i] = r
        carry = r[:, 15]
    return out.reshape(-1)


def sim_block_scan_256n(x, wpb, acc="half"):
    """scan.py:178-243 for one segment (1-D, length 256n)."""
    adt = _adt(acc)
    x = np.asarray(x, np.float64)
    n = x.size // 256
    out = np.zeros(x.size, dtype=adt)
    carry = adt(0)
    for i0 in range(0, n, wpb):
        tiles = x[256 * i0:256 * (i0 + wpb)].reshape(wpb, 16, 16)
        r = _scan_tiles(tiles, np.zeros(wpb), acc)  # unseeded warp scans into sout
        sout = np.zeros(256 * 16, dtype=adt)
        sout[: 256 * wpb] = r.reshape(-1).astype(adt)
        # last_column_scan_16 over the last rows (offset 240, ld 256), fp16 load
        e_last = _h(sout.astype(np.float64)[240::256][:16] if False else
                    np.array([sout[240 + 256 * k + 15] for k in range(16)], dtype=np.float64))
        col = e_last
        prtls = _R(np.concatenate([[0.0], np.cumsum(col)[:-1]]) + float(carry), acc).astype(adt)
        tail_total = adt(e_last[15])
        for w in range(wpb):
            base = 256 * (i0 + w)
            out[base:base + 256] = sout[256 * w:256 * w + 256] + prtls[w]
        carry = adt(prtls[15] + adt(tail_total))
    return out.astype(np.float64)


def sim_grid_scan(values, acc="half", wpb=4, block_elems=4096):
    """scan.py:249-310: block scans, scan of fp16 totals, uniform add."""
    adt = _adt(acc)
    v = np.ascontiguousarray(values, dtype=HALF)
    data, _, _ = _pad(v, block_elems, seg_multiple=block_elems)
    nb = data.size // block_elems
    inter = np.zeros(data.size, dtype=adt)
    totals = np.zeros(nb, dtype=adt)
    for b in range(nb):
        blk = sim_block_scan_256n(data[b * block_elems:(b + 1) * block_elems], wpb, acc)
        inter[b * block_elems:(b + 1) * block_elems] = blk.astype(adt)
        totals[b] = inter[(b + 1) * block_elems - 1]
    tp, _, _ = _pad(totals.astype(HALF), nb, seg_multiple=256)
    ts = sim_scan_256n(tp.reshape(1, -1), acc).reshape(-1).astype(adt)
    offsets = np.zeros(nb, dtype=adt)
    offsets[1:] = ts[: nb - 1]
    for b in range(nb):
        lo, hi = b * block_elems, (b + 1) * block_elems
        inter[lo:hi] = inter[lo:hi] + offsets[b]
    return inter[: v.size].astype(np.float64)


def _unpad_scan(scanned, ps, seg, n):
    segs = np.asarray(scanned).reshape(-1, ps)
    nl = -(-n // seg)
    return segs[:nl, :seg].reshape(-1)[:n]


def sim_segmented_scan(values, seg, variant, acc="half", wpb=4, inclusive=True):
    """scan.py:316-388 (float64 view of the reference's outputs)."""
    v = np.ascontiguousarray(values, dtype=HALF)
    n = v.size
    if variant == "grid":
        out = sim_grid_scan(v, acc, wpb)
    elif variant == "warp16":
        d, ps, _ = _pad(v, 16, 16, 16)
        out = _unpad_scan(sim_scan_16(d, acc), ps, 16, n)
    elif variant == "warp256":
        d, ps, _ = _pad(v, 256, 256)
        out = _unpad_scan(sim_scan_256n(d.reshape(-1, 256), acc), ps, 256, n)
    elif variant == "strided16n":
        d, ps, _ = _pad(v, seg, 16, 16)
        out = _unpad_scan(sim_scan_16n(d, ps, acc), ps, seg, n)
    elif variant == "warp256n":
        d, ps, _ = _pad(v, seg, 256)
        out = _unpad_scan(sim_scan_256n(d.reshape(-1, ps), acc), ps, seg, n)
    elif variant == "block256n":
        d, ps, _ = _pad(v, seg, 256)
        w = clamp_wpb(wpb, ps // 256)
        rows = d.reshape(-1, ps)
        out = _unpad_scan(np.concatenate([sim_block_scan_256n(r, w, acc) for r in rows]), ps, seg, n)
    else:
        raise ValueError(variant)
    if not inclusive:
        segs = np.asarray(out).reshape(-1, seg)
        sh = np.zeros_like(segs)
        sh[:, 1:] = segs[:, :-1]
        out = sh.reshape(-1)
    return out
