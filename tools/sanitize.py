"""Small invocation of every kernel mode, for compute-sanitizer.

usage: compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck \
           python tools/sanitize.py [quick|full] [reduce,scan,chunk,irreg,bn]

Each case runs once at a small size on exact-integer data and is checked
bit-for-bit against the oracle, so a sanitizer run is also a parity run.
Modes covered (tc_collectives.cu MODE_*): LOCAL, ROWS, TILES, GENERAL
(incl. the ragged last segment and the cross-CTA last-CTA fixup), GSCR,
CHUNK (cooperative launch, one and several granules per row, carry-in /
total-out), IRREG reduce / scan (tail pre-pass), batch-norm statistics.
"""

import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (checker only)
from paper_1811_09736_b200 import _device as D  # noqa: E402


def main():
    quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
    parts = set((sys.argv[2] if len(sys.argv) > 2 else "reduce,scan,chunk,irreg,bn").split(","))
    rng = np.random.default_rng(7)
    dev = torch.device("cuda", 0)
    n = (1 << 18) + 77 if quick else (1 << 20) + 4097
    x = rng.integers(-4, 5, n).astype(np.float16)
    xd = torch.from_numpy(x).to(dev)
    done = []
    if "reduce" in parts:
        run_reduce(x, xd, n, done)
    if "scan" in parts:
        run_scan(x, xd, n, done)
    if "chunk" in parts:
        run_chunk(x, xd, n, dev, done)
    if "irreg" in parts:
        run_irreg(x, xd, n, rng, dev, done)
    if "bn" in parts:
        run_bn(rng, dev, done)
    torch.cuda.synchronize()
    print("sanitize cases ok:", "; ".join(done))


def run_reduce(x, xd, n, done):
    # reduce: LOCAL 16, ROWS 256, TILES 16384 (fixup: 8192*3), GENERAL 300 / 48 / 100, GSCR 17 / 3,
    # SPLIT 16411 / 100001 (split granule from the held SMEM stage, cross-CTA fixup)
    for s in (16, 256, 16384, 8192 * 3, 300, 48, 100, 17, 3, 1000, 16411, 100001, n):
        for dt, npdt in ((torch.float16, np.float16), (torch.float32, np.float32),
                         (torch.float64, np.float64)):
            got = D.seg_reduce(xd, s, dt).cpu().numpy()
            exp = O.ref_seg_reduce(x, s).astype(npdt)
            assert np.array_equal(got, exp), ("reduce", s, dt)
        done.append(f"reduce s={s}")


def run_scan(x, xd, n, done):
    # scan: LOCAL, ROWS, TILES, GENERAL (48, 1000), SPLIT (300, 65, 4097: the
    # epilogue-held SMEM stage), SPLITM (33, fp32 out), ROWSEG (3; 17 with fp16 out)
    for s in (16, 256, 16384, 300, 48, 3, 1000, 65, 4097, 33):
        for exc in (False, True):
            got = D.seg_scan(xd, s, torch.float32, exclusive=exc).cpu().numpy()
            exp = O.ref_seg_scan(x, s, inclusive=not exc).astype(np.float32)
            assert np.array_equal(got, exp), ("scan", s, exc)
        done.append(f"scan s={s}")
    for s in (17, 65):
        got = D.seg_scan(xd, s, torch.float16).cpu().numpy()
        assert np.array_equal(got, O.ref_seg_scan(x, s).astype(np.float16)), ("scan f16", s)
        done.append(f"scan s={s} fp16")


def run_chunk(x, xd, n, dev, done):
    for s in ((1 << 18) + 64, n):
        got = D.seg_scan(xd, s, torch.float32).cpu().numpy()
        assert np.array_equal(got, O.ref_seg_scan(x, s).astype(np.float32)), ("chunk", s)
    cin = torch.tensor([5.0], dtype=torch.float64, device=dev)
    tot = torch.zeros(1, dtype=torch.float64, device=dev)
    got = D.seg_scan(xd, n, torch.float32, carry_in=cin, total_out=tot).cpu().numpy()
    exp = O.ref_seg_scan(x, n, carry=5.0).astype(np.float32)
    assert np.array_equal(got, exp), "carry-in scan"
    assert float(tot) == 5.0 + float(x.astype(np.float64).sum()), "total_out"
    done.append("scan carry_in/total_out (CHUNK)")
    # CHUNK with several granules per row: s > 2^18 and not a multiple of 64
    s = (1 << 18) + 100
    got = D.seg_scan(xd, s, torch.float16).cpu().numpy()
    assert np.array_equal(got, O.ref_seg_scan(x, s).astype(np.float16)), "chunk gr>1"
    done.append(f"scan s={s} (CHUNK, GR=16)")


def run_irreg(x, xd, n, rng, dev, done):
    # irregular segments
    off = O.random_offsets(rng, n, 50, empty_frac=0.1)
    offd = torch.from_numpy(off).to(dev)
    got = D.irreg_reduce(xd, offd, torch.float32).cpu().numpy()
    assert np.array_equal(got, O.ref_irreg_reduce(x, off).astype(np.float32)), "irreg reduce"
    got = D.irreg_scan(xd, offd, torch.float32).cpu().numpy()
    assert np.array_equal(got, O.ref_irreg_scan(x, off).astype(np.float32)), "irreg scan"
    done.append("irregular reduce/scan")


def run_bn(rng, dev, done):
    # batch-norm statistics: per-channel kernel (HW 49: 2-B vectors, HW 64:
    # 16-B vectors, last-block combine) and the per-segment kernel (HW 25)
    for shape in ((4, 8, 7, 7), (6, 8, 8, 8), (4, 8, 5, 5)):
        xb = rng.integers(-4, 5, shape).astype(np.float16)
        m, v = D.bn_stats(torch.from_numpy(xb).to(dev), torch.float64)
        em, ev = O.ref_bn_stats(xb)
        assert np.allclose(m.cpu().numpy(), em, rtol=1e-12, atol=1e-12), ("bn mean", shape)
        assert np.allclose(v.cpu().numpy(), ev, rtol=1e-9, atol=1e-9), ("bn var", shape)
        done.append(f"batch-norm stats {shape}")


if __name__ == "__main__":
    main()
