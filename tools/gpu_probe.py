"""Quick GPU probe: run the C-ABI kernels over a matrix of small cases and
print PASS/FAIL per case (used for fast iteration under gpurun; the formal
parity suite is tests/test_parity_gpu.py)."""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1811_09736_b200 import _device as D  # noqa: E402


def ref_reduce(x64, s):
    n = x64.size
    nseg = -(-n // s)
    pad = np.zeros(nseg * s)
    pad[:n] = x64
    return pad.reshape(nseg, s).sum(1)


def ref_scan(x64, s, exclusive=False, carry=None):
    n = x64.size
    nseg = -(-n // s)
    pad = np.zeros(nseg * s)
    pad[:n] = x64
    segs = pad.reshape(nseg, s)
    if carry is not None:
        segs = segs.copy()
        segs[0, 0] += carry
    c = np.cumsum(segs, axis=1)
    if exclusive:
        e = np.zeros_like(c)
        e[:, 1:] = c[:, :-1]
        if carry is not None:
            e[0, 0] = carry
        c = e
    return c.reshape(-1)[:n]


def check(name, got, exp, dt):
    got = got.double().cpu().numpy() if isinstance(got, torch.Tensor) else got
    if dt == torch.float16:
        e16 = exp.astype(np.float16).astype(np.float64)
        ok = np.array_equal(got, e16)
    elif dt == torch.float32:
        e32 = exp.astype(np.float32).astype(np.float64)
        ok = np.array_equal(got, e32)
    else:
        ok = np.array_equal(got, exp)
    if not ok:
        bad = np.nonzero(got != (exp.astype(np.float16).astype(np.float64) if dt == torch.float16 else exp.astype(np.float32).astype(np.float64) if dt == torch.float32 else exp))[0]
        print(f"FAIL {name}: {bad.size} mismatches, first idx {bad[:8].tolist()} "
              f"got {got[bad[:4]].tolist()} exp {exp[bad[:4]].tolist()}", flush=True)
    else:
        print(f"PASS {name}", flush=True)
    return ok


def main():
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(1)
    fails = 0
    total = 0
    ns = [8192, 65536, 1 << 20, 1000, 100, 12345, 64, 8192 * 3 + 70, (1 << 22) + 1234]
    segs = [16, 32, 64, 128, 256, 1024, 8192, 16384, 65536, 48, 300, 7, 1, 24576, 100000,
            1 << 17, (1 << 18) + 8192, 1 << 20]
    only = sys.argv[1] if len(sys.argv) > 1 else "all"
    for n in ns:
        x = rng.integers(0, 8, n).astype(np.float16)
        xd = torch.from_numpy(x).to(dev)
        x64 = x.astype(np.float64)
        for s in segs + [n]:
            if only in ("all", "reduce"):
                for dt in (torch.float32, torch.float16, torch.float64):
                    total += 1
                    t0 = time.time()
                    got = D.seg_reduce(xd, s, dt)
                    torch.cuda.synchronize()
                    fails += not check(f"reduce n={n} s={s} {dt}", got, ref_reduce(x64, s), dt)
            if only in ("all", "scan"):
                for dt in (torch.float32, torch.float16):
                    for exc in (False, True):
                        total += 1
                        got = D.seg_scan(xd, s, dt, exclusive=exc)
                        torch.cuda.synchronize()
                        fails += not check(f"scan n={n} s={s} {dt} excl={exc}", got,
                                           ref_scan(x64, s, exc), dt)
    # carry-in / total-out
    if only in ("all", "scan"):
        for n in (1000, 8192 * 5 + 3, 1 << 20):
            x = rng.integers(0, 8, n).astype(np.float16)
            xd = torch.from_numpy(x).to(dev)
            cin = torch.tensor([37.0], dtype=torch.float64, device=dev)
            tot = torch.zeros(1, dtype=torch.float64, device=dev)
            for exc in (False, True):
                total += 1
                got = D.seg_scan(xd, n, torch.float32, exclusive=exc, carry_in=cin, total_out=tot)
                torch.cuda.synchronize()
                fails += not check(f"scan carry n={n} excl={exc}", got,
                                   ref_scan(x.astype(np.float64), n, exc, carry=37.0), torch.float32)
                t = tot.item()
                expt = 37.0 + x.astype(np.float64).sum()
                if t != expt:
                    fails += 1
                    print(f"FAIL total_out n={n}: {t} vs {expt}")
    print(f"SUMMARY {total - fails}/{total} passed", flush=True)


if __name__ == "__main__":
    main()
