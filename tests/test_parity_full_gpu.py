"""Element-wise parity at the exact BASELINE.json sizes (no sampling).

* configs[1] (C2): segmented reduce of 2^30 fp16, all 13 segment sizes
  16..65536, fp16 and fp32 outputs;
* configs[2] (C3): segmented inclusive scan of 2^30 fp16, all 11 segment
  sizes 16..16384, fp16 and fp32 outputs (plus exclusive, fp32);
* configs[3] (C4): full reduce of 2^33 fp16 (fp64 / fp32 outputs);
* configs[4] (C5): full exclusive scan of 2^33 fp16, fp32 output, and its
  fp64 total_out.

Every output is compared against the exact binary64 oracle by the threaded
C checker (oracle/clib.py; the oracle restates pkg/src/halftile/oracle.py:
47-75 and is pinned to the reference in tests/test_oracle.py), streaming
the device result to the host in chunks.  Bound, as in
tests/test_parity_signed_gpu.py: |got - v| <= 1 ulp_out(v) + GAMMA * A,
A = sum |x| of the output's own elements, GAMMA = 16 * 2^-24.  Data:
uniform [0, 1) (the north star's distribution) and uniform [-1, 1) (signed,
C3 / C5).  The worst observed error / bound ratio is printed.
"""

import numpy as np
import pytest
import torch

from oracle import clib
from paper_1811_09736_b200 import _device as D

pytestmark = pytest.mark.gpu

GAMMA = 16 * 2.0 ** -24
CHUNK = 1 << 27


def _uniform(n, cuda, seed, signed=False):
    g = torch.Generator(device=cuda)
    g.manual_seed(seed)
    x = torch.rand(n, device=cuda, generator=g, dtype=torch.float32)
    if signed:
        x = x * 2 - 1
    return x.to(torch.float16)


def _host(xd):
    """Host copy of a (large) fp16 device vector, via a pinned bounce buffer."""
    n = xd.numel()
    out = np.empty(n, np.float16)
    ot = torch.from_numpy(out)
    for lo in range(0, n, CHUNK):
        hi = min(lo + CHUNK, n)
        ot[lo:hi].copy_(xd[lo:hi])
    return out


def _stream_check(checker, res, ulps=1.0):
    """Feed a device result to a ScanChecker chunk by chunk."""
    n = res.numel()
    buf = torch.empty(CHUNK, dtype=res.dtype, pin_memory=True)
    for lo in range(0, n, CHUNK):
        hi = min(lo + CHUNK, n)
        b = buf[: hi - lo]
        b.copy_(res[lo:hi])
        checker.check(lo, b.numpy(), ulps, GAMMA)
    return checker


@pytest.fixture(scope="module")
def c2c3_input(cuda):
    xd = _uniform(1 << 30, cuda, seed=2)
    return xd, _host(xd)


@pytest.mark.parametrize("s", [1 << k for k in range(4, 17)])
def test_c2_reduce_2p30_elementwise(s, c2c3_input):
    xd, x = c2c3_input
    for dt in (torch.float16, torch.float32):
        got = D.seg_reduce(xd, s, dt).cpu().numpy()
        c = clib.check_seg_reduce(x, s, got, 1.0, GAMMA)
        print(f"C2 s={s} {dt}: {c}")
        assert c.bad == 0, c


@pytest.mark.parametrize("s", [1 << k for k in range(4, 15)])
def test_c3_scan_2p30_elementwise(s, c2c3_input):
    xd, x = c2c3_input
    for dt, exc in ((torch.float16, False), (torch.float32, False), (torch.float32, True)):
        res = D.seg_scan(xd, s, dt, exclusive=exc)
        ch = _stream_check(clib.ScanChecker(x, s, inclusive=not exc), res)
        print(f"C3 s={s} {dt} exclusive={exc}: {ch}")
        assert ch.bad == 0, ch
        del res


@pytest.mark.parametrize("s", [16, 300, 4096, 16384])
def test_c3_scan_2p30_signed(s, cuda):
    xd = _uniform(1 << 30, cuda, seed=30 + s, signed=True)
    x = _host(xd)
    for dt in (torch.float16, torch.float32):
        res = D.seg_scan(xd, s, dt)
        ch = _stream_check(clib.ScanChecker(x, s), res)
        print(f"C3 signed s={s} {dt}: {ch}")
        assert ch.bad == 0, ch
        del res
    red = D.seg_reduce(xd, s, torch.float32).cpu().numpy()
    c = clib.check_seg_reduce(x, s, red, 1.0, GAMMA)
    assert c.bad == 0, c


@pytest.mark.parametrize("signed", [False, True])
def test_c4_c5_full_ops_2p33_elementwise(signed, cuda):
    n = 1 << 33
    xd = _uniform(n, cuda, seed=45 + int(signed), signed=signed)
    x = _host(xd)
    # C4: full reduce, fp64 partial path and fp32 output
    for dt in (torch.float64, torch.float32):
        got = D.full_reduce(xd, dt).cpu().numpy()
        c = clib.check_seg_reduce(x, n, got, 1.0, GAMMA)
        print(f"C4 signed={signed} {dt}: {c}")
        assert c.bad == 0, c
    # C5: full exclusive scan, fp32 output, element-wise; total_out in fp64
    tot = torch.zeros(1, dtype=torch.float64, device=cuda)
    res = D.full_scan(xd, torch.float32, exclusive=True, total_out=tot)
    ch = _stream_check(clib.ScanChecker(x, n, inclusive=False), res)
    print(f"C5 signed={signed}: {ch}")
    assert ch.bad == 0, ch
    exact = ch.exact_total  # running sum after the last element
    mass = sum(float(clib.seg_reduce(np.abs(x[lo:lo + CHUNK]), CHUNK)[0]) for lo in range(0, n, CHUNK))
    err = abs(tot.item() - exact)
    print(f"C5 total_out signed={signed}: got {tot.item()!r} exact {exact!r} "
          f"rel {err / max(abs(exact), 1e-300):.3g} err/mass {err / mass:.3g}")
    assert err <= GAMMA * mass, (tot.item(), exact)
    del res
