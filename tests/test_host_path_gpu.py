"""The drop-in's own host-buffer path (_dispatch -> the native stager
tc_h2d_pageable / tc_d2h_pageable: pinned ring, host thread pool): numpy and pageable torch CPU inputs large enough to
take the staged path must give exactly the device-API results, for reduce
and scan outputs (small and large results), ragged sizes included."""

import numpy as np
import pytest
import torch

import paper_1811_09736_b200 as ht
from paper_1811_09736_b200 import _device as D
from paper_1811_09736_b200 import _dispatch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [(1 << 24) + 7, (1 << 27) + 4096 * 3 + 1])
def test_staged_host_copies_match_device_api(n, cuda):
    rng = np.random.default_rng(n)
    x = (rng.random(n) * 2 - 1).astype(np.float16)
    xd = torch.from_numpy(x).to(cuda)
    single = ht.TileEngine(accumulate="single")
    for s in (16, 300, 65536):
        got = ht.segmented_reduce(x, s, "strided16n" if s < 256 else "efficient256n", single)
        assert isinstance(got, np.ndarray)
        assert np.array_equal(got, D.seg_reduce(xd, s, torch.float32).cpu().numpy())
    # scan: the result is as large as the input (staged device -> host path)
    got = ht.segmented_scan(x, 4096, "warp256n", single)
    assert np.array_equal(got, D.seg_scan(xd, 4096, torch.float32).cpu().numpy())
    got = ht.segmented_scan(x, 4096, "warp256n", ht.TileEngine())
    assert got.dtype == np.float16
    assert np.array_equal(got, D.seg_scan(xd, 4096, torch.float16).cpu().numpy())
    # pageable torch CPU tensor in -> CPU tensor out
    xt = torch.from_numpy(x)
    got = ht.segmented_scan(xt, n, "grid", single)
    assert not got.is_cuda
    assert torch.equal(got, D.full_scan(xd, torch.float32).cpu())


def test_stager_round_trip_bytes(cuda):
    """to_device / from_device (the native pinned-ring stager,
    tc_h2d_pageable / tc_d2h_pageable: 16-MB chunks, 4 in flight) are
    byte-exact for every chunk boundary case and for unaligned host
    buffers (numpy views at odd element offsets)."""
    chunk = 16 << 20
    rng = np.random.default_rng(1)
    # 4 MB + 4 B: a single chunk whose size is not a multiple of the pool's
    # 4-KB slice granularity times its thread count
    for nbytes in (_dispatch._SMALL, _dispatch._SMALL + 4, chunk - 2, chunk * 5 + 18, chunk * 9 + 4096):
        for shift in (0, 1):
            n = nbytes // 2
            base = rng.integers(0, 1 << 16, n + 8, dtype=np.uint16).view(np.float16)
            x = base[shift:shift + n]  # shift 1: a 2-byte aligned source
            d = _dispatch.to_device(x, "numpy")
            assert torch.equal(d.view(torch.int16).cpu(), torch.from_numpy(x.view(np.int16).copy()))
            back = _dispatch.from_device(d, "numpy", np.float16)
            assert np.array_equal(back.view(np.uint16), x.view(np.uint16))
            # back-to-back transfers through the same ring, opposite directions
            y = _dispatch.to_device(x[::-1].copy(), "numpy")
            back2 = _dispatch.from_device(y, "numpy", np.float16)
            assert np.array_equal(back2.view(np.uint16), x[::-1].view(np.uint16))
