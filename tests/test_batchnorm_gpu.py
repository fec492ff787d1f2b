"""GPU parity of the batch-norm statistics consumer (tc_bn_stats) against
the binary64 oracle (oracle.ref_bn_stats).

Tolerances: mean -- the tensor-core segment sums are fp32 within a row and
fp64 across rows / segments, so |mean - exact| <= 1e-6 * max|x| + 1e-6 *
|exact|; var -- centred fp32 squares per lane flushed to fp64 per segment:
relative 1e-5 (plus 1e-7 * max|x|^2 absolute for near-zero variances).
Integer data with an integer mean is exact.
"""

import numpy as np
import pytest
import torch

import paper_1811_09736_b200 as ht
from oracle import oracle as O

pytestmark = pytest.mark.gpu

# per-channel streaming kernel by vector width (HW % 8 / 4 / 2 / odd, HW >= 48)
# and the per-segment kernel (HW < 48)
SHAPES = [(2, 3, 7, 7), (1, 1, 1), (5, 2), (8, 64, 56, 56), (32, 256, 14, 14), (3, 17, 1000),
          (256, 64, 28, 28), (4, 8, 300, 7), (64, 96, 7, 7), (7, 5, 50), (3, 300, 62),
          (1, 2, 4096)]


def check(mean, var, x):
    em, ev = O.ref_bn_stats(x)
    amax = float(np.abs(np.asarray(x, np.float64)).max())
    mean = np.asarray(mean, np.float64)
    var = np.asarray(var, np.float64)
    assert mean.shape == em.shape and var.shape == ev.shape
    assert np.all(np.abs(mean - em) <= 1e-6 * amax + 1e-6 * np.abs(em)), np.abs(mean - em).max()
    assert np.all(np.abs(var - ev) <= 1e-5 * ev + 1e-7 * amax * amax), np.abs(var - ev).max()


@pytest.mark.parametrize("shape", SHAPES)
def test_bn_stats_uniform(cuda, shape):
    g = np.random.default_rng(1)
    x = (g.random(shape) * 4 - 1).astype(np.float16)
    mean, var = ht.batch_norm_stats(x)
    assert mean.dtype == np.float32 and var.dtype == np.float32
    check(mean, var, x)
    m64, v64 = ht.batch_norm_stats(torch.from_numpy(x).to(cuda), out_dtype=np.float64)
    assert m64.is_cuda and m64.dtype == torch.float64
    check(m64.cpu().numpy(), v64.cpu().numpy(), x)


def test_bn_stats_exact_and_offset(cuda):
    # constant channels: variance exactly 0; large offset vs small spread: no cancellation
    x = np.zeros((4, 3, 64), np.float16)
    x[:, 0] = 5.0
    x[:, 1] = np.arange(64) % 2  # mean 0.5, var 0.25 exactly
    x[:, 2] = 1000.0 + (np.arange(64) % 4) * 0.5
    mean, var = ht.batch_norm_stats(x, out_dtype=np.float64)
    assert mean.tolist()[:2] == [5.0, 0.5] and var.tolist()[:2] == [0.0, 0.25]
    check(mean, var, x)


def test_bn_bf16_and_forward_matches_torch(cuda):
    g = torch.Generator(device=cuda)
    g.manual_seed(3)
    x = torch.randn(16, 32, 24, 24, device=cuda, generator=g).to(torch.float16)
    w = torch.rand(32, device=cuda) + 0.5
    b = torch.rand(32, device=cuda)
    y, mean, var = ht.batch_norm(x, w, b, eps=1e-5)
    ref = torch.nn.functional.batch_norm(x.float(), None, None, w, b, training=True, eps=1e-5)
    assert torch.allclose(y.float(), ref, atol=2e-2, rtol=1e-2)
    check(mean.cpu().numpy(), var.cpu().numpy(), x.cpu().numpy())
    xb = x.to(torch.bfloat16)
    mb, vb = ht.batch_norm_stats(xb)
    check(mb.cpu().numpy(), vb.cpu().numpy(), xb.float().cpu().numpy())


def test_bn_repeatable_and_workspace_clean(cuda):
    """Two calls give bit-identical statistics (fixed combine order whichever
    block finishes last), and a later CHUNK scan on the same stream's
    workspace is unaffected (the statistics kernels re-zero their scratch)."""
    from paper_1811_09736_b200 import _device as D

    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    # a CHUNK scan first: its epoch-tagged look-back words stay in the workspace
    xs0 = torch.randint(-4, 5, ((1 << 20) + 5,), device=cuda, generator=g).to(torch.float16)
    assert torch.equal(D.seg_scan(xs0, xs0.numel(), torch.float32), torch.cumsum(xs0.double(), 0).float())
    x = (torch.rand(64, 256, 28, 28, device=cuda, generator=g) * 3 - 1).to(torch.float16)
    m1, v1 = D.bn_stats(x)
    check(m1.cpu().numpy(), v1.cpu().numpy(), x.cpu().numpy())
    m2, v2 = D.bn_stats(x)
    assert torch.equal(m1, m2) and torch.equal(v1, v2)
    xs = torch.randint(-4, 5, ((1 << 21) + 3,), device=cuda, generator=g).to(torch.float16)
    got = D.seg_scan(xs, xs.numel(), torch.float32)
    ref = torch.cumsum(xs.double(), 0).float()
    assert torch.equal(got, ref)
