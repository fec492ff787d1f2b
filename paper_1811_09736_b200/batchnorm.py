"""Batch-norm statistics on the B200 reduction path -- the application the
paper evaluates its TCU reduction on ("the computation
of mu_B (the mean) is a reduction operation and we can leverage the TCU";
SURVEY.md section 8(f)4).  The reference package has no entry point for
it; this one follows its conventions (numpy in -> numpy out, torch CUDA in
-> torch CUDA out, HalftileError subclasses for bad shapes).

``batch_norm_stats(x)`` for x of shape (N, C, *spatial), NCHW-contiguous,
fp16 or bf16 (other dtypes raise TypeError: narrowing fp32 activations to
fp16 would overflow above 65504 and round the statistics):

* ONE read of x (``tc_bn_stats``): every (n, c) segment gives its
  shifted-data moments S1 = sum(x - K_c), S2 = sum((x - K_c)^2) with
  K_c = x[0, c, 0], fp32 per lane and fp64 per segment;
* a per-channel fp64 combine in fixed order: mean[c] = K_c + S1 / M,
  var[c] = S2 / M - (S1 / M)^2 (biased; M = N * HW).  The shift keeps the
  subtraction well conditioned (no E[x^2] - mean^2 cancellation).

The squares need the elements themselves, which a tensor-core MMA against
a constant matrix cannot produce, so the statistics run on CUDA cores; the
mean alone (the paper's TCU use) is ``segmented_reduce(x, HW)``.

``batch_norm(x, weight, bias, eps)`` applies y = (x - mean) / sqrt(var +
eps) * weight + bias with those statistics (the normalisation itself is an
elementwise torch op, outside the reduction path).
"""

from __future__ import annotations

import numpy as np

from . import _dispatch as _d
from .errors import BadLengthError


def batch_norm_stats(x, out_dtype=np.float32):
    """(mean, var) per channel of an (N, C, *spatial) tensor / array."""
    import torch

    from . import _device

    t_dtype = torch.float64 if np.dtype(out_dtype) == np.float64 else torch.float32
    if isinstance(x, torch.Tensor):
        if x.dim() < 2 or x.numel() == 0:
            raise BadLengthError("batch-norm statistics need a non-empty (N, C, ...) tensor")
        if x.is_cuda:
            return _device.bn_stats(x, t_dtype)
        kind, host = "torch_cpu", x
    else:
        host = np.ascontiguousarray(x, dtype=np.float16)
        if host.ndim < 2 or host.size == 0:
            raise BadLengthError("batch-norm statistics need a non-empty (N, C, ...) array")
        kind = "numpy"
    shape = tuple(host.shape)
    flat = host.reshape(-1)
    dev = _d.to_device(flat, kind).reshape(shape)
    mean, var = _device.bn_stats(dev, t_dtype)
    np_dt = np.float64 if t_dtype == torch.float64 else np.float32
    return _d.from_device(mean, kind, np_dt), _d.from_device(var, kind, np_dt)


def batch_norm(x, weight=None, bias=None, eps: float = 1e-5):
    """Training-mode batch norm forward on a CUDA tensor with the statistics
    above; returns (y, mean, var)."""
    import torch

    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        raise TypeError("batch_norm takes a CUDA tensor (use batch_norm_stats for host arrays)")
    mean, var = batch_norm_stats(x)
    shape = (1, -1) + (1,) * (x.dim() - 2)
    inv = torch.rsqrt(var + eps)
    y = (x.float() - mean.view(shape)) * inv.view(shape)
    if weight is not None:
        y = y * weight.float().view(shape)
    if bias is not None:
        y = y + bias.float().view(shape)
    return y.to(x.dtype), mean, var
