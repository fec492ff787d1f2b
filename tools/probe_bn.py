"""Iteration aid: batch-norm statistics bandwidth on typical NCHW shapes."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_1811_09736_b200 import _device as D  # noqa: E402
from perf_probe import PEAK, timeit  # noqa: E402

for shape in [(256, 256, 56, 56), (256, 64, 112, 112), (256, 512, 28, 28), (256, 1024, 14, 14),
              (256, 2048, 7, 7)]:
    x = torch.rand(shape, device="cuda").to(torch.float16)
    n = x.numel()
    ms = timeit(lambda: D.bn_stats(x))
    ms_t = timeit(lambda: torch.var_mean(x, dim=(0, 2, 3), correction=0))
    print(f"bn {str(shape):22} {ms:7.3f} ms  alg {2 * n / ms / 1e6:6.0f} GB/s "
          f"({100 * 2 * n / ms / 1e6 / PEAK:5.1f}%)  actual {4 * n / ms / 1e6:6.0f} GB/s | "
          f"torch.var_mean {ms_t:7.3f} ms", flush=True)
