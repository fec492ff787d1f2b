"""Profiling target: batch-norm statistics of an NCHW fp16 tensor a few times.
usage: python tools/prof_bn.py N C H W [REPS]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_1811_09736_b200 import _device as D  # noqa: E402

N, C, H, W = (int(a) for a in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
x = torch.rand(N, C, H, W, device="cuda").to(torch.float16)
for _ in range(reps):
    D.bn_stats(x)
torch.cuda.synchronize()
