"""Profiling target: one irregular op a few times.
usage: python tools/prof_irreg.py reduce|scan MEAN f16|f32 [REPS]"""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_1811_09736_b200 import _device as D  # noqa: E402
from probe_irreg import device_offsets  # noqa: E402

op, mean, dt = sys.argv[1], int(sys.argv[2]), sys.argv[3]
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
dtype = {"f16": torch.float16, "f32": torch.float32}[dt]
n = 1 << 30
dev = torch.device("cuda:0")
x = torch.rand(n, device=dev, dtype=torch.float32).to(torch.float16)
off = device_offsets(n, mean, dev)
for _ in range(reps):
    if op == "reduce":
        D.irreg_reduce(x, off, dtype, validate=False)
    else:
        D.irreg_scan(x, off, dtype, validate=False)
torch.cuda.synchronize()
