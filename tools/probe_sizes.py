"""Iteration aid: time seg_reduce / seg_scan at given segment sizes, 2^30 fp16.
usage: python tools/probe_sizes.py reduce 300 1000 ... [scan 300 ...]"""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_1811_09736_b200 import _device as D  # noqa: E402
from perf_probe import PEAK, timeit  # noqa: E402

dev = torch.device("cuda:0")
n = 1 << 30
x = torch.rand(n, device=dev, dtype=torch.float32).to(torch.float16)
op = "reduce"
for a in sys.argv[1:]:
    if a in ("reduce", "scan"):
        op = a
        continue
    s = int(a)
    for dt, o in ((torch.float16, 2), (torch.float32, 4)):
        if op == "reduce":
            out = torch.empty(-(-n // s), dtype=dt, device=dev)
            ms = timeit(lambda: D.seg_reduce(x, s, dt, out=out))
            byts = 2 * n + o * (-(-n // s))
        else:
            out = torch.empty(n, dtype=dt, device=dev)
            ms = timeit(lambda: D.seg_scan(x, s, dt, out=out))
            byts = (2 + o) * n
        gbs = byts / ms / 1e6
        print(f"{op:6} s={s:>10} {str(dt):14} {ms:8.3f} ms {gbs:7.0f} GB/s {100 * gbs / PEAK:5.1f}%", flush=True)
