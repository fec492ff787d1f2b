"""Run one op a few times (profiling target for ncu).

usage: python tools/prof_one.py reduce|scan SEG f16|f32 [LOG2N] [REPS]
"""

import sys

import torch

sys.path.insert(0, ".")
from paper_1811_09736_b200 import _device as D  # noqa: E402


def main():
    op, seg, dt = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    log2n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    n = 1 << log2n
    dtype = {"f16": torch.float16, "f32": torch.float32, "f64": torch.float64}[dt]
    x = torch.rand(n, device="cuda", dtype=torch.float32).to(torch.float16)
    for _ in range(reps):
        if op == "reduce":
            D.seg_reduce(x, seg, dtype)
        else:
            D.seg_scan(x, seg, dtype)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
