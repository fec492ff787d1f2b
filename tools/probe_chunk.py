"""CHUNK-mode scans (full scan, pow2 segments > 2^18), 2^30 fp16, fp16 and fp32 out."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_1811_09736_b200 import _device as D  # noqa: E402
from probe_modes import timeit  # noqa: E402

PEAK = float(json.loads(Path("MEASURED_PEAKS.json").read_text())["hbm_gbs"]) if Path("MEASURED_PEAKS.json").exists() else 6450.0
n = 1 << 30
x = (torch.rand(n, device="cuda") * 2 - 1).to(torch.float16)
for dt, o in ((torch.float16, 2), (torch.float32, 4)):
    out = torch.empty(n, dtype=dt, device="cuda")
    row = []
    for s in (1 << 19, 1 << 22, n):
        for exc in (False, True):
            ms = timeit(lambda: D.seg_scan(x, s, dt, exclusive=exc, out=out), reps=10)
            row.append(f"s=2^{s.bit_length() - 1}{' ex' if exc else ''}: {100 * (2 + o) * n / ms / 1e6 / PEAK:5.1f}%")
    print(str(dt), " | ".join(row), flush=True)
