"""fp32-output segmented scan sweep, 2^30 fp16 (A/B aid: run with and
without TC_COLLECTIVES_LIB pointing at an experimental build)."""
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
x = torch.rand(n, device="cuda").to(torch.float16)
out = torch.empty(n, dtype=torch.float32, device="cuda")
row = []
for s in [16, 32, 64, 128, 256, 512, 1024, 4096, 16384]:
    ms = timeit(lambda: D.seg_scan(x, s, torch.float32, out=out), reps=10)
    row.append(f"s={s}: {100 * 6 * n / ms / 1e6 / PEAK:5.1f}%")
print(" | ".join(row), flush=True)
