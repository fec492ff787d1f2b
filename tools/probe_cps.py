"""CTAs-per-SM A/B of the regular reduce sweep (TC_CTAS_PER_SM), 2^30 fp16."""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, ".")
from paper_1811_09736_b200 import _device as D  # noqa: E402

sys.path.insert(0, "tools")
from probe_modes import timeit  # noqa: E402

PEAK = float(json.loads((Path("MEASURED_PEAKS.json")).read_text())["hbm_gbs"]) if Path("MEASURED_PEAKS.json").exists() else 6450.0
n = 1 << 30
x = torch.rand(n, device="cuda").to(torch.float16)
for s in [16, 64, 256, 512, 1024, 2048, 4096, 8192, 65536]:
    out = torch.empty(-(-n // s), dtype=torch.float16, device="cuda")
    res = []
    for c in ("default", "1", "2", "3"):
        if c == "default":
            os.environ.pop("TC_CTAS_PER_SM", None)
        else:
            os.environ["TC_CTAS_PER_SM"] = c
        ms = timeit(lambda: D.seg_reduce(x, s, torch.float16, out=out), reps=20)
        gbs = (2 * n + 2 * (-(-n // s))) / ms / 1e6
        res.append(f"{c}: {ms:.4f} ms {100 * gbs / PEAK:5.1f}%")
    os.environ.pop("TC_CTAS_PER_SM", None)
    print(f"reduce s={s:>6} " + " | ".join(res), flush=True)
