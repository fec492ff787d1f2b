"""Native stager throughput (tc_h2d_pageable / tc_d2h_pageable), 2 GiB."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1811_09736_b200 import _dispatch
n = 1 << 30
x = np.random.default_rng(0).random(n, dtype=np.float32).astype(np.float16)
d = torch.empty(n, dtype=torch.float16, device="cuda")
ts = []
for _ in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _dispatch._h2d(x, d); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
h = np.empty(n, np.float16)
td = []
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    _dispatch._d2h(d, h); td.append(time.perf_counter() - t0)
assert np.array_equal(h.view(np.uint16), x.view(np.uint16))
print(f"h2d {1e3*min(ts):.1f} ms ({2*n/min(ts)/1e9:.1f} GB/s)  d2h {1e3*min(td):.1f} ms ({2*n/min(td)/1e9:.1f} GB/s)", flush=True)
