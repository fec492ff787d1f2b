"""Per-phase cycle costs of the irregular-reduce epilogue groups (debug
build with -DTC_IRREG_TRACE loaded through TC_COLLECTIVES_LIB).
usage: TC_COLLECTIVES_LIB=tools/_tc_trace.so python tools/irreg_trace.py MEAN"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
from paper_1811_09736_b200 import _device as D, _lib  # noqa: E402
from probe_irreg import device_offsets  # noqa: E402

mean = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = 1 << 30
dev = torch.device("cuda:0")
x = torch.rand(n, device=dev).to(torch.float16)
off = device_offsets(n, mean, dev)
for _ in range(3):
    D.irreg_reduce(x, off, torch.float32, validate=False)
torch.cuda.synchronize()
NG = 3
buf = np.zeros((NG, 64, 8), np.int64)
assert _lib.lib.tc_debug_irreg_trace(ctypes.c_void_p(buf.ctypes.data)) == 0
names = ["mark+B1+wait_tfull", "tmem_ld", "slots", "barrier2", "segments+rec", "barrier3", "->next"]
for g in range(NG):
    b = buf[g, 8:60]
    d = np.diff(b[:, :7], axis=1)
    nxt = b[1:, 0] - b[:-1, 6]
    per = (b[1:, 0] - b[:-1, 0])
    print(f"group {g}: cycles per tile {np.median(per):.0f}; phases (median) " +
          ", ".join(f"{nm} {np.median(d[:, k]):.0f}" for k, nm in enumerate(names[:6])) +
          f", next-start {np.median(nxt):.0f}, mark+B1 {np.median(b[:, 7] - b[:, 0]):.0f}")
