"""Host-side copy costs on the GPU box (iteration aid for the drop-in's
numpy -> device path): parallel pageable->pinned memcpy bandwidth by thread
count, cudaHostRegister cost, pinned and pageable H2D, and the stager."""
import concurrent.futures as cf
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")

n = 1 << 30
src = np.random.default_rng(0).random(n, dtype=np.float32).astype(np.float16)
pin = torch.empty(n, dtype=torch.float16, pin_memory=True)
pin_np = pin.numpy()
d = torch.empty(n, dtype=torch.float16, device="cuda")
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), flush=True)


def par_copy(dst, s, k, pool):
    nb = s.size
    cuts = [nb * t // k for t in range(k + 1)]
    fs = [pool.submit(np.copyto, dst[cuts[t]:cuts[t + 1]], s[cuts[t]:cuts[t + 1]]) for t in range(k)]
    for f in fs:
        f.result()


for k in (1, 2, 4, 8, 12, 16, 24, 32):
    with cf.ThreadPoolExecutor(k) as pool:
        par_copy(pin_np, src, k, pool)
        t0 = time.perf_counter()
        for _ in range(3):
            par_copy(pin_np, src, k, pool)
        dt = (time.perf_counter() - t0) / 3
    print(f"pageable->pinned memcpy 2 GiB, {k:2d} threads: {dt * 1e3:7.1f} ms = {2 * n / dt / 1e9:6.1f} GB/s", flush=True)

torch.cuda.synchronize()
for _ in range(2):
    t0 = time.perf_counter()
    d.copy_(pin, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"pinned H2D 2 GiB: {dt * 1e3:.1f} ms = {2 * n / dt / 1e9:.1f} GB/s", flush=True)
for _ in range(2):
    t0 = time.perf_counter()
    d.copy_(torch.from_numpy(src))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"pageable H2D 2 GiB (torch): {dt * 1e3:.1f} ms = {2 * n / dt / 1e9:.1f} GB/s", flush=True)

cudart = ctypes.CDLL("libcudart.so") if False else None
try:
    from cuda.bindings import runtime as rt  # cuda-python
except Exception:  # noqa: BLE001
    rt = None
if rt is not None:
    for trial in range(2):
        buf = np.empty(n, dtype=np.float16)
        buf[:] = src
        ptr = buf.ctypes.data
        t0 = time.perf_counter()
        err = rt.cudaHostRegister(ptr, buf.nbytes, 0)
        t1 = time.perf_counter()
        t = torch.from_numpy(buf)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        d.copy_(t, non_blocking=True)
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        rt.cudaHostUnregister(ptr)
        t4 = time.perf_counter()
        print(f"cudaHostRegister 2 GiB: {err} {1e3 * (t1 - t0):.1f} ms; H2D {1e3 * (t3 - t2):.1f} ms; "
              f"unregister {1e3 * (t4 - t3):.1f} ms", flush=True)

from paper_1811_09736_b200 import _dispatch as DP  # noqa: E402

for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = DP.to_device(src, "numpy")
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
print(f"stager to_device 2 GiB: {dt * 1e3:.1f} ms = {2 * n / dt / 1e9:.1f} GB/s", flush=True)
