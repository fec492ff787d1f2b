"""Iteration aid: irregular (CSR-offset) reduce / scan bandwidth at 2^30 fp16
with geometric segment lengths of the given means."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_1811_09736_b200 import _device as D  # noqa: E402
from perf_probe import PEAK, timeit  # noqa: E402


def device_offsets(n, mean, dev, seed=0):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    m = int(2 * n / mean) + 16
    u = torch.rand(m, device=dev, generator=g, dtype=torch.float64).clamp_min(1e-300)
    lens = torch.ceil(-torch.log(u) * (mean - 0.5)).to(torch.int64)
    ends = torch.cumsum(lens, 0)
    ends = ends[ends < n]
    z = torch.zeros(1, dtype=torch.int64, device=dev)
    return torch.cat([z, ends, torch.full((1,), n, dtype=torch.int64, device=dev)])


def main():
    dev = torch.device("cuda:0")
    n = 1 << 30
    x = torch.rand(n, device=dev, dtype=torch.float32).to(torch.float16)
    means = [int(a) for a in sys.argv[1:]] or [16, 64, 256, 1024, 16384, 1 << 20]
    for mean in means:
        off = device_offsets(n, mean, dev)
        nseg = off.numel() - 1
        for dt, o in ((torch.float32, 4), (torch.float16, 2)):
            out = torch.empty(nseg, dtype=dt, device=dev)
            ms = timeit(lambda: D.irreg_reduce(x, off, dt, out=out, validate=False))
            byts = 2 * n + 8 * (nseg + 1) + o * nseg
            gbs = byts / ms / 1e6
            print(f"irreg reduce mean={mean:>8} nseg={nseg:>9} {str(dt):14} {ms:8.3f} ms {gbs:7.0f} GB/s "
                  f"{100 * gbs / PEAK:5.1f}%", flush=True)
        if os.environ.get("PROBE_REDUCE_ONLY"):
            continue
        for dt, o in ((torch.float32, 4), (torch.float16, 2)):
            out = torch.empty(n, dtype=dt, device=dev)
            ms = timeit(lambda: D.irreg_scan(x, off, dt, out=out, validate=False))
            byts = 2 * n + 8 * (nseg + 1) + o * n
            gbs = byts / ms / 1e6
            print(f"irreg scan   mean={mean:>8} nseg={nseg:>9} {str(dt):14} {ms:8.3f} ms {gbs:7.0f} GB/s "
                  f"{100 * gbs / PEAK:5.1f}%", flush=True)


if __name__ == "__main__":
    main()
