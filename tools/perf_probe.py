"""Quick bandwidth probe of the kernels at 2^30 elements (iteration aid;
the contract benchmark is bench.py)."""

import sys

import torch

sys.path.insert(0, ".")
from paper_1811_09736_b200 import _device as D  # noqa: E402

PEAK = 6533.8


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    dev = torch.device("cuda:0")
    n = 1 << 30
    x = torch.rand(n, device=dev, dtype=torch.float32).to(torch.float16)
    which = sys.argv[1:] or ["reduce", "scan"]
    # copy baseline
    y = torch.empty_like(x)
    ms = timeit(lambda: y.copy_(x))
    print(f"copy fp16 2^30: {ms:.3f} ms  {4 * n / ms / 1e6:.0f} GB/s", flush=True)
    if "reduce" in which:
        for s in [16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536, 300, 1000, n]:
            for dt, o in ((torch.float32, 4), (torch.float16, 2)):
                out = torch.empty(-(-n // s), dtype=dt, device=dev)
                ms = timeit(lambda: D.seg_reduce(x, s, dt, out=out))
                byts = 2 * n + o * (-(-n // s))
                gbs = byts / ms / 1e6
                print(f"reduce s={s:>10} {str(dt):14} {ms:8.3f} ms {n / ms / 1e9:7.1f} Gelem/s "
                      f"{gbs:7.0f} GB/s {100 * gbs / PEAK:5.1f}%", flush=True)
    if "scan" in which:
        out16 = torch.empty(n, dtype=torch.float16, device=dev)
        out32 = torch.empty(n, dtype=torch.float32, device=dev)
        for s in [16, 32, 64, 256, 1024, 4096, 8192, 16384, 300, n]:
            for dt, o, out in ((torch.float16, 2, out16), (torch.float32, 4, out32)):
                ms = timeit(lambda: D.seg_scan(x, s, dt, out=out))
                byts = (2 + o) * n
                gbs = byts / ms / 1e6
                print(f"scan   s={s:>10} {str(dt):14} {ms:8.3f} ms {n / ms / 1e9:7.1f} Gelem/s "
                      f"{gbs:7.0f} GB/s {100 * gbs / PEAK:5.1f}%", flush=True)


def full_probe():
    import os

    dev = torch.device("cuda:0")
    for log2n in ((30,) if os.environ.get("TC_DEBUG") else (30, 33)):
        n = 1 << log2n
        x = torch.empty(n, dtype=torch.float16, device=dev)
        for lo in range(0, n, 1 << 28):
            x[lo:lo + (1 << 28)] = torch.rand(min(1 << 28, n - lo), device=dev)
        y = torch.empty(n, dtype=torch.float32, device=dev)
        y16 = torch.empty(n, dtype=torch.float16, device=dev)
        for k, lag in (("1", "3"), ("2", "3"), ("3", "1"), ("4", "1")):
            os.environ["TC_CHUNK_TILES"] = k
            os.environ["TC_CHUNK_LAG"] = lag
            for dt, o, out in ((torch.float32, 4, y), (torch.float16, 2, y16)):
                ms = timeit(lambda: D.full_scan(x, dt, exclusive=True, out=out), reps=5, warm=2)
                gbs = (2 + o) * n / ms / 1e6
                print(f"full excl scan 2^{log2n} K={k:>2} L={lag} {str(dt):14} {ms:8.3f} ms "
                      f"{n / ms / 1e6:7.1f} Gelem/s {gbs:7.0f} GB/s {100 * gbs / PEAK:5.1f}%",
                      flush=True)
        os.environ.pop("TC_CHUNK_TILES")
        for s_ in (1 << 19, 1 << 22):
            ms = timeit(lambda: D.seg_scan(x, s_, torch.float32, out=y), reps=5, warm=2)
            gbs = 6 * n / ms / 1e6
            print(f"seg scan 2^{log2n} s={s_} f32 {ms:8.3f} ms {gbs:7.0f} GB/s {100 * gbs / PEAK:5.1f}%",
                  flush=True)
        del x, y, y16
        torch.cuda.empty_cache()


if __name__ == "__main__":
    if sys.argv[1:] == ["full"]:
        full_probe()
        sys.exit(0)
    main()
