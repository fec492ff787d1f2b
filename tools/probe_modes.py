"""Bandwidth of the GENERAL / GSCR reduce kernels (odd and non-power-of-two
segment sizes), scans of the same sizes, and batch-norm statistics, at 2^30
fp16 (iteration aid; bench.py is the contract benchmark).

usage: python tools/probe_modes.py [reduce] [scan] [bn]
"""

import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, ".")
from paper_1811_09736_b200 import _device as D  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent
try:
    PEAK = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
except Exception:  # noqa: BLE001
    PEAK = 6548.5


def set_ab(var, val):
    """A/B setting: var=val, or with var "multi" a value "A=1:B=0" setting several variables
    (None clears them)."""
    import os

    if var != "multi":
        if val is None:
            os.environ.pop(var, None)
        else:
            os.environ[var] = val
        return
    for k in list(os.environ):
        if k.startswith("TC_") and k in os.environ.get("PROBE_MULTI_VARS", "").split(","):
            os.environ.pop(k)
    if val is not None:
        for kv in val.split(":"):
            k, v = kv.split("=")
            os.environ[k] = v


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
    which = sys.argv[1:] or ["reduce", "scan", "bn"]
    if "reduce" in which:
        import os

        sizes = [3, 5, 7, 9, 12, 17, 20, 24, 33, 40, 48, 49, 63, 65, 100, 127, 129, 300, 1000,
                 4097, 100001]
        if os.environ.get("PROBE_SIZES"):
            sizes = [int(v) for v in os.environ["PROBE_SIZES"].split(",")]
        for s in sizes:
            for dt, o in ((torch.float16, 2), (torch.float32, 4)):
                out = torch.empty(-(-n // s), dtype=dt, device=dev)
                res = []
                abr = os.environ.get("PROBE_AB_R", "TC_ROWSEG")  # A/B switch of the reduce rows
                for rs in os.environ.get("PROBE_AB_VALS", "1,0").split(","):  # e.g. MODE_ROWSEG on / off
                    set_ab(abr, rs)
                    ms = timeit(lambda: D.seg_reduce(x, s, dt, out=out))
                    gbs = (2 * n + o * (-(-n // s))) / ms / 1e6
                    res.append(f"{abr}={rs} {ms:7.3f} ms {gbs:6.0f} GB/s {100 * gbs / PEAK:5.1f}%")
                set_ab(abr, None)
                print(f"reduce s={s:>7} {str(dt):14} " + " | ".join(res), flush=True)
    if "scan" in which:
        import os

        sizes = [3, 5, 6, 7, 9, 10, 12, 17, 20, 33, 34, 48, 63, 65, 66, 100, 130, 300, 1000, 4097, 100000,
                 100001, (1 << 19) + 3, (1 << 19) + 4, n]
        if os.environ.get("PROBE_SCAN_SIZES"):
            sizes = [int(v) for v in os.environ["PROBE_SCAN_SIZES"].split(",")]
        for s in sizes:
            for dt, o in ((torch.float16, 2), (torch.float32, 4)):
                out = torch.empty(n, dtype=dt, device=dev)
                res = []
                ab = os.environ.get("PROBE_AB", "TC_ROWSEG")  # A/B switch of the scan rows
                for rs in os.environ.get("PROBE_AB_VALS", "1,0").split(","):
                    set_ab(ab, rs)
                    ms = timeit(lambda: D.seg_scan(x, s, dt, out=out))
                    gbs = (2 + o) * n / ms / 1e6
                    res.append(f"{ab}={rs} {ms:7.3f} ms {gbs:6.0f} GB/s {100 * gbs / PEAK:5.1f}%")
                set_ab(ab, None)
                print(f"scan   s={s:>10} {str(dt):14} " + " | ".join(res), flush=True)
    if "bn" in which:
        for shape in ((256, 256, 56, 56), (256, 512, 28, 28), (256, 1024, 14, 14),
                      (256, 2048, 7, 7), (64, 96, 35, 35), (32, 384, 17, 17)):
            xb = torch.rand(shape, device=dev).to(torch.float16)
            ms = timeit(lambda: D.bn_stats(xb))
            gbs = 2 * xb.numel() / ms / 1e6
            # the same call replayed from a CUDA graph (no host overhead)
            D.bn_stats(xb)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                D.bn_stats(xb)
            msg = timeit(g.replay)
            gbsg = 2 * xb.numel() / msg / 1e6
            print(f"bn {shape}: {ms:7.3f} ms {gbs:6.0f} GB/s {100 * gbs / PEAK:5.1f}% | graph "
                  f"{msg:7.3f} ms {gbsg:6.0f} GB/s {100 * gbsg / PEAK:5.1f}%", flush=True)
            del xb


if __name__ == "__main__":
    main()
