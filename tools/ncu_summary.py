"""Summarise an ncu report (raw metrics + hottest source lines by stall).

usage: python tools/ncu_summary.py REPORT.ncu-rep [--lines N]
Prints the key roofline metrics (duration, DRAM bytes / throughput, tensor
pipe activity, occupancy) and the source lines with the most warp-stall
samples, for the profiles/ summaries.
"""

import argparse
import csv
import io
import subprocess

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def ncu(report, page):
    out = subprocess.run(["ncu", "-i", report, "--page", page, "--csv"], capture_output=True,
                         text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--lines", type=int, default=15)
    args = ap.parse_args()
    rows = ncu(args.report, "raw")
    hdr = rows[0]
    units = rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name[:120]}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:90s} {r[i]:>16s} {units[i]}")
    try:
        src = ncu(args.report, "source")
    except subprocess.CalledProcessError:
        return
    # first row may be a "Kernel Name" banner
    while src and "Address" not in src[0] and "#" not in src[0]:
        src = src[1:]
    if not src:
        return
    h = src[0]
    cols = {c: i for i, c in enumerate(h)}
    il = cols.get("Warp Stall Sampling (All Samples)")
    if il is None:
        return
    srccol = cols.get("Source", 1)
    stall_cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    totals = {c: 0.0 for c in stall_cols}
    data = []
    for r in src[1:]:
        try:
            data.append((float(r[il] or 0), r[cols.get("Address", 0)], r[srccol].strip()[:100]))
            for c in stall_cols:
                totals[c] += float(r[cols[c]] or 0)
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1.0
    print(f"  stall reasons (share of {tot:.0f} samples):")
    for c, v in sorted(totals.items(), key=lambda kv: -kv[1])[:8]:
        print(f"    {c:28s} {100 * v / tot:5.1f}%")
    print("  hottest instructions by warp-stall samples:")
    for s_, ad, txt in sorted(data, reverse=True)[: args.lines]:
        print(f"    {100 * s_ / tot:5.1f}%  {ad[-5:]}  {txt}")


if __name__ == "__main__":
    main()
