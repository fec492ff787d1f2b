"""Distil one gpurun session (gpurun_out/<tag>/) into tracked evidence under
profiles/<round>/:

  launches_summary.md   per-kernel launch list from the ncu launch pass
                        (gpu__time_duration + DRAM bytes per launch), share
                        of the timed step per kernel
  ncu_<cfg>.txt         --set full summaries (tools/ncu_summary.py output)
  bench.json / bench_ref.json   the bench lines of the same session
  profiles/traffic.json per-launch DRAM traffic of the dominant kernel
                        (read by bench.py for roofline.traffic)

usage: python tools/make_profiles.py TAG ROUND
"""

import csv
import json
import shutil
import statistics
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    per = defaultdict(dict)
    names = {}
    grids = {}
    for r in rows[i + 1:]:
        if len(r) < len(h):
            continue
        lid = int(r[h.index("ID")])
        names[lid] = r[h.index("Kernel Name")]
        grids[lid] = r[h.index("Grid Size")]
        per[lid][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
    return [(lid, names[lid], grids[lid], per[lid]) for lid in sorted(per)]


def main():
    tag, rnd = sys.argv[1], sys.argv[2]
    src = ROOT / "gpurun_out" / tag
    dst = ROOT / "profiles" / rnd
    dst.mkdir(parents=True, exist_ok=True)
    for f in ("bench.json", "bench_ref.json", "pytest_gpu.log", "smoke.log"):
        if (src / f).exists():
            shutil.copy(src / f, dst / f)
    for f in sorted(src.glob("prof_*.txt")):
        shutil.copy(f, dst / f.name.replace("prof_", "ncu_"))
    lf = src / "launches.csv"
    if not lf.exists():
        return
    ls = launches(lf)
    ours = [x for x in ls if "tc::seg_kernel" in x[1]]
    by = defaultdict(list)
    for lid, name, grid, m in ours:
        # group by instantiation and input size (bench sweep 2^30 vs e2e chunks 2^27)
        gb = round(m.get("dram__bytes_read.sum", 0) / 2 ** 30, 1)
        key = (name.split("(")[0].replace("void ", ""), gb)
        by[key].append((grid, m))
    lines = ["# Launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
             "dram__bytes_write.sum --clock-control none)", "",
             f"Source: `{lf.relative_to(ROOT)}` of session `{tag}` (bench.py --steps 2 "
             "--warmup 3 --no-cpu --e2e-steps 1, first 400 launches). Cold-cache, "
             "serialised: compare shares, not absolutes.", "",
             f"Total launches: {len(ls)}; tc::seg_kernel launches: {len(ours)}", "",
             "| kernel | input | grid | launches | mean us | DRAM read GB | DRAM write MB |",
             "|---|---|---|---|---|---|---|"]
    tot = sum(m.get("gpu__time_duration.sum", 0) for _, _, _, m in ours)
    rd_all = []
    for key, v in by.items():
        t = statistics.mean(m["gpu__time_duration.sum"] for _, m in v) / 1e3
        rd = statistics.mean(m.get("dram__bytes_read.sum", 0) for _, m in v)
        wr = statistics.mean(m.get("dram__bytes_write.sum", 0) for _, m in v)
        kname, gb = key
        if kname.startswith("tc::seg_kernel<0,") and gb >= 1.5:  # the 2^30 sweep launches
            rd_all.extend(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                          for _, m in v)
        size = "2^30" if gb >= 1.5 else "2^27 (e2e chunk)"
        lines.append(f"| `{kname}` | {size} | {v[0][0]} | {len(v)} | {t:.1f} | {rd / 1e9:.4f} | "
                     f"{wr / 1e6:.2f} |")
    lines += ["", f"tc::seg_kernel total device time in the list: {tot / 1e6:.3f} ms"]
    (dst / "launches_summary.md").write_text("\n".join(lines) + "\n")
    if rd_all:
        (ROOT / "profiles" / "traffic.json").write_text(json.dumps({
            "per_launch_bytes": statistics.mean(rd_all),
            "what": "mean dram__bytes_read.sum + dram__bytes_write.sum per tc::seg_kernel "
                    "reduce launch of the bench sweep (2^30 fp16 input, 13 segment sizes)",
            "source": f"profiles/{rnd}/launches_summary.md",
        }, indent=1) + "\n")


if __name__ == "__main__":
    main()
