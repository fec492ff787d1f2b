"""Aggregate an ncu SASS source-page CSV (per-instruction stall samples) onto
CUDA source lines, using the cubin's line table (nvdisasm -g).

usage: python tools/ncu_lines.py SOURCE.csv CUBIN KERNEL_MANGLED [N]
"""
import collections
import csv
import re
import subprocess
import sys


def line_table(cubin, fn):
    out = subprocess.run(["/usr/local/cuda/bin/nvdisasm", "-g", "-c", cubin],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    start = [i for i, ln in enumerate(lines) if ln.startswith("//----") and f".text.{fn} " in ln][0]
    cur = None
    table = {}
    for ln in lines[start + 1:]:
        if ln.startswith("//----"):
            break
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            table[int(m.group(1), 16)] = cur
    return table


def main():
    src, cubin, fn = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
    h = rows[hi]
    ia, iw, ie = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    data = [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
    base = int(data[0][ia], 16)
    table = line_table(cubin, fn)
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for r in data:
        off = int(r[ia], 16) - base
        key = table.get(off, "?")
        agg[key][0] += float(r[iw] or 0)
        agg[key][1] += float(r[ie] or 0)
    tot = sum(v[0] for v in agg.values()) or 1
    toti = sum(v[1] for v in agg.values()) or 1
    print(f"{len(table)} mapped instrs; stall samples {tot:.0f}; warp instrs {toti:.0f}")
    for k, (w, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"  {100 * w / tot:5.1f}% stall {100 * e / toti:5.1f}% instr  {k}")


if __name__ == "__main__":
    main()
