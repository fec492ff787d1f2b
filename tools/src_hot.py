"""Instruction-count / stall hot blocks of an ncu source-page CSV (SASS)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Address" in r][0]
h = rows[hi]
data = rows[hi + 1:]
ia, isrc = h.index("Address"), h.index("Source")
ie, iw = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[ie] or 0) for r in data)
totw = sum(float(r[iw] or 0) for r in data)
print(f"total warp instrs {tot:.0f}  stall samples {totw:.0f}")
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 32
blocks = collections.OrderedDict()
for k, r in enumerate(data):
    b = blocks.setdefault(k // blk, [0.0, 0.0, r[ia][-5:], []])
    b[0] += float(r[ie] or 0)
    b[1] += float(r[iw] or 0)
    b[3].append(r[isrc].strip()[:48])
for b, (e, w, ad, src) in sorted(blocks.items(), key=lambda kv: -kv[1][0])[:12]:
    print(f"block {b} @{ad}: {100 * e / tot:5.1f}% instr {100 * w / totw:5.1f}% stall")
    print("     " + " | ".join(src[:6]))
