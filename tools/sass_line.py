"""Map SASS offsets of one kernel (nvdisasm -g listing) to CUDA source lines.

usage: python tools/sass_line.py KERNEL.sass OFFSET_HEX [OFFSET_HEX ...]
The listing comes from `nvdisasm -g -c <cubin>` cut to one .text section;
ncu's PCs map to these offsets by subtracting the function base (find it by
matching one hot instruction's branch distance)."""
import re
import sys

cur = None
table = []
for ln in open(sys.argv[1]):
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}"
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m:
        table.append((int(m.group(1), 16), cur, m.group(2).strip()))
for h in sys.argv[2:]:
    a = int(h, 16)
    best = [t for t in table if t[0] == a]
    print(h, best[0][1] if best else "?", best[0][2] if best else "")
