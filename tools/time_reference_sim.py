"""Time the reference's OWN CPU path -- the halftile simulator behind
cli.run / segmented_reduce (pkg/src/halftile/reduce.py:379-446), imported
from /root/reference in the build container (it cannot travel to the GPU
box) -- on bounded samples of BASELINE configs[1] / configs[2] (fp16, the
reference's default half-precision engine), next to the oracle C port that
bench.py's reference arm times.  Writes profiles/<round>/reference_sim.json.

usage: python tools/time_reference_sim.py ROUND
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import halftile  # noqa: E402  (the reference package, read-only mount)

rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
rng = np.random.default_rng(0)
rows = []
for op, n, segs in (("reduce", 1 << 22, (16, 256, 4096, 65536)), ("scan", 1 << 20, (16, 256, 4096, 16384))):
    x = rng.random(n).astype(np.float16)
    for s in segs:
        plan = halftile.select_algorithm(op, s, n)
        eng = halftile.TileEngine()
        fn = halftile.segmented_reduce if op == "reduce" else halftile.segmented_scan
        t0 = time.perf_counter()
        fn(x, s, plan.variant, eng)
        dt = time.perf_counter() - t0
        rows.append({"op": op, "n": n, "seg": s, "variant": plan.variant, "s": round(dt, 3),
                     "elems_per_s": round(n / dt, 1)})
        print(rows[-1], flush=True)
out = {
    "what": "the reference simulator (halftile, pure numpy) timed on this build container's CPU, "
            "one call per row, default TileEngine (half)",
    "host_cpus": os.cpu_count(),
    "rows": rows,
    "reduce_elems_per_s_median": float(np.median([r["elems_per_s"] for r in rows if r["op"] == "reduce"])),
    "scan_elems_per_s_median": float(np.median([r["elems_per_s"] for r in rows if r["op"] == "scan"])),
}
os.makedirs(f"profiles/{rnd}", exist_ok=True)
json.dump(out, open(f"profiles/{rnd}/reference_sim.json", "w"), indent=1)
print(json.dumps({k: v for k, v in out.items() if k != "rows"}))
