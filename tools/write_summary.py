"""Write profiles/<round>/SUMMARY.md from the distilled bench / ncu files.
usage: python tools/write_summary.py ROUND SESSION_TAG TESTS_PASSED"""
import glob
import json
import os
import re
import sys

rnd, tag, passed = sys.argv[1], sys.argv[2], sys.argv[3]
D = f"profiles/{rnd}"
d = json.load(open(f"{D}/bench.json"))
r = json.load(open(f"{D}/bench_ref.json"))
ex = d["extras"]
L = [f"# Round {rnd.lstrip('r').lstrip('0')} profile summary (session {tag}, one B200)\n"]
L.append(f"All numbers below come from `bench.json` / `bench_ref.json` / `ncu_*.txt` / `launches_summary.md` in this directory (one gpurun session, this round's code; `pytest_gpu.log`: {passed} GPU tests passed, `smoke.log` ok). Peak = measured copy bandwidth {d['roofline']['peak']:.1f} GB/s (`MEASURED_PEAKS.json`); read-dominated kernels can exceed it (a pure read stream is not bounded by the copy figure).\n")
L.append("## Headline (BASELINE configs[1]: segmented reduce, 2^30 fp16, s = 16..65536)\n")
L.append(f"* value: {d['value']/1e9:.0f} Gelem/s device-resident ({d['ms_per_step']:.2f} ms per 13-launch sweep); roofline {d['roofline']['achieved']} GB/s = {100*d['roofline']['frac']:.1f} % of measured copy; DRAM traffic per launch {d['roofline']['traffic']/1e9:.3f} GB vs algorithmic 2.147-2.281 GB.")
L.append(f"* e2e (pinned host -> chunked H2D -> public API -> D2H): {d['e2e']['value']/1e9:.0f} Gelem/s ({d['e2e']['ms_per_step']} ms/step, PCIe-bound: 2 GiB H2D per step).")
pc = d.get("e2e_per_call")
if pc:
    L.append(f"* e2e per call (numpy in -> numpy out, one public call per size, each copying its own 2 GiB pageable input through the native stager): {pc['ms_per_call']} ms per call = {100*pc['frac_of_h2d_bound']:.0f} % of the pinned-H2D bound ({pc['pinned_h2d_gbs']} GB/s).")
L.append(f"* reference arm (oracle/oracle.c, {r['cpu_baseline']['cores']} host threads): {r['value']/1e9:.1f} Gelem/s -> e2e / reference = {d['e2e']['value']/r['value']:.1f}x; device / reference = {d['value']/r['value']:.0f}x.")
L.append(f"* clocks during the timed region: {d['clocks']}.\n")
L.append("| s | ms | Gelem/s | GB/s | % of copy |\n|---|---|---|---|---|")
for row in d["sweep"]:
    L.append(f"| {row['seg']} | {row['ms']} | {row['gelem_s']} | {row['gbs']} | {100*row['frac']:.1f} |")
L.append("\n## Other configs and widened rows (bench extras)\n")
L.append("| config | ms | GB/s | % of copy |\n|---|---|---|---|")
for row in ex["scan_sweep_f16"]["rows"]:
    L.append(f"| seg scan fp16->fp16 2^30, s={row['seg']} | {row['ms']} | {row['gbs_per_gpu']} | {100*row['frac']:.1f} |")
fr, fs = ex["full_reduce_2^33"], ex["full_exclusive_scan_2^33"]
L.append(f"| full reduce 2^33 -> fp32 | {fr['ms']} | {fr['gbs_per_gpu']} | {100*fr['frac']:.1f} |")
L.append(f"| full exclusive scan 2^33 -> fp32 | {fs['ms']} | {fs['gbs_per_gpu_algorithmic']} | {100*fs['frac']:.1f} |")
for row in ex["reduce_bf16_input"]["rows"]:
    L.append(f"| seg reduce bf16 in, s={row['seg']} | {row['ms']} | {row['gbs_per_gpu']} | {100*row['frac']:.1f} |")
for row in ex["non_pow2_segments"]["rows"]:
    m = row.get("modes", {})
    f32 = f" / {100*row['scan_f32_frac']:.1f} (f32 out)" if "scan_f32_frac" in row else ""
    L.append(f"| non-pow2 s={row['seg']} reduce / scan (fp16 out){' / scan (fp32 out)' if f32 else ''} {m} | {row['reduce_ms']} / {row['scan_ms']} | | {100*row['reduce_frac']:.1f} / {100*row['scan_frac']:.1f}{f32} |")
for row in ex["irregular_segments"]["rows"]:
    L.append(f"| irregular (CSR) mean {row['mean_seg']} ({row['nseg']} segs) reduce / scan, fp32 out | {row['reduce_ms']} / {row['scan_ms']} | | {100*row['reduce_frac']:.1f} / {100*row['scan_frac']:.1f} |")
bn = ex["batch_norm_stats"]
L.append(f"| batch-norm stats NCHW (256,256,56,56) | {bn['ms']} (graph {bn.get('ms_graph')}) | {bn['gbs_algorithmic']} | {100*bn['frac_algorithmic']:.1f} (one read) |")
for row in ex.get("scan_sweep_f32", {}).get("rows", []):
    L.append(f"| seg scan fp16->fp32 2^30, s={row['seg']} | {row['ms']} | {row['gbs_per_gpu']} | {100*row['frac']:.1f} |")
L.append("\n## ncu --set full captures (2^30 inputs unless noted)\n")
L.append("| capture | duration | DRAM read | DRAM write | regs | grid |\n|---|---|---|---|---|---|")
for f in sorted(glob.glob(f"{D}/ncu_*.txt")):
    t = open(f).read()

    def g(k):
        m = re.search(k + r"\s+([0-9.]+ ?\S*)", t)
        return m.group(1) if m else "?"
    L.append(f"| {os.path.basename(f)[4:-4]} | {g('gpu__time_duration.sum')} | {g('dram__bytes_read.sum')} | {g('dram__bytes_write.sum')} | {g('launch__registers_per_thread')} | {g('launch__grid_size')} |")
L.append(open("tools/summary_tail.md").read())
open(f"{D}/SUMMARY.md", "w").write("\n".join(L))
