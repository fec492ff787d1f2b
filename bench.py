"""bench.py -- the driver's benchmark contract for the B200 tensor-core
segmented reduction / scan (arXiv 1811.09736).

Workload (BASELINE.json configs[1], the config the headline metric is quoted
on): segmented reduction of 2^30 fp16 elements, swept over the 13
power-of-two segment sizes 16..65536; output fp16 (the reference's default
``TileEngine(accumulate="half")``).  One STEP = one pass of the hot path
over the input at every segment size of the sweep (13 kernel launches).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 (torchrun, one process per GPU): weak scaling -- every rank owns its
own 2^30-element shard of whole segments and runs the same sweep with NO
data-path collective (segmented ops shard by whole segments, SURVEY.md
section 8(e)); the full-reduce / full-scan extras shard 2^33 elements across
the ranks and use one NCCL all_gather of per-rank fp64 partials.

Reported (rank 0, one JSON line):
  value     whole-job elements/s with inputs resident in HBM (device time,
            CUDA events, max over ranks);
  e2e       the same sweep through the public drop-in API
            (``segmented_reduce`` on pinned host tensors: H2D + kernel + D2H
            inside the timed region);
  roofline  algorithmic bytes (2n + 2*ceil(n/s) per launch) / measured
            kernel time against MEASURED_PEAKS.json's copy bandwidth;
  cpu_baseline  the C restatement of the reference oracle (oracle/oracle.c)
            on the host cores, on a bounded prefix of the same input;
  extras    scan sweep (configs[2]), full reduce / full exclusive scan of
            2^33 elements (configs[3], configs[4]).

``--impl reference`` times the reference's CPU path instead (the oracle
port, all host threads) on the same metric/config and prints the same line
with ``"impl": "reference"``.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

REDUCE_SEGS = [1 << k for k in range(4, 17)]  # 16 .. 65536
SCAN_SEGS = [1 << k for k in range(4, 15)]    # 16 .. 16384
LOG2N = 30
FULL_LOG2N = 33
METRIC = "seg reduce/scan elems/s and HBM GB/s (% of peak) vs segment size, 1/2/4/8 B200"
UNIT = "elems/s"
WORKLOAD = ("segmented reduction fp16, 2^30 elements, segment-size sweep 16-65536 "
            "(13 power-of-two sizes, one launch each per step), fp16 sums")


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def reduce_bytes(n, s, o=2):
    return 2 * n + o * (-(-n // s))


# ----------------------------------------------------------------- CPU side


def load_oracle():
    so = ROOT / "oracle" / "build" / "liboracle.so"
    if not so.exists():
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)
    lib = ctypes.CDLL(str(so))
    lib.or_seg_reduce.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                  ctypes.c_void_p, ctypes.c_int]
    lib.or_seg_reduce.restype = None
    lib.or_init()
    return lib


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_sweep(lib, xh: np.ndarray, threads: int) -> float:
    """One reference-CPU sweep over xh (all segment sizes); returns seconds."""
    n = xh.size
    outs = {s: np.empty(-(-n // s), np.float64) for s in REDUCE_SEGS}
    t0 = time.perf_counter()
    for s in REDUCE_SEGS:
        lib.or_seg_reduce(xh.ctypes.data, n, s, outs[s].ctypes.data, threads)
    return time.perf_counter() - t0


def cpu_sample_size(lib, threads, budget_s, xh_full=None):
    """Largest power-of-two prefix (<= 2^30) whose sweep takes ~budget_s."""
    probe_n = 1 << 22
    xp = xh_full[:probe_n] if xh_full is not None else synth_host(probe_n)
    cpu_sweep(lib, xp, threads)  # warm the decode table / pages
    t = cpu_sweep(lib, xp, threads)
    rate = probe_n / max(t, 1e-9)
    n = 1 << 22
    while n < (1 << LOG2N) and 2 * n / rate <= budget_s:
        n *= 2
    return n


def synth_host(n, seed=0):
    rng = np.random.default_rng(seed)
    return rng.random(n, dtype=np.float32).astype(np.float16)


def run_reference(args):
    """--impl reference: the reference's CPU path (the oracle port) on the
    host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    lib = load_oracle()
    threads = host_threads()
    n = cpu_sample_size(lib, threads, args.ref_step_seconds)
    xh = synth_host(n)
    for _ in range(args.warmup):
        cpu_sweep(lib, xh, threads)
    ts = [cpu_sweep(lib, xh, threads) for _ in range(args.steps)]
    total = sum(ts)
    value = len(REDUCE_SEGS) * n * args.steps / total
    sample = (f"sweep of {len(REDUCE_SEGS)} segment sizes over a 2^{n.bit_length() - 1}-element "
              f"prefix per step (uniform [0,1) fp16), oracle/oracle.c or_seg_reduce, "
              f"{threads} pthreads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
        "config": config_dict(args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(world):
    return {
        "workload": WORKLOAD,
        "n_per_gpu": 1 << LOG2N,
        "segment_sizes": REDUCE_SEGS,
        "out_dtype": "f16",
        "l2": "inputs 2 GiB per GPU >> 126 MB L2 (no flush needed)",
        "parallelism": f"whole-segment shards, {world} GPU(s), no data-path collective",
    }


# ----------------------------------------------------------------- GPU side


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.15)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, smax, reasons = [], None, set()
        for r in self.samples:
            try:
                sm.append(float(r[1]))
                smax = float(r[2])
                for nm, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                continue
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def hbm_read_peak(x, dev, reps=10):
    """Measured HBM read-stream bandwidth (tools/csrc/hbm_probe.cu, a plain
    16-byte streaming-load kernel) over the bench input: the roofline of a
    read-only kernel.  Best of ``reps``; None if the probe is not built."""
    import torch

    so = ROOT / "tools" / "_hbm_probe.so"
    if not so.exists():
        return None
    lib = ctypes.CDLL(str(so))
    lib.hbm_read_stream.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                                    ctypes.c_int, ctypes.c_void_p]
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    sink = torch.zeros(sms * 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    nbytes = x.numel() * x.element_size()
    best = None
    for blocks in (sms * 2, sms * 4):
        for _ in range(2):
            lib.hbm_read_stream(x.data_ptr(), nbytes, sink.data_ptr(), blocks, stream.cuda_stream)
        torch.cuda.synchronize()
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            lib.hbm_read_stream(x.data_ptr(), nbytes, sink.data_ptr(), blocks, stream.cuda_stream)
            b.record(stream)
            b.synchronize()
            gbs = nbytes / a.elapsed_time(b) / 1e6
            best = gbs if best is None else max(best, gbs)
    return round(best, 1)


def gen_device(n, device, seed):
    """Uniform [0, 1) fp16 on the device, generated in chunks."""
    import torch

    x = torch.empty(n, dtype=torch.float16, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    chunk = 1 << 28
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        x[lo:hi] = torch.rand(hi - lo, generator=g, device=device, dtype=torch.float32)
    return x


def irregular_offsets(n, mean, device, seed):
    """int64 CSR offsets over [0, n] with geometric segment lengths (mean `mean`)."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    m = int(2 * n / mean) + 16
    u = torch.rand(m, device=device, generator=g, dtype=torch.float64).clamp_min(1e-300)
    lens = torch.ceil(-torch.log(u) * (mean - 0.5)).to(torch.int64)
    ends = torch.cumsum(lens, 0)
    ends = ends[ends < n]
    z = torch.zeros(1, dtype=torch.int64, device=device)
    return torch.cat([z, ends, torch.full((1,), n, dtype=torch.int64, device=device)])


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_DIST_BACKEND=gloo (test only): several ranks may share one GPU,
    # which NCCL refuses -- used to exercise the N > 1 path on a 1-GPU box
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    import paper_1811_09736_b200 as ht
    from paper_1811_09736_b200 import _device as D
    from paper_1811_09736_b200 import _lib

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    peak, peak_src = peaks()
    n = 1 << LOG2N
    x = gen_device(n, dev, seed=1000 + rank)
    outs = {s: torch.empty(-(-n // s), dtype=torch.float16, device=dev) for s in REDUCE_SEGS}
    stream = torch.cuda.current_stream(dev)

    def sweep():
        for s in REDUCE_SEGS:
            D.seg_reduce(x, s, torch.float16, out=outs[s])

    for _ in range(args.warmup):
        sweep()
    barrier()

    # ---- timed region: K steps, per-launch CUDA events on the launch stream
    nl = len(REDUCE_SEGS)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps * nl + 1)]
    _lib.lib.tc_reset_launch_count()
    with ClockSampler(local) as clk:
        barrier()
        evs[0].record(stream)
        for k in range(args.steps):
            for i, s in enumerate(REDUCE_SEGS):
                D.seg_reduce(x, s, torch.float16, out=outs[s])
                evs[k * nl + i + 1].record(stream)
        barrier()
    launches = int(_lib.lib.tc_launch_count())
    per = [evs[j].elapsed_time(evs[j + 1]) for j in range(args.steps * nl)]
    total_ms = evs[0].elapsed_time(evs[-1])
    total_ms = max_over_ranks(total_ms)
    ms_per_step = total_ms / args.steps
    value = world * nl * n / (ms_per_step / 1e3)

    sweep_rows = []
    tot_bytes, tot_ms = 0.0, 0.0
    for i, s in enumerate(REDUCE_SEGS):
        ms = statistics.median(per[k * nl + i] for k in range(args.steps))
        b = reduce_bytes(n, s)
        tot_bytes += b
        tot_ms += ms
        sweep_rows.append({"seg": s, "ms": round(ms, 4), "gelem_s": round(n / ms / 1e6, 1),
                           "gbs": round(b / ms / 1e6, 1), "frac": round(b / ms / 1e6 / peak, 4)})
    achieved = tot_bytes / tot_ms / 1e6
    read_peak = hbm_read_peak(x, dev)
    if read_peak:
        for r in sweep_rows:
            r["frac_read"] = round(r["gbs"] / read_peak, 4)
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("per_launch_bytes")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "peak_source": peak_src,
                "read_peak": read_peak,
                "frac_read": round(achieved / read_peak, 4) if read_peak else None,
                "read_peak_source": "measured in this run: tools/csrc/hbm_probe.cu 16-B "
                                    "streaming-load kernel over the 2 GiB input, best of 20",
                "kernel": "tc::seg_kernel<OP_REDUCE,...> (13 launches/step)",
                "algorithmic_bytes": "2n + 2*ceil(n/s) per launch, n = 2^30"}

    # ---- e2e through the public drop-in API with pinned host buffers: the
    # step's input is copied host->device ONCE per step, in 8 chunks of whole
    # segments on a copy stream, and every chunk is swept (13 public-API
    # calls on the device chunk) as soon as it lands, overlapping the next
    # chunk's copy; the 13 results go back device->host into pinned buffers.
    xh = torch.empty(n, dtype=torch.float16, pin_memory=True)
    xh.copy_(x)
    eng = ht.TileEngine()
    plans = {s: ht.select_algorithm("reduce", s, n).variant for s in REDUCE_SEGS}
    nchunk = 8
    clen = n // nchunk  # multiple of every segment size (2^27 / 2^16)
    xdev = torch.empty(n, dtype=torch.float16, device=dev)
    res_h = {s: torch.empty(-(-n // s), dtype=torch.float16, pin_memory=True) for s in REDUCE_SEGS}
    copy_stream = torch.cuda.Stream(dev)
    d2h_stream = torch.cuda.Stream(dev)  # PCIe is full duplex: results go back while inputs come in
    landed = [torch.cuda.Event() for _ in range(nchunk)]
    reduced = [torch.cuda.Event() for _ in range(nchunk)]

    def e2e_sweep():
        with torch.cuda.stream(copy_stream):
            for c in range(nchunk):
                xdev[c * clen:(c + 1) * clen].copy_(xh[c * clen:(c + 1) * clen], non_blocking=True)
                landed[c].record(copy_stream)
        parts = []
        for c in range(nchunk):
            stream.wait_event(landed[c])
            xc = xdev[c * clen:(c + 1) * clen]
            outs_c = {s: ht.segmented_reduce(xc, s, plans[s], eng) for s in REDUCE_SEGS}
            reduced[c].record(stream)
            parts.append(outs_c)  # alive until the step's final synchronize
            d2h_stream.wait_event(reduced[c])
            with torch.cuda.stream(d2h_stream):
                for s in REDUCE_SEGS:
                    k = clen // s
                    res_h[s][c * k:(c + 1) * k].copy_(outs_c[s], non_blocking=True)
        d2h_stream.synchronize()
        stream.synchronize()
        return res_h

    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    e2e_sweep()
    barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_sweep()
    e1.record(stream)
    barrier()
    wall_ms = (time.perf_counter() - t0) * 1e3
    e2e_ms = max_over_ranks(max(e0.elapsed_time(e1), wall_ms)) / e2e_steps
    # the e2e path must return what the device-resident sweep computed
    for s_chk in (REDUCE_SEGS[0], REDUCE_SEGS[-1]):
        assert torch.equal(res_h[s_chk], outs[s_chk].cpu()), f"e2e result mismatch at s={s_chk}"
    e2e = {"value": world * nl * n / (e2e_ms / 1e3), "unit": UNIT,
           "h2d_bytes_per_step": 2 * n,
           "d2h_bytes_per_step": sum(2 * (-(-n // s)) for s in REDUCE_SEGS),
           "ms_per_step": round(e2e_ms, 3),
           "api": "pinned host fp16 -> 8 chunked H2D copies (copy stream) -> per chunk "
                  "paper_1811_09736_b200.segmented_reduce(chunk, s, select_algorithm(...)."
                  "variant, TileEngine()) for the 13 sizes -> per chunk D2H of its 13 "
                  "results into pinned host buffers (third stream, overlapping the next "
                  "chunks' H2D)"}
    del xh, xdev, res_h
    e2e_per_call = None
    if not args.no_per_call:
        e2e_per_call = run_e2e_per_call(args, x, dev, world, barrier, max_over_ranks, outs, plans)

    extras = {}
    if not args.no_extras:
        extras = run_extras(args, x, dev, world, rank, barrier, max_over_ranks, peak)

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if world == 1 and not args.no_cpu:
        lib = load_oracle()
        threads = host_threads()
        host = x.cpu().numpy()
        ncpu = cpu_sample_size(lib, threads, args.cpu_seconds / 2, host)
        xs = np.ascontiguousarray(host[:ncpu])
        t = min(cpu_sweep(lib, xs, threads) for _ in range(2))
        cpu = {"value": len(REDUCE_SEGS) * ncpu / t, "unit": UNIT, "cores": threads,
               "kind": "port",
               "sample": (f"same sweep on the first 2^{ncpu.bit_length() - 1} elements of the "
                          f"bench input, oracle/oracle.c or_seg_reduce (binary64), "
                          f"{threads} pthreads, best of 2")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic (uniform [0,1) fp16, torch.rand seeded per rank)",
            "config": config_dict(world),
            "gbs_per_gpu": round(achieved, 1),
            "e2e": e2e, "e2e_per_call": e2e_per_call, "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": cpu, "clocks": clk.summary(), "sweep": sweep_rows,
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e_per_call(args, x, dev, world, barrier, max_over_ranks, outs, plans):
    """The drop-in exactly as a reference user calls it: a numpy fp16 array
    in, a numpy array out, ONE public ``segmented_reduce`` call per segment
    size -- every call copies its own 2 GiB input to the device (the
    package's staged host path: pinned ring + host threads + copy stream) and
    its sums back.  Host wall clock (the numpy path synchronises), max over
    ranks; compared with the measured pinned-H2D bandwidth, the bound of a
    call that must move its input over PCIe."""
    import torch

    import paper_1811_09736_b200 as ht

    n = x.numel()
    xn = x.cpu().numpy()
    eng = ht.TileEngine()
    # pinned H2D bandwidth (the per-call bound): 2 GiB pinned -> device, best of 3
    hp = torch.empty(n, dtype=torch.float16, pin_memory=True)
    hp.copy_(x)
    dst = torch.empty_like(x)
    h2d = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst.copy_(hp, non_blocking=True)
        torch.cuda.synchronize()
        h2d = max(h2d, 2 * n / (time.perf_counter() - t0) / 1e9)
    del hp, dst
    segs = REDUCE_SEGS
    res = {s: ht.segmented_reduce(xn, s, plans[s], eng) for s in segs}  # warm the stager
    barrier()
    steps = max(1, min(args.steps, args.e2e_steps))
    t0 = time.perf_counter()
    for _ in range(steps):
        res = {s: ht.segmented_reduce(xn, s, plans[s], eng) for s in segs}
    dt = max_over_ranks(time.perf_counter() - t0) / steps
    for s_chk in (segs[0], segs[-1]):
        assert np.array_equal(res[s_chk], outs[s_chk].cpu().numpy()), f"per-call mismatch s={s_chk}"
    bound = len(segs) * 2 * n / (h2d * 1e9)
    return {"value": world * len(segs) * n / dt, "unit": UNIT, "ms_per_step": round(dt * 1e3, 2),
            "ms_per_call": round(dt * 1e3 / len(segs), 2),
            "h2d_bytes_per_step": len(segs) * 2 * n,
            "d2h_bytes_per_step": sum(2 * (-(-n // s)) for s in segs),
            "pinned_h2d_gbs": round(h2d, 1),
            "h2d_bound_ms_per_step": round(bound * 1e3, 2),
            "frac_of_h2d_bound": round(bound / dt, 4),
            "api": "numpy fp16 (pageable) -> paper_1811_09736_b200.segmented_reduce(x, s, "
                   "select_algorithm(...).variant, TileEngine()) -> numpy, one call per size, "
                   "each call copying its own input"}


def _time_op(fn, reps, warm, stream, barrier, max_over_ranks):
    import torch

    for _ in range(warm):
        fn()
    barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    barrier()
    return max_over_ranks(a.elapsed_time(b)) / reps


def dist_backend():
    import torch.distributed as dist

    return str(dist.get_backend()).upper() if dist.is_initialized() else "none"


def run_extras(args, x, dev, world, rank, barrier, max_over_ranks, peak):
    """configs[2..4]: scan sweep (1 GPU each rank), full reduce / full
    exclusive scan of 2^33 elements sharded over the ranks."""
    import torch

    from paper_1811_09736_b200 import _device as D
    from paper_1811_09736_b200 import distributed as PD

    stream = torch.cuda.current_stream(dev)
    n = x.numel()
    reps = max(3, args.steps)
    out = {}
    # segmented inclusive scan sweep, fp16 out (paper accounting 4 B/elem)
    y = torch.empty(n, dtype=torch.float16, device=dev)
    rows = []
    for s in SCAN_SEGS:
        ms = _time_op(lambda: D.seg_scan(x, s, torch.float16, out=y), reps, 2, stream, barrier,
                      max_over_ranks)
        b = 4 * n
        rows.append({"seg": s, "ms": round(ms, 4), "gelem_s": round(world * n / ms / 1e6, 1),
                     "gbs_per_gpu": round(b / ms / 1e6, 1), "frac": round(b / ms / 1e6 / peak, 4)})
    out["scan_sweep_f16"] = {"workload": "segmented inclusive scan fp16, 2^30 per GPU, fp16 out",
                             "rows": rows}
    del y
    # configs[2] with fp32 output (6 B/elem)
    y = torch.empty(n, dtype=torch.float32, device=dev)
    rows = []
    for s in SCAN_SEGS:
        ms = _time_op(lambda: D.seg_scan(x, s, torch.float32, out=y), reps, 2, stream, barrier,
                      max_over_ranks)
        b = 6 * n
        rows.append({"seg": s, "ms": round(ms, 4), "gelem_s": round(world * n / ms / 1e6, 1),
                     "gbs_per_gpu": round(b / ms / 1e6, 1), "frac": round(b / ms / 1e6 / peak, 4)})
    out["scan_sweep_f32"] = {"workload": "segmented inclusive scan fp16, 2^30 per GPU, fp32 out",
                             "rows": rows}
    del y
    # configs[1] with fp32 output
    rows = []
    for s in REDUCE_SEGS:
        o = torch.empty(-(-n // s), dtype=torch.float32, device=dev)
        ms = _time_op(lambda: D.seg_reduce(x, s, torch.float32, out=o), reps, 2, stream, barrier,
                      max_over_ranks)
        b = reduce_bytes(n, s, 4)
        rows.append({"seg": s, "ms": round(ms, 4), "gelem_s": round(world * n / ms / 1e6, 1),
                     "gbs_per_gpu": round(b / ms / 1e6, 1), "frac": round(b / ms / 1e6 / peak, 4)})
        del o
    out["reduce_sweep_f32"] = {"workload": "segmented reduce fp16, 2^30 per GPU, fp32 out",
                               "rows": rows}
    # widened rows: bf16 input, non-power-of-two segment sizes
    xb = x.to(torch.bfloat16)
    rows = []
    for s in (16, 256, 4096, 65536):
        o = torch.empty(-(-n // s), dtype=torch.float16, device=dev)
        ms = _time_op(lambda: D.seg_reduce(xb, s, torch.float16, out=o), reps, 2, stream,
                      barrier, max_over_ranks)
        b = reduce_bytes(n, s)
        rows.append({"seg": s, "ms": round(ms, 4), "gbs_per_gpu": round(b / ms / 1e6, 1),
                     "frac": round(b / ms / 1e6 / peak, 4)})
    out["reduce_bf16_input"] = {"workload": "segmented reduce, 2^30 bf16 per GPU, fp16 out",
                                "rows": rows}
    del xb
    rows = []
    y = torch.empty(n, dtype=torch.float16, device=dev)
    y32 = torch.empty(n, dtype=torch.float32, device=dev)
    for s in (3, 7, 17, 33, 48, 63, 300, 1000, 4097, 100000, 100001):
        o = torch.empty(-(-n // s), dtype=torch.float16, device=dev)
        ms = _time_op(lambda: D.seg_reduce(x, s, torch.float16, out=o), reps, 2, stream,
                      barrier, max_over_ranks)
        b = reduce_bytes(n, s)
        ms2 = _time_op(lambda: D.seg_scan(x, s, torch.float16, out=y), reps, 2, stream,
                       barrier, max_over_ranks)
        ms3 = _time_op(lambda: D.seg_scan(x, s, torch.float32, out=y32), reps, 2, stream,
                       barrier, max_over_ranks)
        rows.append({"seg": s, "reduce_ms": round(ms, 4),
                     "reduce_frac": round(b / ms / 1e6 / peak, 4), "scan_ms": round(ms2, 4),
                     "scan_frac": round(4 * n / ms2 / 1e6 / peak, 4),
                     "scan_f32_ms": round(ms3, 4),
                     "scan_f32_frac": round(6 * n / ms3 / 1e6 / peak, 4),
                     "modes": {"reduce": D.plan_info("reduce", n, s)[0],
                               "scan_f16": D.plan_info("scan", n, s)[0],
                               "scan_f32": D.plan_info("scan", n, s, torch.float32)[0]}})
    out["non_pow2_segments"] = {"workload": "segmented reduce (fp16 out) / inclusive scan (fp16 "
                                            "and fp32 out), 2^30 fp16, ragged last segment",
                                "rows": rows}
    del y, y32
    # irregular (CSR-offset) segments: geometric lengths
    rows = []
    y = torch.empty(n, dtype=torch.float32, device=dev)
    for mean in (64, 1024, 16384):
        off = irregular_offsets(n, mean, dev, seed=11 + rank)
        nseg = off.numel() - 1
        o = torch.empty(nseg, dtype=torch.float32, device=dev)
        ms = _time_op(lambda: D.irreg_reduce(x, off, torch.float32, out=o, validate=False), reps,
                      2, stream, barrier, max_over_ranks)
        b = 2 * n + 8 * (nseg + 1) + 4 * nseg
        ms2 = _time_op(lambda: D.irreg_scan(x, off, torch.float32, out=y, validate=False), reps,
                       2, stream, barrier, max_over_ranks)
        b2 = 2 * n + 8 * (nseg + 1) + 4 * n
        rows.append({"mean_seg": mean, "nseg": nseg, "reduce_ms": round(ms, 4),
                     "reduce_frac": round(b / ms / 1e6 / peak, 4), "scan_ms": round(ms2, 4),
                     "scan_frac": round(b2 / ms2 / 1e6 / peak, 4)})
        del off, o
    out["irregular_segments"] = {
        "workload": "irregular segmented reduce / inclusive scan, 2^30 fp16, int64 CSR offsets, "
                    "geometric segment lengths, fp32 out",
        "bytes": "2n + 8(nseg+1) + 4 nseg (reduce), 2n + 8(nseg+1) + 4n (scan)", "rows": rows}
    del y
    # batch-norm statistics consumer, ResNet-50 conv2_x activation shape
    xbn = gen_device(256 * 256 * 56 * 56, dev, seed=21 + rank).view(256, 256, 56, 56)
    ms = _time_op(lambda: D.bn_stats(xbn), reps, 2, stream, barrier, max_over_ranks)
    # the same call replayed from a CUDA graph: device time without the
    # Python call overhead (~20 us per call at this size)
    g = torch.cuda.CUDAGraph()
    D.bn_stats(xbn)
    torch.cuda.synchronize(dev)
    with torch.cuda.graph(g):
        D.bn_stats(xbn)
    msg = _time_op(g.replay, reps, 2, stream, barrier, max_over_ranks)
    nb = xbn.numel()
    out["batch_norm_stats"] = {
        "workload": "per-channel mean + biased variance, NCHW fp16 (256, 256, 56, 56), fp32 out",
        "ms": round(ms, 4), "gelem_s": round(nb / ms / 1e6, 1),
        "gbs_algorithmic": round(2 * nb / ms / 1e6, 1),
        "frac_algorithmic": round(2 * nb / ms / 1e6 / peak, 4),
        "ms_graph": round(msg, 4), "frac_algorithmic_graph": round(2 * nb / msg / 1e6 / peak, 4),
        "gbs_actual": round(2 * nb / ms / 1e6, 1),
        "passes": "one read of x (tc_bn_stats: per-channel streaming kernel, shifted moments, "
                  "last-block fp64 combine; one launch)"}
    del g
    del xbn
    # full ops over 2^33 elements sharded across the ranks
    nf = 1 << FULL_LOG2N
    lo, hi = PD.even_bounds(nf, world, rank)
    xl = gen_device(hi - lo, dev, seed=7 + rank)
    def freduce():
        if world > 1:
            return PD.sharded_full_reduce(xl, torch.float32)
        return D.full_reduce(xl, torch.float32)

    ms = _time_op(freduce, reps, 2, stream, barrier, max_over_ranks)
    b = 2 * (hi - lo) + 4
    out["full_reduce_2^33"] = {"ms": round(ms, 4), "gelem_s": round(nf / ms / 1e6, 1),
                               "gbs_per_gpu": round(b / ms / 1e6, 1),
                               "frac": round(b / ms / 1e6 / peak, 4),
                               "exchange": (f"{dist_backend()} all_gather of fp64 partials"
                                            if world > 1 else "none")}
    yl = torch.empty(hi - lo, dtype=torch.float32, device=dev)

    def fscan():
        if world > 1:
            return PD.sharded_full_scan(xl, torch.float32, exclusive=True)
        return D.full_scan(xl, torch.float32, exclusive=True, out=yl)

    ms = _time_op(fscan, reps, 2, stream, barrier, max_over_ranks)
    b = 6 * (hi - lo)
    actual = b + (2 * (hi - lo) if world > 1 else 0)
    out["full_exclusive_scan_2^33"] = {
        "ms": round(ms, 4), "gelem_s": round(nf / ms / 1e6, 1),
        "gbs_per_gpu_algorithmic": round(b / ms / 1e6, 1),
        "frac": round(b / ms / 1e6 / peak, 4),
        "gbs_per_gpu_actual": round(actual / ms / 1e6, 1), "out_dtype": "f32"}
    del xl, yl
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="approximate CPU-baseline budget (ours arm)")
    ap.add_argument("--ref-step-seconds", type=float, default=4.0,
                    help="approximate seconds per reference-arm step")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-per-call", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # contract: W >= 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
