"""Generate tests/golden/halftile_golden.npz from the REAL reference package.

Run in the build container (the reference is importable only here):

    python tests/golden/make_golden.py

It imports ``halftile`` read-only from /root/reference/pkg/src and records,
for a fixed list of cases, the binary16 input bits, the reference
simulator's output (its own tile-MMA algorithms, half and single
accumulate) and the reference's exact oracle (oracle.py:47-75 applied
through pad_segmented exactly as cli._check_against_oracle does,
cli.py:113-124).  It also records the known-answer tests of
pkg/tests/test_reduce.py and pkg/tests/test_scan.py.  Nothing at test or
bench time reads /root/reference: only this file's output travels.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent / "halftile_golden.npz"


def main():
    sys.path.insert(0, REF)
    import halftile as H  # noqa: E402

    rng = np.random.default_rng(20260810)  # pkg/tests/conftest.py:27-29
    arrays = {}
    manifest = []

    def exact_int(total, seg, cap=2048, hi=8):
        # pkg/tests/conftest.py:7-19
        x = rng.integers(0, hi, total).astype(np.float64)
        segs = x.reshape(-1, seg)
        segs[segs.cumsum(axis=1) > cap] = 0
        return segs.reshape(-1).astype(np.float16)

    def add(kind, op, variant, seg, x, accs=("half", "single"), inclusive=True):
        k = len(manifest)
        arrays[f"x{k}"] = x.view(np.uint16)
        entry = dict(id=k, kind=kind, op=op, variant=variant, seg=int(seg), n=int(x.size),
                     inclusive=bool(inclusive))
        for acc in accs:
            eng = H.TileEngine(accumulate=acc)
            if op == "reduce":
                out = H.segmented_reduce(x, seg, variant, eng)
            else:
                out = H.segmented_scan(x, seg, variant, eng, inclusive=inclusive)
            arrays[f"sim_{acc}{k}"] = np.asarray(out).astype(np.float64)
        # exact oracle through pad_segmented (cli.py:113-124)
        s_eff = x.size if variant == "grid" else seg
        sv = H.pad_segmented(x, s_eff)
        if op == "reduce":
            ex = H.oracle_segmented_reduce(sv.data, sv.seg_size)[: sv.n_logical_segments]
        else:
            ex = sv.unpad_scan(H.oracle_segmented_scan(sv.data, sv.seg_size))
            if not inclusive:
                e = ex.reshape(-1, s_eff).copy()
                sh = np.zeros_like(e)
                sh[:, 1:] = e[:, :-1]
                ex = sh.reshape(-1)
        arrays[f"exact{k}"] = np.asarray(ex, dtype=np.float64)
        manifest.append(entry)

    red = [("warp16", [16]), ("warp256", [256]), ("strided16n", [16, 32, 48, 64, 80, 272]),
           ("coalesced16n", [16, 48, 272, 512]), ("efficient256n", [256, 300, 1024, 4096]),
           ("inefficient256n", [256, 300, 1024]), ("block256n", [256, 300, 2048, 4096])]
    scn = [("warp16", [16]), ("warp256", [256]), ("strided16n", [16, 32, 48, 80]),
           ("warp256n", [256, 300, 1024, 4096]), ("block256n", [256, 300, 2048])]
    for variant, segs in red:
        for seg in segs:
            add("exact_int", "reduce", variant, seg, exact_int(seg * 8, seg))
            add("ragged_int", "reduce", variant, seg, exact_int(seg * 7, seg)[: seg * 6 + seg // 2 + 1])
            add("uniform", "reduce", variant, seg,
                rng.random(seg * 6, dtype=np.float32).astype(np.float16))
    for variant, segs in scn:
        for seg in segs:
            add("exact_int", "scan", variant, seg, exact_int(seg * 8, seg))
            add("ragged_int", "scan", variant, seg, exact_int(seg * 7, seg)[: seg * 6 + seg // 2 + 1])
            add("uniform", "scan", variant, seg,
                rng.random(seg * 6, dtype=np.float32).astype(np.float16))
            add("exact_int_excl", "scan", variant, seg, exact_int(seg * 4, seg), inclusive=False)
    for n in (1000, 3000, 4096, 3 * 4096 + 256, 1 << 14):
        x = exact_int(1 << 14, 1 << 14)[:n]
        add("grid_int", "reduce", "grid", n, x)
        add("grid_int", "scan", "grid", n, x)
    x = rng.random(5000, dtype=np.float32).astype(np.float16)
    add("grid_uniform", "reduce", "grid", 5000, x)
    add("grid_uniform", "scan", "grid", 5000, x)

    # known-answer tests (pkg/tests/test_reduce.py, test_scan.py)
    e = H.TileEngine
    kats = {
        "reduce_16_arange": (np.arange(1, 257, dtype=np.float16), H.reduce_16(np.arange(1, 257, dtype=np.float16), e())),
        "reduce_256_zeros": (np.zeros(256, np.float16), [H.reduce_256(np.zeros(256, np.float16), e())]),
        "reduce_256_ones": (np.ones(256, np.float16), [H.reduce_256(np.ones(256, np.float16), e())]),
        "reduce_256_halves": (np.full(256, 0.5, np.float16), [H.reduce_256(np.full(256, 0.5, np.float16), e())]),
        "efficient_1024_ones": (np.ones(1024, np.float16), [H.reduce_256n_efficient(np.ones(1024, np.float16), 4, e())]),
        "strided_512_ones_seg32": (np.ones(512, np.float16), H.reduce_16n_strided(np.ones(512, np.float16), 32, e())),
        "coalesced_seg512_ones": (np.ones(16 * 512, np.float16), H.reduce_16n_coalesced(np.ones(16 * 512, np.float16), 512, e())),
        "block_wpb4_4096_ones": (np.ones(4096, np.float16), [H.block_reduce_256n(np.ones(4096, np.float16), H.BlockConfig(wpb=4), e())]),
        "grid_1024_ones": (np.ones(1024, np.float16), [H.grid_reduce(np.ones(1024, np.float16), e())]),
        "grid_100_ones": (np.ones(100, np.float16), [H.grid_reduce(np.ones(100, np.float16), e())]),
        "scan_16_ones": (np.ones(256, np.float16), H.scan_16(np.ones(256, np.float16), e())),
        "scan_256_ones": (np.ones(256, np.float16), H.scan_256(np.ones(256, np.float16), e())),
        "scan_16n_512_ones_seg32": (np.ones(512, np.float16), H.scan_16n(np.ones(512, np.float16), 32, e())),
        "scan_256n_512_ones": (np.ones(512, np.float16), H.scan_256n(np.ones(512, np.float16), 2, e())),
        "block_scan_wpb4_4096_ones": (np.ones(4096, np.float16), H.block_scan_256n(np.ones(4096, np.float16), H.BlockConfig(wpb=4), e())),
        "grid_scan_4096_ones_blk1024": (np.ones(4096, np.float16), H.grid_scan(np.ones(4096, np.float16), e(), block_elems=1024)),
    }
    kat_names = []
    for name, (xin, out) in kats.items():
        arrays[f"kat_x_{name}"] = np.asarray(xin, np.float16).view(np.uint16)
        arrays[f"kat_y_{name}"] = np.asarray(out, dtype=np.float64)
        kat_names.append(name)
    # last_column_scan_16 KATs (test_scan.py:177-205): tile whose last column is col
    for name, col, carry in (("ones", np.ones(16), 0.0), ("seq", np.arange(1, 17), 0.0),
                             ("ones_carry5", np.ones(16), 5.0)):
        buf = np.zeros(256, np.float16)
        buf[15::16] = col
        frag = e().load_tile(buf, 0, H.Layout.ROW_MAJOR, 16, H.FragmentKind.MATRIX_A)
        arrays[f"lcs_tile_{name}"] = buf.view(np.uint16)
        arrays[f"lcs_y_{name}"] = np.asarray(H.last_column_scan_16(frag, e(), carry=carry), np.float64)
        arrays[f"lcs_carry_{name}"] = np.array([carry])
    # select_algorithm table (plan.py:46-77)
    plan = []
    for op in ("reduce", "scan"):
        for s in (1, 2, 15, 16, 17, 32, 48, 255, 256, 257, 4096, 2 ** 15, 2 ** 15 + 1, 2 ** 20):
            plan.append([op, s, None, H.select_algorithm(op, s).variant])
            plan.append([op, s, 4096, H.select_algorithm(op, s, total_len=4096).variant])
    meta = dict(manifest=manifest, kats=kat_names, plan=plan,
                generator="tests/golden/make_golden.py", reference="/root/reference/pkg (halftile 0.1.0)",
                numpy=np.__version__)
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {len(manifest)} cases, {len(kat_names)} KATs)")


if __name__ == "__main__":
    main()
