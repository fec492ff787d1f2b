"""Facade parity on the GPU: the CLI ``run``/``main`` and the sklearn
transformers routed through the sm_100a kernels, against the oracle
(mirrors pkg/tests/test_cli.py and pkg/tests/test_estimators.py; the cost
columns count B200 tcgen05.mma / TMA tiles, not the simulator's 16x16 MMAs).
"""

import subprocess
import sys

import numpy as np
import pytest
from sklearn.pipeline import Pipeline

import paper_1811_09736_b200 as ht
from paper_1811_09736_b200 import cli
from paper_1811_09736_b200.cli import CSV_HEADER, _check_against_oracle, main, run
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def write_f16(path, values):
    path.write_bytes(ht.halves_to_bytes(np.asarray(values, np.float16)))


def test_run_reduce_and_scan(cuda, rng):
    out, rep = run("reduce", np.ones(4096, np.float16), 16, check=True)
    assert out.size == 256 and np.all(out == 16.0)
    assert rep.check == "pass" and rep.variant == "warp16"
    out, rep = run("scan", np.ones(256, np.float16), 256, algo="warp256", check=True)
    assert out.tolist() == list(range(1, 257)) and rep.check == "pass"
    assert rep.counters.mma_count == 4 and rep.counters.tile_loads == 1  # one 8192-elem tile
    _, rep = run("reduce", np.ones(300, np.float16), 256)
    assert rep.padded_elements == 212 and rep.check == "skipped"


def test_every_variant_passes_check(cuda, rng):
    x = O.exact_int_segments(rng, 8192, 512)
    for algo in ("strided16n", "coalesced16n", "efficient256n", "inefficient256n",
                 "block256n", "grid"):
        assert run("reduce", x, 512, algo=algo, check=True)[1].check == "pass", algo
    for algo in ("strided16n", "warp256n", "block256n", "grid"):
        assert run("scan", x, 512, algo=algo, check=True)[1].check == "pass", algo


def test_check_detects_wrong_output(cuda, rng):
    x = O.exact_int_segments(rng, 512, 16)
    good = x.reshape(-1, 16).astype(np.float64).sum(axis=1)
    assert _check_against_oracle("reduce", x, 16, good) == "pass"
    bad = good.copy()
    bad[3] += 1000.0
    assert _check_against_oracle("reduce", x, 16, bad) == "fail"


def test_main_end_to_end(cuda, tmp_path, rng, monkeypatch, capsys):
    inp, outp, csvp = tmp_path / "in.f16", tmp_path / "o.f16", tmp_path / "c.csv"
    x = O.exact_int_segments(rng, 1024, 16)
    write_f16(inp, x)
    assert main(["reduce", "--input", str(inp), "--output", str(outp),
                 "--segment-size", "16", "--check"]) == 0
    got = ht.halves_from_bytes(outp.read_bytes())
    assert np.array_equal(got, O.ref_seg_reduce(x, 16).astype(np.float16))
    for _ in range(2):
        assert main(["reduce", "--input", str(inp), "--output", str(outp),
                     "--segment-size", "16", "--cost-csv", str(csvp)]) == 0
    lines = csvp.read_text().strip().split("\n")
    assert lines[0] == CSV_HEADER and len(lines) == 3
    # text format, scan, strict flag accepted
    tin, tout = tmp_path / "in.txt", tmp_path / "o.txt"
    tin.write_text("\n".join(["1"] * 300) + "\n")
    assert main(["scan", "--input", str(tin), "--output", str(tout), "--segment-size", "256",
                 "--strict-wmma", "--check"]) == 0
    assert ht.parse_half_text(tout.read_text())[-1] == 44.0  # ragged 44-element tail
    # env threshold changes the reported variant
    monkeypatch.setenv("TCU_THRESHOLD_BLOCK", "1024")
    y = O.exact_int_segments(rng, 8192, 4096)
    write_f16(inp, y)
    capsys.readouterr()
    main(["reduce", "--input", str(inp), "--output", str(outp), "--segment-size", "4096"])
    assert "variant=block256n" in capsys.readouterr().out


def test_failed_check_exits_1(cuda, tmp_path, rng, monkeypatch):
    real_run = cli.run

    def tampered(*a, **k):
        out, rep = real_run(*a, **k)
        rep.check = "fail"
        return out, rep

    monkeypatch.setattr(cli, "run", tampered)
    inp = tmp_path / "in.f16"
    write_f16(inp, O.exact_int_segments(rng, 512, 16))
    assert main(["reduce", "--input", str(inp), "--output", str(tmp_path / "o.f16"),
                 "--segment-size", "16", "--check"]) == 1


def test_console_entrypoint_and_determinism(cuda, tmp_path, rng):
    inp = tmp_path / "in.f16"
    write_f16(inp, O.exact_int_segments(rng, 4096, 64))
    outs = []
    for i in range(2):
        outp = tmp_path / f"o{i}.f16"
        proc = subprocess.run([sys.executable, "-m", "paper_1811_09736_b200.cli", "reduce",
                               "--input", str(inp), "--output", str(outp), "--segment-size",
                               "64", "--check"], capture_output=True, text=True)
        assert proc.returncode == 0, proc.stderr
        assert "check=pass" in proc.stdout
        outs.append(outp.read_bytes())
    assert outs[0] == outs[1]


def test_estimator_values(cuda, rng):
    x = np.stack([O.exact_int_segments(rng, 1024, 64) for _ in range(3)])
    out = ht.SegmentedReduce(segment_size=64).fit(x).transform(x)
    assert out.shape == (3, 16)
    for row_in, row_out in zip(x, out):
        assert np.array_equal(row_out, O.ref_seg_reduce(row_in, 64).astype(np.float16))
    y = O.exact_int_segments(rng, 2048, 128)
    sc = ht.SegmentedScan(segment_size=128).fit(y).transform(y)
    assert sc.shape == y.shape and np.array_equal(sc, O.ref_seg_scan(y, 128).astype(np.float16))
    v = O.exact_int_segments(rng, 512, 16)
    r = ht.SegmentedReduce(segment_size=16).fit(v).transform(v)
    assert r.ndim == 1 and r.size == 32
    # rows whose length is not a segment multiple: per-row launches, ragged tails
    z = np.stack([O.exact_int_segments(rng, 300, 300) for _ in range(4)])
    zr = ht.SegmentedReduce(segment_size=64).fit(z).transform(z)
    assert zr.shape == (4, 5)
    for row_in, row_out in zip(z, zr):
        assert np.array_equal(row_out, O.ref_seg_reduce(row_in, 64).astype(np.float16))
    est = ht.SegmentedReduce(segment_size=16).fit(v)
    est.transform(v)
    assert est.counters_.mma_count == 4
    single = ht.SegmentedScan(segment_size=256, accumulate="single").fit(y).transform(y)
    assert single.dtype == np.float32


def test_estimator_pipeline_and_strict(cuda, rng):
    x = O.exact_int_segments(rng, 1024, 16).reshape(2, 512)
    pipe = Pipeline([("scan", ht.SegmentedScan(segment_size=16)),
                     ("reduce", ht.SegmentedReduce(segment_size=512, algo="efficient256n"))])
    out = pipe.fit_transform(x)
    assert out.shape == (2, 1)
    exp = [O.ref_seg_reduce(O.ref_seg_scan(r, 16).astype(np.float16), 512)[0] for r in x]
    assert np.array_equal(out[:, 0], np.array(exp).astype(np.float16))
    y = O.exact_int_segments(rng, 2048, 256)
    relaxed = ht.SegmentedScan(segment_size=256).fit(y).transform(y)
    strict = ht.SegmentedScan(segment_size=256, strict_wmma=True).fit(y).transform(y)
    assert np.array_equal(relaxed, strict)
