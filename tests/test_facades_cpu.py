"""Facade parity that needs no GPU: binary16 codecs, CLI parsing / CSV /
exit codes for unusable input, validation, sklearn protocol (mirrors the
host-side parts of pkg/tests/test_cli.py and pkg/tests/test_estimators.py)."""

import io

import numpy as np
import pytest
from sklearn.base import clone

import paper_1811_09736_b200 as ht
from paper_1811_09736_b200.segmented import padded_extent as _padding
from paper_1811_09736_b200.cli import (CSV_HEADER, emit_cost_csv, main, read_values,
                                       write_values)
from paper_1811_09736_b200.errors import BadConfigError, BadLengthError, ParseError
from paper_1811_09736_b200.estimators import _as_batch, _positive
from oracle import oracle as O


def test_f16_codec_roundtrip_all_bit_patterns():
    bits = np.arange(1 << 16, dtype=np.uint16)
    vals = bits.view(np.float16)
    back = ht.halves_from_bytes(ht.halves_to_bytes(vals))
    assert np.array_equal(back.view(np.uint16), bits)  # NaN payloads included
    assert ht.halves_to_bytes(np.array([1.0], np.float16)) == b"\x00\x3c"  # little endian
    with pytest.raises(ParseError):
        ht.halves_from_bytes(b"\x00")


def test_text_codec():
    assert np.array_equal(ht.parse_half_text("1.5\n# c\n\n-2e0\n0\n"),
                          np.array([1.5, -2.0, 0.0], np.float16))
    assert ht.format_half_text(np.array([1.5, -2.0], np.float16)) == "1.5\n-2.0\n"
    with pytest.raises(ParseError):
        ht.parse_half_text("1.0\nbogus\n")


def test_file_formats(tmp_path, rng):
    vals = O.exact_int_segments(rng, 512, 16)
    p = tmp_path / "x.f16"
    write_values(str(p), vals)
    assert np.array_equal(read_values(str(p)).view(np.uint16), vals.view(np.uint16))
    p2 = tmp_path / "x.txt"
    write_values(str(p2), np.array([1.5, -2.0, 0.0], np.float16))
    assert np.array_equal(read_values(str(p2)), np.array([1.5, -2.0, 0.0], np.float16))
    p3 = tmp_path / "data.bin"
    write_values(str(p3), np.ones(4, np.float16), "f16")
    assert np.array_equal(read_values(str(p3), "f16"), np.ones(4, np.float16))


def test_csv_header_and_padding():
    buf = io.StringIO()
    emit_cost_csv([], buf)
    assert buf.getvalue() == CSV_HEADER + "\n"
    # pad_segmented(ones(300), 256): two 256-segments -> 212 padded elements
    assert _padding(300, 256) == (512, 212)
    assert _padding(4096, 16) == (4096, 0)


def test_unusable_input_exits_2(tmp_path):
    bad = tmp_path / "in.txt"
    bad.write_text("1.0\nbogus\n")
    assert main(["scan", "--input", str(bad), "--output", str(tmp_path / "o.txt"),
                 "--segment-size", "16"]) == 2
    assert main(["reduce", "--input", str(tmp_path / "nope.f16"),
                 "--output", str(tmp_path / "o.f16"), "--segment-size", "16"]) == 2
    empty = tmp_path / "e.f16"
    empty.write_bytes(b"")
    assert main(["reduce", "--input", str(empty), "--output", str(tmp_path / "o.f16"),
                 "--segment-size", "16"]) == 2


def test_validation_helpers():
    b, was_1d = _as_batch([1, 2])
    assert b.dtype == np.float16 and b.shape == (1, 2) and was_1d
    for bad in ([], np.ones((2, 0)), np.ones((2, 2, 2)), np.array(["a"])):
        with pytest.raises(BadLengthError):
            _as_batch(bad)
    b, was_1d = _as_batch(np.ones((3, 8)))
    assert b.shape == (3, 8) and not was_1d
    with pytest.raises(BadConfigError):
        _positive("wpb", 0)
    with pytest.raises(BadConfigError):
        _positive("wpb", 2.0)
    assert _positive("wpb", np.int64(3)) == 3


def test_estimator_protocol(rng):
    est = ht.SegmentedReduce(segment_size=64, wpb=8)
    params = est.get_params()
    assert params["segment_size"] == 64 and params["wpb"] == 8
    est.set_params(segment_size=32)
    assert est.segment_size == 32
    scan = ht.SegmentedScan(segment_size=128, algo="strided16n")
    assert clone(scan).get_params() == scan.get_params()
    x = O.exact_int_segments(rng, 4096, 256)
    fitted = ht.SegmentedReduce(segment_size=256).fit(x)
    assert fitted.variant_ == "warp256" and fitted.n_features_in_ == 4096
    with pytest.raises(BadConfigError):
        ht.SegmentedReduce().transform(np.ones(256, np.float16))
    with pytest.raises(BadConfigError):
        ht.SegmentedReduce(segment_size=16, algo="bogus").fit(x)
    with pytest.raises(BadConfigError):
        ht.SegmentedReduce(segment_size=0).fit(x)
    with pytest.raises(BadLengthError):
        ht.SegmentedReduce().fit(np.array(["a", "b"]))
    with pytest.raises(BadConfigError):
        fitted.transform(np.ones(128, np.float16))
