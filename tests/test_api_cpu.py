"""Host-side behaviour of the drop-in that needs no GPU (CPU suite).

* The C-ABI library loads and exports every symbol include/tc_collectives.h
  declares; its argument checks return the documented status codes before
  any device work.
* The Python boundary raises the reference's exceptions in the reference's
  order (reduce.py:379-446, scan.py:316-388, segmented.py:57-89,
  plan.py:46-77) -- all before touching the device.
* Without a GPU the product fails loudly: there is no CPU fallback.
"""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1811_09736_b200 as ht
from paper_1811_09736_b200 import _lib
from paper_1811_09736_b200.errors import BadConfigError, BadLengthError

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "tc_collectives.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tc_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 10
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for s in syms:
        assert hasattr(lib, s), f"missing export {s}"
    assert set(syms) == set(_lib.SIGNATURES), "ctypes binding out of sync with the header"


def test_abi_helpers():
    L = _lib.lib
    assert L.tc_abi_version() >> 16 == 1
    assert _lib.status_string(_lib.TC_BAD_LENGTH) == "bad length"
    assert _lib.status_string(_lib.TC_BAD_CONFIG) == "bad config"
    small = L.tc_workspace_bytes(_lib.TC_OP_REDUCE, 1 << 20, 256)
    big = L.tc_workspace_bytes(_lib.TC_OP_SCAN, 1 << 33, 1 << 33)
    assert 0 < small < big
    assert big < 64 << 20  # workspace stays small even at 2^33 elements


def test_c_abi_argument_errors_before_launch():
    L = _lib.lib
    ws = ctypes.create_string_buffer(1 << 16)
    wsp = (ctypes.addressof(ws) + 255) & ~255
    x = 1 << 20  # fake, aligned "device" pointers: checks must fire first
    out = 2 << 20
    assert L.tc_seg_reduce(x, 0, 16, out, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_LENGTH
    assert L.tc_seg_reduce(x, 100, 0, out, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_LENGTH
    assert L.tc_seg_reduce(x, 1 << 37, 16, out, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_LENGTH
    assert L.tc_seg_reduce(x + 2, 100, 16, out, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_ALIGNMENT
    assert L.tc_seg_reduce(None, 100, 16, out, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_CONFIG
    assert L.tc_seg_reduce(x, 100, 16, out, 9, wsp, 60000, None) == _lib.TC_BAD_CONFIG
    assert L.tc_seg_reduce(x, 100, 16, out, _lib.TC_F32, wsp, 10, None) == _lib.TC_WORKSPACE_TOO_SMALL
    # scans have no fp64 output
    assert L.tc_seg_scan(x, 100, 16, out, _lib.TC_F64, 0, None, None, wsp, 60000, None) == _lib.TC_BAD_CONFIG
    assert "segment size" in _lib.last_error() or "dtype" in _lib.last_error()
    # *_ex: unknown input dtype -> bad config, before any launch
    assert L.tc_seg_reduce_ex(x, 7, 100, 16, out, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_CONFIG
    assert "input dtype" in _lib.last_error()
    assert L.tc_seg_scan_ex(x, 7, 100, 16, out, _lib.TC_F32, 0, None, None, wsp, 60000,
                            None) == _lib.TC_BAD_CONFIG


def test_select_algorithm_matches_reference_table(golden):
    _, meta = golden
    for op, s, total, variant in meta["plan"]:
        assert ht.select_algorithm(op, s, total_len=total).variant == variant, (op, s, total)


def test_select_algorithm_env_override(monkeypatch):
    # pkg/tests/test_plan.py:43-51
    monkeypatch.setenv("TCU_THRESHOLD_BLOCK", "1024")
    assert ht.select_algorithm("reduce", 2048).variant == "block256n"
    assert ht.select_algorithm("reduce", 2048, block_thresh=4096).variant == "efficient256n"
    with pytest.raises(BadConfigError):
        ht.select_algorithm("sort", 16)
    with pytest.raises(BadConfigError):
        ht.select_algorithm("reduce", 0)


def test_block_config_and_engine():
    with pytest.raises(BadConfigError):
        ht.BlockConfig(wpb=0)
    with pytest.raises(BadConfigError):
        ht.BlockConfig(wpb=17)
    with pytest.raises(BadConfigError):
        ht.BlockConfig(coarsening=0)
    assert ht.clamp_block_config(ht.BlockConfig(wpb=4), 6).wpb == 3
    assert ht.TileEngine().acc_dtype == np.float16
    assert ht.TileEngine(accumulate="single").acc_dtype == np.float32
    with pytest.raises(ValueError):
        ht.TileEngine(accumulate="double")
    c = ht.CostCounters(mma_count=2)
    assert c.cycle_estimate == 64  # reference formula (engine.py:110-114)
    assert ht.coalesced_group_mma_count(272) == 16 * 2 + 1


def test_reduce_validation_matches_reference():
    e = ht.TileEngine()
    with pytest.raises(BadLengthError):
        ht.segmented_reduce(np.ones((4, 4), np.float16), 16, "warp16", e)
    with pytest.raises(BadConfigError):
        ht.segmented_reduce(np.ones(64, np.float16), 32, "warp16", e)  # test_reduce.py:246-250
    with pytest.raises(BadConfigError):
        ht.segmented_reduce(np.ones(64, np.float16), 32, "no_such", e)
    with pytest.raises(BadConfigError):
        ht.segmented_reduce(np.ones(64, np.float16), 64, "warp256", e)
    with pytest.raises(BadLengthError):
        ht.segmented_reduce(np.ones(0, np.float16), 16, "strided16n", e)
    with pytest.raises(BadLengthError):
        ht.segmented_reduce(np.ones(10, np.float16), 0, "strided16n", e)
    with pytest.raises(BadLengthError):
        ht.reduce_16(np.ones(255, np.float16), e)
    with pytest.raises(BadLengthError):
        ht.reduce_256(np.ones(512, np.float16), e)
    with pytest.raises(BadLengthError):
        ht.reduce_256n_efficient(np.ones(512, np.float16), 3, e)
    with pytest.raises(BadLengthError):
        ht.reduce_16n_strided(np.ones(512, np.float16), 24, e)
    with pytest.raises(BadLengthError):
        ht.reduce_16n_coalesced(np.ones(500, np.float16), 32, e)
    with pytest.raises(BadConfigError):
        ht.block_reduce_256n(np.ones(256 * 3, np.float16), ht.BlockConfig(wpb=2), e)
    with pytest.raises(BadLengthError):
        ht.block_reduce_256n(np.ones(300, np.float16), ht.BlockConfig(wpb=1), e)
    with pytest.raises(BadConfigError):
        ht.grid_reduce(np.ones(4096, np.float16), e, block_elems=1000)
    with pytest.raises(BadLengthError):
        ht.grid_reduce(np.ones(0, np.float16), e)


def test_scan_validation_matches_reference():
    e = ht.TileEngine()
    with pytest.raises(BadConfigError):
        ht.segmented_scan(np.ones(1024, np.float16), 256, "grid", e)  # test_scan.py:342-344
    with pytest.raises(BadConfigError):
        ht.segmented_scan(np.ones(64, np.float16), 32, "warp16", e)
    with pytest.raises(BadConfigError):
        ht.segmented_scan(np.ones(64, np.float16), 32, "bogus", e)
    with pytest.raises(BadLengthError):
        ht.segmented_scan(np.ones(100, np.float16), 64, "strided16n", e, inclusive=False)
    with pytest.raises(BadLengthError):
        ht.scan_16(np.ones(128, np.float16), e)
    with pytest.raises(BadLengthError):
        ht.scan_256n(np.ones(512, np.float16), 3, e)
    with pytest.raises(BadLengthError):
        ht.scan_16n(np.ones(500, np.float16), 32, e)
    with pytest.raises(BadConfigError):
        ht.block_scan_256n(np.ones(256 * 5, np.float16), ht.BlockConfig(wpb=4), e)
    with pytest.raises(BadLengthError):
        ht.last_column_scan_16(np.ones((8, 8)), e)


def test_no_cpu_fallback():
    """Valid arguments on a machine without a GPU must fail loudly."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible; covered by the gpu suite")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ht.segmented_reduce(np.ones(64, np.float16), 16, "warp16", ht.TileEngine())
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ht.segmented_scan(np.ones(64, np.float16), 16, "warp16", ht.TileEngine())


def test_pad_segmented_semantics():
    sv = ht.pad_segmented(np.arange(1, 8, dtype=np.float16), 3, seg_multiple=4, count_multiple=2)
    assert sv.seg_size == 4 and sv.n_segments == 4 and sv.n_logical_segments == 3
    assert sv.data.reshape(4, 4).tolist() == [[1, 2, 3, 0], [4, 5, 6, 0], [7, 0, 0, 0], [0, 0, 0, 0]]
    assert sv.unpad_scan(sv.data).tolist() == list(range(1, 8))
    with pytest.raises(BadLengthError):
        ht.pad_segmented(np.ones(0, np.float16), 4)


def test_oracle_is_not_imported_by_the_product():
    for p in (ROOT / "paper_1811_09736_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p


def test_irregular_validation_before_device():
    """Irregular (CSR-offset) entry points: offset errors raise before any
    device work; the C ABI rejects bad counts / pointers with status codes."""
    x = np.ones(100, np.float16)
    for bad in ([0, 50, 40, 100], [1, 100], [0, 99], [[0, 100]]):
        exc = BadLengthError if np.ndim(bad) != 1 else BadConfigError
        with pytest.raises(exc):
            ht.irregular_segmented_reduce(x, bad)
        with pytest.raises(exc):
            ht.irregular_segmented_scan(x, bad)
    with pytest.raises(BadLengthError):
        ht.irregular_segmented_reduce(x, [0])
    with pytest.raises(BadLengthError):
        ht.irregular_segmented_reduce(np.ones(0, np.float16), [0, 0])
    L = _lib.lib
    ws = ctypes.create_string_buffer(1 << 16)
    wsp = (ctypes.addressof(ws) + 255) & ~255
    xp, out, offp = 1 << 20, 2 << 20, 3 << 20
    assert L.tc_irreg_reduce(xp, 0, 100, offp, 0, out, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_LENGTH
    assert L.tc_irreg_reduce(xp, 0, 100, offp + 4, 3, out, _lib.TC_F32, wsp, 60000,
                             None) == _lib.TC_BAD_ALIGNMENT
    assert L.tc_irreg_reduce(xp, 0, 100, None, 3, out, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_ALIGNMENT
    assert L.tc_irreg_reduce(xp, 7, 100, offp, 3, out, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_CONFIG
    assert L.tc_irreg_scan(xp, 0, 100, offp, 3, out, _lib.TC_F64, 0, wsp, 60000, None) == _lib.TC_BAD_CONFIG
    assert L.tc_irreg_scan(xp, 0, 0, offp, 3, out, _lib.TC_F32, 0, wsp, 60000, None) == _lib.TC_BAD_LENGTH


def test_irregular_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible; covered by the gpu suite")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ht.irregular_segmented_reduce(np.ones(64, np.float16), [0, 10, 64])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        ht.irregular_segmented_scan(np.ones(64, np.float16), [0, 10, 64])


def test_batchnorm_validation_before_device():
    with pytest.raises(BadLengthError):
        ht.batch_norm_stats(np.ones(10, np.float16))
    with pytest.raises(BadLengthError):
        ht.batch_norm_stats(np.ones((0, 3), np.float16))
    L = _lib.lib
    ws = ctypes.create_string_buffer(1 << 16)
    wsp = (ctypes.addressof(ws) + 255) & ~255
    xp, m, v = 1 << 20, 2 << 20, 3 << 20
    assert L.tc_bn_stats(xp, 0, 0, 3, 4, m, v, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_LENGTH
    assert L.tc_bn_stats(xp, 0, 2, 3, 4, m, v, _lib.TC_F16, wsp, 60000, None) == _lib.TC_BAD_CONFIG
    assert L.tc_bn_stats(xp, 0, 2, 3, 4, None, v, _lib.TC_F32, wsp, 60000, None) == _lib.TC_BAD_CONFIG
    assert L.tc_bn_stats(xp, 0, 2, 3, 4, m, v, _lib.TC_F32, wsp, 10, None) == _lib.TC_WORKSPACE_TOO_SMALL
    need = L.tc_workspace_bytes(_lib.TC_OP_BN_STATS, 2 * 3 * 4, 4)
    assert need >= L.tc_workspace_bytes(_lib.TC_OP_REDUCE, 2 * 3 * 4, 4)


def test_batch_norm_forward_needs_cuda_tensor():
    with pytest.raises(TypeError):
        ht.batch_norm(np.ones((2, 3, 4), np.float16))


def test_plan_info_modes():
    """tc_plan_info mirrors the dispatch (host only): which kernel runs."""
    import torch

    from paper_1811_09736_b200 import _device as D

    n = 1 << 30
    assert D.plan_info("reduce", n, 16) == ("LOCAL", 64)
    assert D.plan_info("reduce", n, 256) == ("ROWS", 64)
    assert D.plan_info("reduce", n, 65536) == ("TILES", 64)
    assert D.plan_info("reduce", n, 48) == ("GENERAL", 64)
    mode, L = D.plan_info("reduce", n, 3)
    assert mode == "ROWSEG" and L % 3 == 0 and (2 * L) % 16 == 0
    mode, L = D.plan_info("reduce", n, 3, torch.float32)
    assert mode == "ROWSEG" and (L // 3) * 4 <= 64
    assert D.plan_info("reduce", n, 100001)[0] == "SPLIT"
    assert D.plan_info("reduce", n, 1000)[0] == "GENERAL"  # gcd 8: whole granules
    assert D.plan_info("reduce", n, 4097)[0] == "GENERAL"  # SPLIT only from 1.5 tiles per segment
    assert D.plan_info("reduce", n, 8193)[0] == "GENERAL"
    assert D.plan_info("reduce", n, 12289)[0] == "SPLIT"
    # ROWSEG scan rows (fp16 out): up to 16 chunks, whole 32-B sectors among equal-cost layouts
    assert D.plan_info("scan", n, 63) == ("ROWSEG", 1008)
    assert D.plan_info("scan", n, 23) == ("ROWSEG", 368)
    assert D.plan_info("scan", n, 49) == ("ROWSEG", 784)
    assert D.plan_info("scan", n, n)[0] == "CHUNK"
    assert D.plan_info("scan", n, 4096, carry_in=True)[0] == "CHUNK"
    assert D.plan_info("scan", n, 17)[0] == "ROWSEG"
    assert D.plan_info("scan", n, 17, torch.float32)[0] == "SPLITM"
    assert D.plan_info("scan", n, 63, torch.float32)[0] == "SPLITM"
    assert D.plan_info("scan", n, 34, torch.float32)[0] == "GENERAL"
    assert D.plan_info("scan", n, 9, torch.float32)[0] == "ROWSEG"
    assert D.plan_info("scan", n, 3, torch.float32)[0] == "ROWSEG"
    assert D.plan_info("scan", n, 17, total_out=True)[0] == "GENERAL"
    assert D.plan_info("scan", n, 12)[0] == "GENERAL"
    for s in (65, 66, 100, 300, 4097, 100001, 1000003):
        assert D.plan_info("scan", n, s)[0] == "SPLIT", s
    assert D.plan_info("scan", n, 300, total_out=True)[0] == "GENERAL"
    assert D.plan_info("scan", n, 1000)[0] == "GENERAL"
    assert D.plan_info("scan", n, (1 << 21) + 1)[0] == "CHUNK"
