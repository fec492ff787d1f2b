"""GPU parity: the sm_100a kernels (through the C ABI and the drop-in API)
against the oracle (tests/test_oracle.py pins the oracle to the reference).

Tolerances (stated here):
* exact-integer inputs (every partial sum representable): BIT-EXACT against
  fp16(exact) / fp32(exact) -- which on these inputs is also exactly what
  the reference simulator returns in half / single mode;
* non-integer inputs, fp16 output: |got - exact| <= 1 fp16 ulp of the exact
  value (the kernel accumulates in fp32/fp64 and rounds once; the only
  deviation from fp16(exact) is a double rounding near a midpoint);
* non-integer inputs, fp32 output: |got - exact| <= 1e-5 * |exact| + 2^-24
  (exact >= 0 for the uniform [0, 1) test data, so the running sum is the
  error scale for scans too).  The north-star ceiling is 1e-3.
* segment counts, output positions and boundaries: identical.
"""

import numpy as np
import pytest
import torch

import paper_1811_09736_b200 as ht
from paper_1811_09736_b200 import _device as D
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def ulp16(v):
    a = np.abs(np.asarray(v, np.float64)).astype(np.float16)
    return np.spacing(a).astype(np.float64)


def assert_bits(got, exp64, dtype):
    got = np.asarray(got)
    exp = np.asarray(exp64, np.float64).astype(dtype)
    assert got.dtype == exp.dtype, (got.dtype, exp.dtype)
    assert got.shape == exp.shape, (got.shape, exp.shape)
    bad = np.nonzero(got.view(np.uint16 if dtype == np.float16 else np.uint32) !=
                     exp.view(np.uint16 if dtype == np.float16 else np.uint32))[0]
    assert bad.size == 0, f"{bad.size} mismatches, first {bad[:5]}: {got[bad[:3]]} vs {exp[bad[:3]]}"


def assert_close(got, exact, dtype):
    got = np.asarray(got, np.float64)
    exact = np.asarray(exact, np.float64)
    assert got.shape == exact.shape
    if dtype == np.float16:
        err = np.abs(got - exact)
        assert np.all(err <= ulp16(exact)), float((err / ulp16(exact)).max())
    else:
        assert np.all(np.abs(got - exact) <= 1e-5 * np.abs(exact) + 2.0 ** -24)


# ----------------------------------------------------------- golden fixtures


def test_golden_cases_through_dropin_api(golden, cuda):
    z, meta = golden
    for case in meta["manifest"]:
        k, op, seg, variant = case["id"], case["op"], case["seg"], case["variant"]
        x = z[f"x{k}"].view(np.float16)
        exact = z[f"exact{k}"]
        for acc, dt in (("half", np.float16), ("single", np.float32)):
            eng = ht.TileEngine(accumulate=acc)
            if op == "reduce":
                got = ht.segmented_reduce(x, x.size if variant == "grid" else seg, variant, eng)
            else:
                got = ht.segmented_scan(x, x.size if variant == "grid" else seg, variant, eng,
                                        inclusive=case["inclusive"])
            assert isinstance(got, np.ndarray) and got.dtype == dt
            if "int" in case["kind"]:
                assert_bits(got, exact, dt)
                # ... which is also the reference simulator's own answer
                assert np.array_equal(got.astype(np.float64), z[f"sim_{acc}{k}"]), case
            else:
                assert_close(got, exact, dt)
                if acc == "half":  # never less accurate than the reference simulator
                    e_ours = np.abs(got.astype(np.float64) - exact).max()
                    e_ref = np.abs(z[f"sim_half{k}"] - exact).max()
                    assert e_ours <= e_ref + 1e-12, (case, e_ours, e_ref)


def test_known_answers_through_primitives(golden, cuda):
    z, meta = golden
    kat = {n: (z[f"kat_x_{n}"].view(np.float16), z[f"kat_y_{n}"]) for n in meta["kats"]}
    e = ht.TileEngine
    x, y = kat["reduce_16_arange"]
    assert np.array_equal(ht.reduce_16(x, e()).astype(np.float64), y)
    for name in ("reduce_256_zeros", "reduce_256_ones", "reduce_256_halves"):
        x, y = kat[name]
        assert float(ht.reduce_256(x, e())) == y[0]
    x, y = kat["efficient_1024_ones"]
    assert float(ht.reduce_256n_efficient(x, 4, e())) == y[0]
    assert float(ht.reduce_256n_inefficient(x, 4, e())) == y[0]
    x, y = kat["strided_512_ones_seg32"]
    assert ht.reduce_16n_strided(x, 32, e()).tolist() == y.tolist()
    x, y = kat["coalesced_seg512_ones"]
    assert ht.reduce_16n_coalesced(x, 512, e()).tolist() == y.tolist()
    x, y = kat["block_wpb4_4096_ones"]
    cap = {}
    assert float(ht.block_reduce_256n(x, ht.BlockConfig(wpb=4), e(), debug_capture=cap)) == y[0]
    assert cap["partials"].tolist() == [1024.0] * 4
    for name in ("grid_1024_ones", "grid_100_ones"):
        x, y = kat[name]
        assert float(ht.grid_reduce(x, e())) == y[0]
    x, y = kat["scan_16_ones"]
    assert np.array_equal(ht.scan_16(x, e()).astype(np.float64), y)
    x, y = kat["scan_256_ones"]
    assert np.array_equal(ht.scan_256(x, e()).astype(np.float64), y)
    x, y = kat["scan_16n_512_ones_seg32"]
    assert np.array_equal(ht.scan_16n(x, 32, e()).astype(np.float64), y)
    x, y = kat["scan_256n_512_ones"]
    assert np.array_equal(ht.scan_256n(x, 2, e()).astype(np.float64), y)
    x, y = kat["block_scan_wpb4_4096_ones"]
    assert np.array_equal(ht.block_scan_256n(x, ht.BlockConfig(wpb=4), e()).astype(np.float64), y)
    x, y = kat["grid_scan_4096_ones_blk1024"]
    assert np.array_equal(ht.grid_scan(x, e(), block_elems=1024).astype(np.float64), y)
    for name in ("ones", "seq", "ones_carry5"):
        tile = z[f"lcs_tile_{name}"].view(np.float16).reshape(16, 16)
        got = ht.last_column_scan_16(tile, e(), carry=float(z[f"lcs_carry_{name}"][0]))
        assert np.array_equal(got.astype(np.float64), z[f"lcs_y_{name}"]), name


# ------------------------------------------------------ C-ABI matrix (exact)

NS = [1, 2, 63, 64, 65, 100, 1000, 8191, 8192, 8193, 65536, 12345, 8192 * 3 + 70,
      (1 << 20), (1 << 22) + 1234]
SEGS = [1, 2, 3, 7, 16, 32, 48, 64, 100, 128, 256, 300, 1024, 4096, 8192, 16384, 24576,
        65536, 100000, 1 << 17, (1 << 18) + 8192, 1 << 20]


@pytest.mark.parametrize("n", NS)
def test_c_abi_matrix_bit_exact(n, cuda, rng):
    x = rng.integers(0, 8, n).astype(np.float16)
    xd = torch.from_numpy(x).to(cuda)
    for s in SEGS + [n, n + 5]:
        sums = O.ref_seg_reduce(x, s)
        for dt, npdt in ((torch.float16, np.float16), (torch.float32, np.float32),
                         (torch.float64, np.float64)):
            got = D.seg_reduce(xd, s, dt).cpu().numpy()
            assert np.array_equal(got, sums.astype(npdt)), (n, s, dt)
        for exc in (False, True):
            ref = O.ref_seg_scan(x, s, inclusive=not exc)
            for dt, npdt in ((torch.float16, np.float16), (torch.float32, np.float32)):
                got = D.seg_scan(xd, s, dt, exclusive=exc).cpu().numpy()
                assert np.array_equal(got, ref.astype(npdt)), (n, s, dt, exc)


@pytest.mark.parametrize("n", [1000, 8192 * 5 + 3, 1 << 20, (1 << 22) + 77])
def test_scan_carry_in_total_out(n, cuda, rng):
    x = rng.integers(0, 8, n).astype(np.float16)
    xd = torch.from_numpy(x).to(cuda)
    cin = torch.tensor([37.0], dtype=torch.float64, device=cuda)
    tot = torch.zeros(1, dtype=torch.float64, device=cuda)
    for exc in (False, True):
        got = D.seg_scan(xd, n, torch.float32, exclusive=exc, carry_in=cin, total_out=tot)
        exp = O.ref_seg_scan(x, n, inclusive=not exc, carry=37.0)
        assert np.array_equal(got.cpu().numpy(), exp.astype(np.float32))
        assert tot.item() == 37.0 + x.astype(np.float64).sum()
    tot.zero_()
    D.seg_scan(xd, 1000, torch.float32, total_out=tot)
    last = O.ref_seg_scan(x, 1000)[-1]
    assert tot.item() == last


@pytest.mark.parametrize("k", ["1", "2", "3", "4"])
def test_chunked_scan_modes(k, cuda, monkeypatch):
    """MODE_CHUNK (full scans, segments > 2^18, carry-in): P1/P2 chunk
    walk at several unit sizes (TC_CHUNK_TILES), ragged lengths, long
    non-power-of-two segments, inclusive/exclusive, with and without a
    carry -- bit-exact on sparse-ones data (every prefix an exact integer)."""
    monkeypatch.setenv("TC_CHUNK_TILES", k)
    rs = np.random.default_rng(int(k))
    for n in ((1 << 22) + 1234, 3 << 20, 8192 * 300 + 5):
        x = (rs.random(n) < 1 / 16).astype(np.float16)
        xd = torch.from_numpy(x).to(cuda)
        for s in (n, 300001, (1 << 18) + 8192, 1 << 20):
            for exc in (False, True):
                exp = O.ref_seg_scan(x, s, inclusive=not exc)
                got = D.seg_scan(xd, s, torch.float32, exclusive=exc).cpu().numpy()
                assert np.array_equal(got, exp.astype(np.float32)), (n, s, exc)
        cin = torch.tensor([5.0], dtype=torch.float64, device=cuda)
        tot = torch.zeros(1, dtype=torch.float64, device=cuda)
        for s in (n, 4096):
            got = D.seg_scan(xd, s, torch.float32, exclusive=True, carry_in=cin, total_out=tot)
            exp = O.ref_seg_scan(x, s, inclusive=False, carry=5.0)
            assert np.array_equal(got.cpu().numpy(), exp.astype(np.float32)), (n, s)
            assert tot.item() == O.ref_seg_scan(x, s, carry=5.0)[-1]
        # deterministic across reruns (fixed composition order)
        g = torch.rand(n, device=cuda).to(torch.float16)
        a = D.full_scan(g, torch.float32)
        b = D.full_scan(g, torch.float32)
        assert torch.equal(a, b)


@pytest.mark.parametrize("n", [1000, (1 << 20) + 77, (1 << 22) + 1234])
def test_bf16_input(n, cuda, rng):
    """bf16 input (tcgen05 kind::f16 with BF16 operands; extension beyond the
    fp16-only reference): bit-exact on small integers (exact in bf16 and in
    every partial sum), and within the fp32 tolerance on uniform data, across
    the LOCAL / ROWS / TILES / GENERAL / SPLIT / SPLITM / ROWSEG / CHUNK modes
    (SPLIT / SPLITM convert the raw bf16 elements of split granules too)."""
    xi = rng.integers(0, 8, n).astype(np.float32)
    xd = torch.from_numpy(xi).to(cuda).to(torch.bfloat16)
    x64 = xd.double().cpu().numpy()
    # modes: LOCAL 16, GENERAL 48, ROWS 256, TILES 8192, SPLIT 300 / 100001,
    # SPLITM 33 (fp32 out), ROWSEG 3 / 17, CHUNK 2^19 and n
    for s in (16, 48, 256, 8192, 300, 100001, 33, 17, 3, 1 << 19, n):
        got = D.seg_reduce(xd, s, torch.float32).cpu().numpy()
        assert np.array_equal(got, O.ref_seg_reduce(x64, s).astype(np.float32)), (n, s)
        for exc in (False, True):
            got = D.seg_scan(xd, s, torch.float32, exclusive=exc).cpu().numpy()
            exp = O.ref_seg_scan(x64, s, inclusive=not exc).astype(np.float32)
            assert np.array_equal(got, exp), (n, s, exc)
    xu = torch.rand(n, device=cuda).to(torch.bfloat16)
    u64 = xu.double().cpu().numpy()
    for s in (64, 1000, n):
        assert_close(D.seg_reduce(xu, s, torch.float32).cpu().numpy(), O.ref_seg_reduce(u64, s),
                     np.float32)
        assert_close(D.seg_scan(xu, s, torch.float32).cpu().numpy(), O.ref_seg_scan(u64, s),
                     np.float32)


# ------------------------------------------------ non-integer data tolerance


@pytest.mark.parametrize("s", [16, 64, 256, 300, 4096, 65536])
def test_uniform_tolerance(s, cuda, rng):
    n = (1 << 20) + 333
    x = rng.random(n, dtype=np.float32).astype(np.float16)
    xd = torch.from_numpy(x).to(cuda)
    sums = O.ref_seg_reduce(x, s)
    scans = O.ref_seg_scan(x, s)
    for dt, npdt in ((torch.float16, np.float16), (torch.float32, np.float32)):
        assert_close(D.seg_reduce(xd, s, dt).cpu().numpy(), sums, npdt)
        assert_close(D.seg_scan(xd, s, dt).cpu().numpy(), scans, npdt)
    # the reference's own check (cli.py:41-42, test_acceptance.py:230-243)
    got = D.seg_scan(xd, s, torch.float16).cpu().numpy().astype(np.float64)
    assert np.all(np.abs(got - scans) <= 2.0 ** -24 + 2.0 ** -8 * np.abs(scans))


# --------------------------------------------------- full-size configurations


def test_config1_exact(cuda):
    """BASELINE config 1: 2^20 elements, segment 256, exact_int_segments
    with the reference seed -- bit-exact through the drop-in API."""
    x = O.exact_int_segments(np.random.default_rng(20260810), 1 << 20, 256)
    got = ht.segmented_reduce(x, 256, "warp256", ht.TileEngine())
    assert_bits(got, O.ref_seg_reduce(x, 256), np.float16)
    assert np.array_equal(got.astype(np.float64), O.sim_segmented_reduce(x, 256, "warp256"))


def _big_uniform(n, cuda, seed=0):
    g = torch.Generator(device=cuda)
    g.manual_seed(seed)
    return torch.rand(n, device=cuda, generator=g, dtype=torch.float32).to(torch.float16)


@pytest.mark.parametrize("s", [16, 32, 256, 4096, 65536])
def test_config2_reduce_2p30(s, cuda):
    """BASELINE config 2 at full size (2^30): every sum within tolerance of
    the exact oracle (computed on the host copy)."""
    n = 1 << 30
    xd = _big_uniform(n, cuda, seed=s)
    x = xd.cpu().numpy()
    sums = O.ref_seg_reduce(x, s)
    assert_close(D.seg_reduce(xd, s, torch.float32).cpu().numpy(), sums, np.float32)
    assert_close(D.seg_reduce(xd, s, torch.float16).cpu().numpy(), sums, np.float16)


@pytest.mark.parametrize("s", [16, 1024, 16384])
def test_config3_scan_2p30_properties(s, cuda):
    """BASELINE config 3 at full size: size-independent properties --
    scan tail of every segment == segment reduce (acceptance c5), exactness
    against the oracle on 64 sampled segments, and exclusive == shifted
    inclusive everywhere."""
    n = 1 << 30
    xd = _big_uniform(n, cuda, seed=s + 1)
    inc = D.seg_scan(xd, s, torch.float32)
    exc = D.seg_scan(xd, s, torch.float32, exclusive=True)
    red = D.seg_reduce(xd, s, torch.float32)
    tails = inc.view(-1, s)[:, -1]
    assert torch.allclose(tails.double(), red.double(), rtol=2e-6, atol=0)
    # exclusive == shifted inclusive: bit-exact on exact-integer data (matrix
    # test above); on float data the two are rounded through different
    # (equally accurate) associations at row boundaries
    assert torch.allclose(exc.view(-1, s)[:, 1:].double(), inc.view(-1, s)[:, :-1].double(),
                          rtol=2e-6, atol=0)
    assert torch.all(exc.view(-1, s)[:, 0] == 0)
    rs = np.random.default_rng(s)
    segs = rs.integers(0, n // s, 64)
    inc_h = inc.view(-1, s)[torch.from_numpy(segs).to(cuda)].cpu().numpy()
    for i, k in enumerate(segs):
        xs = xd[k * s:(k + 1) * s].cpu().numpy()
        assert_close(inc_h[i], O.ref_seg_scan(xs, s), np.float32)
    del inc, exc


def test_config4_5_full_ops_2p32_exact(cuda):
    """Full reduce / full exclusive scan of 2^32 + 7 sparse-ones fp16
    elements (Bernoulli 2^-10, SURVEY 8(d) parity data: every prefix is an
    exact integer < 2^24 so fp32 outputs are exact)."""
    n = (1 << 32) + 7
    g = torch.Generator(device=cuda)
    g.manual_seed(4)
    xd = (torch.rand(n, device=cuda, generator=g) < 2.0 ** -10).to(torch.float16)
    # exact oracle on a host copy, by blocks (restates oracle.py:47-75)
    x = xd.cpu().numpy()
    total = O.ref_seg_reduce(x, n)[0]
    got = D.full_reduce(xd, torch.float64).item()
    assert got == total
    assert D.full_reduce(xd, torch.float32).item() == np.float32(total)
    exc = D.full_scan(xd, torch.float32, exclusive=True)
    # sampled positions: exact prefix = sum of everything before
    blocks = 1 << 20
    bsum = O.ref_seg_reduce(x, blocks)
    bpre = np.concatenate([[0.0], np.cumsum(bsum)])
    rs = np.random.default_rng(9)
    pos = np.concatenate([[0, 1, n - 1], rs.integers(0, n, 200)])
    got_p = exc[torch.from_numpy(pos).to(cuda)].cpu().numpy()
    for p, gp in zip(pos, got_p):
        b = p // blocks
        exp = bpre[b] + x[b * blocks:p].astype(np.float64).sum()
        assert gp == exp, (p, gp, exp)
    del exc


# ----------------------------------------------------------------- edge cases


def test_edge_semantics(cuda):
    e = ht.TileEngine()
    # signed zero canonicalised to +0 like the simulator
    z = np.full(64, -0.0, np.float16)
    out = ht.segmented_scan(z, 16, "warp16", e)
    assert np.all(out.view(np.uint16) == 0)
    out = ht.segmented_reduce(z, 16, "warp16", e)
    assert np.all(out.view(np.uint16) == 0)
    # fp16 overflow -> inf in half mode, exact in single mode (engine.py:347-348)
    big = np.full(4096, 60000.0, np.float16)
    assert np.isinf(ht.grid_reduce(big, ht.TileEngine()))
    assert float(ht.grid_reduce(big, ht.TileEngine(accumulate="single"))) == 4096 * 60000.0
    # misaligned torch views are handled (copied), results unchanged
    xd = torch.arange(1, 1002, device=cuda, dtype=torch.float16)
    a = D.seg_reduce(xd[1:], 10, torch.float32).cpu().numpy()
    assert np.array_equal(a, O.ref_seg_reduce(np.arange(2, 1002, dtype=np.float16), 10).astype(np.float32))
    # output counts: ceil(n / s) sums, n prefix sums
    for n, s in ((1, 5), (17, 16), (8193, 8192), (100, 100), (100, 1)):
        x = np.ones(n, np.float16)
        assert ht.segmented_reduce(x, s, "strided16n", e).size == -(-n // s)
        assert ht.segmented_scan(x, s, "strided16n", e).size == n


def test_torch_inputs_stay_in_their_domain(cuda):
    e = ht.TileEngine(accumulate="single")
    x = torch.ones(4096, dtype=torch.float16)
    y = ht.segmented_reduce(x.to(cuda), 256, "warp256", e)
    assert y.is_cuda and y.dtype == torch.float32 and y.tolist() == [256.0] * 16
    xp = x.pin_memory()
    y = ht.segmented_scan(xp, 4096, "grid", e)
    assert not y.is_cuda and y[-1].item() == 4096.0
    assert e.counters.mma_count > 0 and e.counters.tile_loads > 0


def test_determinism(cuda):
    g = torch.Generator(device=cuda)
    g.manual_seed(1)
    xd = torch.rand((1 << 22) + 5, device=cuda, generator=g).to(torch.float16)
    for s in (300, 65536, xd.numel()):
        a = D.seg_reduce(xd, s, torch.float32)
        b = D.seg_reduce(xd, s, torch.float32)
        assert torch.equal(a, b)
    for s in (300, 16384, 100000):
        a = D.seg_scan(xd, s, torch.float32)
        b = D.seg_scan(xd, s, torch.float32)
        assert torch.equal(a, b)


def test_nccl_single_rank_sharded_ops(cuda):
    """The multi-GPU wrappers on the product path (DeviceOps + NCCL) with a
    one-rank group on this GPU; the 2-rank exchange logic is covered by
    tests/test_distributed_cpu.py."""
    import os

    import torch.distributed as dist

    from paper_1811_09736_b200 import distributed as Dist

    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        x = O.exact_int_segments(np.random.default_rng(3), 1 << 20, 1 << 20)
        xd = torch.from_numpy(x).to(cuda)
        tot = Dist.sharded_full_reduce(xd, torch.float64)
        assert tot.item() == x.astype(np.float64).sum()
        sc = Dist.sharded_full_scan(xd, torch.float32, exclusive=True)
        assert np.array_equal(sc.cpu().numpy(), O.ref_seg_scan(x, x.size, inclusive=False).astype(np.float32))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("s", [17, 49, 63, 300, 1001, 100001])
def test_general_and_odd_segments_2p28(s, cuda):
    """Large-n parity of the GENERAL-mode paths (cumulative-B one/two-end
    selects, MODE_GSCR's SMEM-staged ends, the granule walk) against the
    exact oracle, exact-integer data: fp32 bit-exact, fp16 = fp16(exact)."""
    rng = np.random.default_rng(s)
    n = (1 << 28) + 5
    x = rng.integers(0, 8, n).astype(np.float16)
    xd = torch.from_numpy(x).to(cuda)
    exp = O.ref_seg_reduce(x, s)
    got32 = D.seg_reduce(xd, s, torch.float32).cpu().numpy()
    assert np.array_equal(got32, exp.astype(np.float32))
    got16 = D.seg_reduce(xd, s, torch.float16).cpu().numpy()
    assert np.array_equal(got16, exp.astype(np.float16))
