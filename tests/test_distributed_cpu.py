"""Multi-process (gloo, world_size 2, CPU) tests of the sharding / exchange
logic in paper_1811_09736_b200.distributed.  The per-shard compute is a
plain float64 stand-in defined here (the exchange logic is what is under
test); results are checked against the oracle on the unsharded input."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_09736_b200 import distributed as D


class CpuOps:
    """Shard-local stand-in with the DeviceOps interface (float64 on CPU)."""

    @staticmethod
    def full_reduce_f64(x):
        return x.double().sum().reshape(1)

    @staticmethod
    def seg_reduce(x, seg, out_dtype):
        n = x.numel()
        k = -(-n // seg)
        pad = torch.zeros(k * seg, dtype=torch.float64)
        pad[:n] = x.double()
        return pad.view(k, seg).sum(1).to(out_dtype)

    @staticmethod
    def seg_scan(x, seg, out_dtype, exclusive, carry_in):
        xs = x.double().clone()
        c = torch.cumsum(xs, 0)
        if carry_in is not None:
            c = c + carry_in.double()
        if exclusive:
            c = torch.cat([carry_in.double() if carry_in is not None else torch.zeros(1, dtype=torch.float64), c[:-1]])
        return c.to(out_dtype)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        x = rng.integers(0, 8, n).astype(np.float16)
        lo, hi = D.even_bounds(n, world, rank)
        xl = torch.from_numpy(x[lo:hi].copy())
        tot = D.sharded_full_reduce(xl, torch.float64, ops=CpuOps)
        inc = D.sharded_full_scan(xl, torch.float64, exclusive=False, ops=CpuOps)
        exc = D.sharded_full_scan(xl, torch.float64, exclusive=True, ops=CpuOps)
        slo, shi = D.shard_bounds(n, 100, world, rank)
        sr = D.sharded_segmented_reduce(torch.from_numpy(x[slo:shi].copy()), 100, torch.float64,
                                        ops=CpuOps)
        q.put((rank, float(tot.item()), inc.numpy(), exc.numpy(), (lo, hi), (slo, shi), sr.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [10_001, 4096])
def test_two_rank_full_ops_and_shards(n):
    from oracle import oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    x = rng.integers(0, 8, n).astype(np.float16)
    total = x.astype(np.float64).sum()
    inc = O.ref_seg_scan(x, n)
    exc = O.ref_seg_scan(x, n, inclusive=False)
    sums = O.ref_seg_reduce(x, 100)
    got_inc = np.concatenate([r[2] for r in res])
    got_exc = np.concatenate([r[3] for r in res])
    assert all(r[1] == total for r in res)  # every rank gets the same total
    assert np.array_equal(got_inc, inc)
    assert np.array_equal(got_exc, exc)
    got_sums = np.concatenate([r[6] for r in res])
    assert np.array_equal(got_sums, sums)  # whole-segment shards need no exchange
    assert res[0][5][1] % 100 == 0


def test_shard_bounds_cover_whole_segments():
    for n, seg, world in [(1 << 20, 256, 8), (1000, 300, 3), (5, 10, 4), (1 << 30, 65536, 8)]:
        spans = [D.shard_bounds(n, seg, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c and b % seg == 0


def test_virtual_shards_match_the_process_group_path():
    """The single-process virtual-shards mode runs the same
    exchange arithmetic as a W-rank group: compare it with the 2-rank gloo
    run above and with the oracle, for W = 1..8 (CPU stand-in ops)."""
    from oracle import oracle as O

    rng = np.random.default_rng(5)
    for n in (10_001, 4096, 77):
        x = rng.integers(-8, 8, n).astype(np.float16)
        xt = torch.from_numpy(x)
        for w in (1, 2, 3, 8):
            assert D.virtual_full_reduce(xt, w, torch.float64, ops=CpuOps).item() == x.astype(np.float64).sum()
            for exc in (False, True):
                got = D.virtual_full_scan(xt, w, torch.float64, exclusive=exc, ops=CpuOps).numpy()
                assert np.array_equal(got, O.ref_seg_scan(x, n, inclusive=not exc))
            got = D.virtual_segmented_reduce(xt, 100, w, torch.float64, ops=CpuOps).numpy()
            assert np.array_equal(got, O.ref_seg_reduce(x, 100))


def test_even_bounds_aligned():
    for n, w in [(1 << 33, 8), (10_001, 3), (77, 8), (5, 4)]:
        b = [D.even_bounds(n, w, r) for r in range(w)]
        assert b[0][0] == 0 and b[-1][1] == n
        for (a, c), (d, e) in zip(b, b[1:]):
            assert c == d and c % 8 == 0 and a <= c
