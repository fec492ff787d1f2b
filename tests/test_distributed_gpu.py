"""Multi-process runs of the sharded collectives with the REAL per-shard
kernels (DeviceOps -> tc_* on the GPU), several ranks sharing this one GPU.

The product backend is NCCL (one process per GPU); NCCL refuses two ranks on
one device, so these ranks exchange through gloo -- the exchange logic and
the arithmetic (fp64 partials, rank-order combine, carry-seeded CHUNK scan
through ``carry_in``) are the product's.  Checked against the oracle on the
unsharded input, and bit-for-bit against the single-process virtual-shards
mode and, for exact-integer data, the 1-GPU ops."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1811_09736_b200 import distributed as Dist

pytestmark = pytest.mark.gpu

N = (1 << 22) + 40
SEG = 300


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(kind):
    rng = np.random.default_rng(17)
    if kind == "int":
        return rng.integers(-8, 8, N).astype(np.float16)
    return (rng.random(N) * 2 - 1).astype(np.float16)


def _worker(rank, world, port, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = _data(kind)
        lo, hi = Dist.even_bounds(N, world, rank)
        xl = torch.from_numpy(x[lo:hi].copy()).cuda()
        tot = Dist.sharded_full_reduce(xl, torch.float64)
        inc = Dist.sharded_full_scan(xl, torch.float32, exclusive=False)
        exc = Dist.sharded_full_scan(xl, torch.float32, exclusive=True)
        slo, shi = Dist.shard_bounds(N, SEG, world, rank)
        xs = torch.from_numpy(x[slo:shi].copy()).cuda()
        sr = Dist.sharded_segmented_reduce(xs, SEG, torch.float32)
        ss = Dist.sharded_segmented_scan(xs, SEG, torch.float32)
        torch.cuda.synchronize()
        q.put((rank, tot.item(), inc.cpu().numpy(), exc.cpu().numpy(), sr.cpu().numpy(),
               ss.cpu().numpy()))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e), None, None, None, None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("kind", ["int", "uniform_pm1"])
def test_multiprocess_sharded_ops_real_kernels(world, kind, cuda):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert r[2] is not None, f"rank {r[0]} failed: {r[1]}"
    assert all(p.exitcode == 0 for p in procs)
    x = _data(kind)
    xd = torch.from_numpy(x).to(cuda)
    inc = np.concatenate([r[2] for r in res])
    exc = np.concatenate([r[3] for r in res])
    sr = np.concatenate([r[4] for r in res])
    ss = np.concatenate([r[5] for r in res])
    # every rank holds the same total, equal to the virtual-shards combine
    vt = Dist.virtual_full_reduce(xd, world, torch.float64).item()
    assert all(r[1] == vt for r in res)
    # bit-identical to the single-process virtual G shards mode
    assert np.array_equal(inc, Dist.virtual_full_scan(xd, world, torch.float32).cpu().numpy())
    assert np.array_equal(exc, Dist.virtual_full_scan(xd, world, torch.float32, True).cpu().numpy())
    assert np.array_equal(sr, Dist.virtual_segmented_reduce(xd, SEG, world, torch.float32).cpu().numpy())
    assert np.array_equal(ss, Dist.virtual_segmented_scan(xd, SEG, world, torch.float32).cpu().numpy())
    e_inc = O.ref_seg_scan(x, N)
    e_exc = O.ref_seg_scan(x, N, inclusive=False)
    e_sr = O.ref_seg_reduce(x, SEG)
    e_ss = O.ref_seg_scan(x, SEG)
    if kind == "int":
        # exact data: the sharded results equal the oracle (and the 1-GPU ops)
        assert vt == x.astype(np.float64).sum()
        assert np.array_equal(inc, e_inc.astype(np.float32))
        assert np.array_equal(exc, e_exc.astype(np.float32))
        assert np.array_equal(sr, e_sr.astype(np.float32))
        assert np.array_equal(ss, e_ss.astype(np.float32))
    else:
        gamma = 16 * 2.0 ** -24
        ax = np.abs(x)
        m_inc = O.ref_seg_scan(ax, N)
        m_exc = O.ref_seg_scan(ax, N, inclusive=False)
        for got, e, m in ((inc, e_inc, m_inc), (exc, e_exc, m_exc),
                          (sr, e_sr, O.ref_seg_reduce(ax, SEG)), (ss, e_ss, O.ref_seg_scan(ax, SEG))):
            ulp = np.spacing(np.abs(e).astype(np.float32)).astype(np.float64)
            assert np.all(np.abs(got.astype(np.float64) - e) <= ulp + gamma * m)
        assert abs(vt - x.astype(np.float64).sum()) <= gamma * float(ax.astype(np.float64).sum())


@pytest.mark.parametrize("shards", [1, 2, 8])
def test_virtual_shards_match_single_gpu_2p31(shards, cuda):
    """Virtual G shards of 2^31 elements (the C5 per-GPU shard size at G = 4): the
    carry-seeded CHUNK scans reproduce the 1-GPU result on sparse-ones data
    (every prefix exact) and the full reduce the exact total."""
    n = 1 << 31
    g = torch.Generator(device=cuda)
    g.manual_seed(shards)
    xd = (torch.rand(n, device=cuda, generator=g) < 2.0 ** -9).to(torch.float16)
    total = xd.double().sum().item()
    assert Dist.virtual_full_reduce(xd, shards, torch.float64).item() == total
    a = Dist.virtual_full_scan(xd, shards, torch.float32, exclusive=True)
    from paper_1811_09736_b200 import _device as D
    b = D.full_scan(xd, torch.float32, exclusive=True)
    assert torch.equal(a, b)
