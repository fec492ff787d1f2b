"""The ABI's concurrency claims (include/tc_collectives.h: stream-ordered,
reentrant across host threads on different streams, each with its own
workspace) and CUDA-graph capture of the launch-bound inner loop."""

import threading

import numpy as np
import pytest
import torch

from paper_1811_09736_b200 import _device as D

pytestmark = pytest.mark.gpu


def _ops(x, off):
    return [
        D.seg_reduce(x, 300, torch.float32),
        D.seg_scan(x, 4096, torch.float32),
        D.full_scan(x, torch.float32, exclusive=True),
        D.irreg_reduce(x, off, torch.float32, validate=False),
        D.irreg_scan(x, off, torch.float32, validate=False),
    ]


def _inputs(cuda, seed):
    g = torch.Generator(device=cuda)
    g.manual_seed(seed)
    n = (1 << 22) + 4099
    x = torch.randint(0, 4, (n,), device=cuda, generator=g, dtype=torch.int32).to(torch.float16)
    lens = torch.randint(0, 200, (n // 90,), device=cuda, generator=g, dtype=torch.int64)
    ends = torch.cumsum(lens, 0)
    ends = ends[ends < n]
    off = torch.cat([torch.zeros(1, dtype=torch.int64, device=cuda), ends,
                     torch.tensor([n], device=cuda)])
    return x, off


def test_concurrent_host_threads_on_streams(cuda):
    inputs = [_inputs(cuda, s) for s in range(4)]
    ref = [[o.clone() for o in _ops(x, off)] for x, off in inputs]
    torch.cuda.synchronize()
    results = [None] * 4
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream(device=cuda)
            with torch.cuda.stream(s):
                outs = []
                for _ in range(3):
                    outs = _ops(*inputs[i])
                s.synchronize()
            results[i] = outs
        except Exception as e:  # pragma: no cover - surfaced below
            errors.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
    for i in range(4):
        for a, b in zip(results[i], ref[i]):
            assert torch.equal(a, b)


def test_cuda_graph_capture_and_replay(cuda):
    x, off = _inputs(cuda, 9)
    ref = [o.clone() for o in _ops(x, off)]
    s = torch.cuda.Stream(device=cuda)
    s.wait_stream(torch.cuda.current_stream(cuda))
    with torch.cuda.stream(s):
        _ops(x, off)  # warm: workspace + function attributes outside the capture
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            outs = _ops(x, off)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    for a, b in zip(outs, ref):
        assert torch.equal(a, b)
    # new data through the same graph: results follow the input buffer
    x.copy_(torch.flip(x, [0]))
    g.replay()
    torch.cuda.synchronize()
    exp = D.seg_reduce(x, 300, torch.float32)
    assert torch.equal(outs[0], exp)
    assert np.isfinite(outs[2].cpu().numpy()).all()
