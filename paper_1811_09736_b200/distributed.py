"""Multi-GPU sharding of the collectives (one process per GPU, NCCL over
NVLink/NVSwitch through ``torch.distributed``).

SURVEY.md section 8(e):

* Segmented reduce / scan shard by WHOLE segments with no communication:
  rank r owns segments [nseg*r/W, nseg*(r+1)/W) (``shard_bounds``).
* Full reduce: every rank computes one fp64 partial of its shard on the
  device (tc_full_reduce, TC_F64), one NCCL ``all_gather`` of the W
  partials (8 B each), then every rank sums them in rank order 0..W-1 --
  deterministic and symmetric -- and rounds once to the output dtype.
* Full scan: local fp64 total -> ``all_gather`` of the W totals -> on
  device carry_r = sum_{h<r} total_h (rank order) -> one carry-seeded scan
  of the shard (tc_seg_scan with carry_in), i.e. the carry-add is fused
  into the scan's epilogue.  Reduce-then-scan reads the shard twice
  ((4 + o) bytes/element) but needs exactly one exchange and no second
  pass over the output.

The per-shard device work goes through ``ops`` (default: the CUDA kernels
in ``_device``), so the host-side exchange logic is testable on CPU with
the gloo backend (tests/test_distributed_cpu.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n: int, seg: int, world: int, rank: int) -> tuple[int, int]:
    """Element range [lo, hi) of rank's shard: contiguous whole segments."""
    if seg < 1 or n < 0 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")
    nseg = -(-n // seg)
    k0 = nseg * rank // world
    k1 = nseg * (rank + 1) // world
    return min(k0 * seg, n), min(k1 * seg, n)


def even_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Element range of rank's shard for one-segment (full) ops.  Interior
    bounds are multiples of 8 elements, so every shard of a 16-byte aligned
    vector is itself 16-byte aligned (the kernels' TMA requirement: no copy)."""
    if n < 0 or not 0 <= rank < world:
        raise ValueError("bad shard arguments")

    def cut(r):
        return n if r >= world else (n * r // world) // 8 * 8

    return cut(rank), cut(rank + 1)


class DeviceOps:
    """Per-shard compute on the local GPU (the product path)."""

    @staticmethod
    def full_reduce_f64(x: torch.Tensor) -> torch.Tensor:
        from . import _device

        return _device.full_reduce(x, torch.float64)

    @staticmethod
    def seg_reduce(x: torch.Tensor, seg: int, out_dtype) -> torch.Tensor:
        from . import _device

        return _device.seg_reduce(x, seg, out_dtype)

    @staticmethod
    def seg_scan(x: torch.Tensor, seg: int, out_dtype, exclusive: bool,
                 carry_in: torch.Tensor | None) -> torch.Tensor:
        from . import _device

        return _device.seg_scan(x, seg, out_dtype, exclusive=exclusive, carry_in=carry_in)


def _world(group):
    return dist.get_world_size(group), dist.get_rank(group)


def _gather_partials(part: torch.Tensor, group) -> list[torch.Tensor]:
    world, _ = _world(group)
    bufs = [torch.empty_like(part) for _ in range(world)]
    dist.all_gather(bufs, part, group=group)
    return bufs


# The exchange arithmetic, shared by the process-group path and the
# single-process virtual-shards path so both are bit-identical: every rank
# sums the gathered fp64 partials in rank order 0..W-1.


def combine_partials(parts: list[torch.Tensor]) -> torch.Tensor:
    """Full-reduce result from the W per-shard fp64 partials (rank order)."""
    acc = parts[0].clone()
    for p in parts[1:]:
        acc += p
    return acc


def carry_for(parts: list[torch.Tensor], rank: int) -> torch.Tensor:
    """Exclusive carry entering shard ``rank``: sum of the partials of the
    lower ranks in rank order (fp64, on the partials' device)."""
    carry = torch.zeros(1, dtype=torch.float64, device=parts[0].device)
    for p in parts[:rank]:
        carry += p
    return carry


def sharded_segmented_reduce(x_local: torch.Tensor, seg: int, out_dtype=torch.float16,
                             ops=DeviceOps) -> torch.Tensor:
    """Sums of the local whole segments (no communication)."""
    return ops.seg_reduce(x_local, seg, out_dtype)


def sharded_segmented_scan(x_local: torch.Tensor, seg: int, out_dtype=torch.float16,
                           exclusive: bool = False, ops=DeviceOps) -> torch.Tensor:
    """Prefix sums of the local whole segments (no communication)."""
    return ops.seg_scan(x_local, seg, out_dtype, exclusive, None)


def sharded_full_reduce(x_local: torch.Tensor, out_dtype=torch.float32, group=None,
                        ops=DeviceOps) -> torch.Tensor:
    """Sum over all ranks' shards; every rank receives the 1-element result."""
    part = ops.full_reduce_f64(x_local).reshape(1).to(torch.float64)
    return combine_partials(_gather_partials(part, group)).to(out_dtype)


def sharded_full_scan(x_local: torch.Tensor, out_dtype=torch.float32, exclusive: bool = False,
                      group=None, ops=DeviceOps) -> torch.Tensor:
    """One-segment scan over the concatenation of all ranks' shards (rank
    order); returns this rank's slice of the result."""
    _, rank = _world(group)
    part = ops.full_reduce_f64(x_local).reshape(1).to(torch.float64)
    carry = carry_for(_gather_partials(part, group), rank)
    return ops.seg_scan(x_local, max(int(x_local.numel()), 1), out_dtype, exclusive, carry)


# ---------------------------------------------------------------------------
# Virtual G shards ("a single-process virtual G shards
# mode for CI"): the same per-shard kernels and the same exchange arithmetic,
# with the all_gather replaced by an in-process list -- G shards of one
# vector processed one after another on the local GPU.  Results are
# bit-identical to a G-rank run of the functions above (same shard bounds,
# same rank-order fp64 combine).


def virtual_full_reduce(x: torch.Tensor, shards: int, out_dtype=torch.float32,
                        ops=DeviceOps) -> torch.Tensor:
    n = int(x.numel())
    parts = [ops.full_reduce_f64(x[slice(*even_bounds(n, shards, r))]).reshape(1).to(torch.float64)
             for r in range(shards)]
    return combine_partials(parts).to(out_dtype)


def virtual_full_scan(x: torch.Tensor, shards: int, out_dtype=torch.float32,
                      exclusive: bool = False, ops=DeviceOps) -> torch.Tensor:
    n = int(x.numel())
    bounds = [even_bounds(n, shards, r) for r in range(shards)]
    parts = [ops.full_reduce_f64(x[lo:hi]).reshape(1).to(torch.float64) for lo, hi in bounds]
    outs = [ops.seg_scan(x[lo:hi], max(hi - lo, 1), out_dtype, exclusive, carry_for(parts, r))
            for r, (lo, hi) in enumerate(bounds)]
    return torch.cat(outs)


def virtual_segmented_reduce(x: torch.Tensor, seg: int, shards: int, out_dtype=torch.float16,
                             ops=DeviceOps) -> torch.Tensor:
    n = int(x.numel())
    outs = [ops.seg_reduce(x[lo:hi], seg, out_dtype)
            for lo, hi in (shard_bounds(n, seg, shards, r) for r in range(shards)) if hi > lo]
    return torch.cat(outs)


def virtual_segmented_scan(x: torch.Tensor, seg: int, shards: int, out_dtype=torch.float16,
                           exclusive: bool = False, ops=DeviceOps) -> torch.Tensor:
    n = int(x.numel())
    outs = [ops.seg_scan(x[lo:hi], seg, out_dtype, exclusive, None)
            for lo, hi in (shard_bounds(n, seg, shards, r) for r in range(shards)) if hi > lo]
    return torch.cat(outs)
