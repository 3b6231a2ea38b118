"""Multi-GPU placement for the KV-buffered decode path.

Every (request slot, V head) pair is independent, so the path
shards with no exchange step:

* data parallel over requests (the headline mode): rank g of G owns a
  contiguous block of the global batch; each rank runs its own la_buf
  handles, no collective on the data path ("scaling": "weak" when the per-GPU
  batch is fixed);
* tensor parallel over heads: rank g owns QK heads [g Hk/G, (g+1) Hk/G) and
  the V heads that read them (V head h reads QK head h // (Hv/Hk)), so every
  GQA group stays on one rank; head outputs are gathered with one all-gather
  (la_tp_allgather) into a head-major [Hv][B][d_v] buffer.

Only host-side arithmetic lives here (index ranges, the config-5 long/short
mix, and the max-over-ranks timing reduction); the kernels never see a rank.
"""
from __future__ import annotations

from dataclasses import dataclass


def shard_range(global_batch: int, rank: int, world: int):
    """Contiguous slot block [first, first + n) of `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(global_batch, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def head_range(n_qk_heads: int, n_v_heads: int, rank: int, world: int):
    """(qk_first, n_qk, v_first, n_v) for tensor parallelism over heads."""
    if n_qk_heads % world or n_v_heads % n_qk_heads:
        raise ValueError("heads must divide evenly over ranks")
    nq = n_qk_heads // world
    g = n_v_heads // n_qk_heads
    return rank * nq, nq, rank * nq * g, nq * g


@dataclass(frozen=True)
class MixedShard:
    """Config 5 placement: this rank's long (chunkwise) and short (direct)
    requests, assigned round-robin so every rank gets the same mix."""
    long_ids: tuple
    short_ids: tuple


def mixed_assignment(n_long: int, n_short: int, rank: int, world: int) -> MixedShard:
    return MixedShard(tuple(range(rank, n_long, world)), tuple(range(n_long + rank, n_long + n_short, world)))


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank timing over the default process group (1 rank: x)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
