"""Query sharding across ranks (one process per GPU, no data-path collective).

Queries are independent given the immutable index (SPEC.md:335-336 of the
reference), so the only multi-GPU work is: replicate the index, give rank r
a contiguous shard, and gather results on the host.  torch.distributed is
used for plumbing only (barriers and the max-over-ranks timing reduction).
"""

from __future__ import annotations

import os

import numpy as np


def env_rank() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def shard_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of `count` queries for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = count * rank // world
    hi = count * (rank + 1) // world
    return lo, hi


def gather_fixed(local: np.ndarray, world: int) -> np.ndarray:
    """All-gather of a fixed-width per-query result (e.g. (N_r, 2) intervals), rank order.

    Uses torch.distributed (gloo on CPU tensors); off the timed path.
    """
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    local = np.ascontiguousarray(local)
    dtype = local.dtype
    # gloo carries no unsigned 32/64-bit tensors: ship the same bytes as signed
    wire = {np.dtype(np.uint32): np.int32, np.dtype(np.uint64): np.int64, np.dtype(np.uint16): np.int16}
    if dtype in wire:
        local = local.view(wire[dtype])
    t = torch.from_numpy(local)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([t.shape[0]], dtype=torch.int64))
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype)
    pad[: t.shape[0]] = t
    bufs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return np.concatenate([b[: int(s.item())].numpy() for b, s in zip(bufs, sizes)]).view(dtype)


def gather_csr(offsets: np.ndarray, values: list[np.ndarray], world: int):
    """All-gather of CSR results (per-query variable-length lists), rank order.

    Returns (offsets, values) for the concatenated query range with the
    offsets re-based: the host gather of SURVEY §8(e).
    """
    counts = np.diff(offsets.astype(np.int64))
    all_counts = gather_fixed(counts, world)
    all_vals = [gather_fixed(v, world) for v in values]
    out = np.zeros(all_counts.size + 1, dtype=np.uint64)
    np.cumsum(all_counts, out=out[1:])
    return out, all_vals


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank timing over all ranks (the bench reports the slowest rank)."""
    if world == 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
