"""Rank-level sharding of one merge: Algorithm 2 with one
worker per GPU rank.

Rank r of `world` owns output ranks [floor(r*T/world), floor((r+1)*T/world))
(partition_output, parallel.hpp:60-67) and needs only the input windows
A[j_r, j_{r+1}) and B[k_r, k_{r+1}) given by the co-ranks of its two ends --
no data-path collective.  On GPUs the co-ranks come from the device batch
kernel (`co_rank_batch`) and the window merge from the device merge kernel;
`shard_ranges` / `windows_from_coranks` are pure host arithmetic (tested with
gloo on CPU).
"""
from __future__ import annotations

from dataclasses import dataclass

from .comerge import co_rank_batch, partition_output, stable_merge


@dataclass(frozen=True)
class Shard:
    rank: int
    out_begin: int
    out_end: int
    a_begin: int = 0
    a_end: int = 0
    b_begin: int = 0
    b_end: int = 0


def shard_ranges(total: int, world: int):
    """Output range of every rank (sizes differ by at most one)."""
    return [(partition_output(total, world, r), partition_output(total, world, r + 1))
            for r in range(world)]


def windows_from_coranks(rank: int, out_begin: int, out_end: int, j_begin: int, j_end: int):
    """Input windows of a rank from the co-ranks (A prefix lengths) of its ends."""
    return Shard(rank, out_begin, out_end, j_begin, j_end, out_begin - j_begin,
                 out_end - j_end)


def merge_shard(a, b, rank: int, world: int, out=None):
    """Merge this rank's share of stable_merge(a, b) on its GPU (a, b: device
    tensors holding the full inputs, e.g. replicated by a broadcast)."""
    import torch
    total = int(a.numel() + b.numel())
    lo, hi = shard_ranges(total, world)[rank]
    ranks = torch.tensor([lo, hi], dtype=torch.uint64, device=a.device)
    j = co_rank_batch(ranks, a, b).cpu().tolist()
    sh = windows_from_coranks(rank, lo, hi, int(j[0]), int(j[1]))
    if out is None:
        out = torch.empty(hi - lo, dtype=a.dtype, device=a.device)
    stable_merge(a[sh.a_begin:sh.a_end], b[sh.b_begin:sh.b_end], out)
    return sh, out
