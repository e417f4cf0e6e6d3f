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


def merge_distributed(a_local, b_local, group=None, a_vals=None, b_vals=None):
    """Multi-GPU stable merge of a distributed input.

    Rank r of the process group holds the r-th contiguous piece of A and of B
    (device tensors; every piece but the last a multiple of 16 bytes, and of 4
    elements with payloads), optionally with uint32 payload pieces.  The ranks
    exchange CUDA IPC handles of their pieces once (a host-side all-gather of
    handles, no data), then each rank merges ITS output range
    [floor(r*T/world), floor((r+1)*T/world)) in one kernel that co-ranks its
    tiles and streams its windows straight out of the peers' memory over
    NVLink -- Algorithm 2 with one worker per GPU, no data-path collective.
    Returns (out_begin, out_keys) or (out_begin, out_keys, out_vals).  The peer
    mappings are dropped after a barrier (every rank done reading)."""
    import torch
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor

    from .comerge import merge_pieces
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    pairs = a_vals is not None

    def share(t):  # CUDA IPC handle of a piece (None for an empty one)
        return reduce_tensor(t) if t is not None and t.numel() else None

    mine = (share(a_local), share(b_local), share(a_vals), share(b_vals))
    handles = [None] * world
    dist.all_gather_object(handles, (rank, mine, int(a_local.numel()), int(b_local.numel())),
                           group=group)
    handles.sort(key=lambda h: h[0])
    local = (a_local, b_local, a_vals, b_vals)
    pieces = [[], [], [], []]
    for r, hs, _, _ in handles:
        for x in range(4 if pairs else 2):
            if r == rank:
                pieces[x].append(local[x])
            else:
                h = hs[x]
                pieces[x].append(h[0](*h[1]) if h else local[x][:0])
    total = sum(h[2] + h[3] for h in handles)
    lo, hi = shard_ranges(total, world)[rank]
    if pairs:
        ok, ov = merge_pieces(pieces[0], pieces[1], lo, hi, a_val_pieces=pieces[2],
                              b_val_pieces=pieces[3])
    else:
        ok = merge_pieces(pieces[0], pieces[1], lo, hi)
    torch.cuda.synchronize()
    dist.barrier(group=group)  # every rank is done reading its peers' pieces
    del pieces
    return (lo, ok, ov) if pairs else (lo, ok)
