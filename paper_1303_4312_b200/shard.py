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


class DistributedMerge:
    """A multi-GPU stable merge of a distributed input, set up once and run
    many times (Algorithm 2 with one worker per GPU,
    PAPER.md:770-786).

    Rank r of the process group holds the r-th contiguous piece of A and of B
    (device tensors; every piece but the last a multiple of 16 bytes, and of 4
    elements with payloads), optionally with uint32 payload pieces.  Set-up
    exchanges CUDA IPC handles of the pieces once (a host-side all-gather of
    handles, no data).  Each `run()` then merges THIS rank's output range
    [floor(r*T/world), floor((r+1)*T/world)) in one kernel launch on the
    current stream: the kernel co-ranks its tiles through a piece table and
    streams every window straight out of the owning GPU's memory (NVLink for
    peer pieces) -- no data-path collective.  `close()` waits until every rank
    is done reading its peers' pieces and drops the mappings."""

    def __init__(self, a_local, b_local, group=None, a_vals=None, b_vals=None):
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor

        self.group = group
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        self.pairs = a_vals is not None

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
            for x in range(4 if self.pairs else 2):
                if r == rank:
                    pieces[x].append(local[x])
                else:
                    h = hs[x]
                    pieces[x].append(h[0](*h[1]) if h else local[x][:0])
        self.pieces = pieces
        self.total = sum(h[2] + h[3] for h in handles)
        self.lo, self.hi = shard_ranges(self.total, world)[rank]
        dev = a_local.device
        self.out = torch.empty(self.hi - self.lo, dtype=a_local.dtype, device=dev)
        self.out_vals = (torch.empty(self.hi - self.lo, dtype=torch.uint32, device=dev)
                         if self.pairs else None)

    def run(self):
        """Enqueue this rank's range merge on the current stream."""
        from .comerge import merge_pieces
        p = self.pieces
        if self.pairs:
            merge_pieces(p[0], p[1], self.lo, self.hi, out=self.out, a_val_pieces=p[2],
                         b_val_pieces=p[3], out_vals=self.out_vals)
        else:
            merge_pieces(p[0], p[1], self.lo, self.hi, out=self.out)

    def close(self):
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        dist.barrier(group=self.group)  # every rank is done reading its peers' pieces
        self.pieces = None


def merge_distributed(a_local, b_local, group=None, a_vals=None, b_vals=None):
    """One multi-GPU stable merge of a distributed input (see DistributedMerge).
    Returns (out_begin, out_keys) or (out_begin, out_keys, out_vals)."""
    dm = DistributedMerge(a_local, b_local, group, a_vals, b_vals)
    dm.run()
    dm.close()
    return (dm.lo, dm.out, dm.out_vals) if dm.pairs else (dm.lo, dm.out)
