"""World-size-2 gloo test of the rank-level sharding (host logic, CPU).

Each rank computes its output range (partition_output through the C ABI's host
function) and its input windows from co-ranks of its ends (oracle co-ranks: the
checker), merges its windows with the oracle, and the ranks all-gather: the
ranges must tile [0, m+n) with sizes differing by <= 1 and the concatenated
shards must equal the full stable merge (payload tags prove stability)."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.py import Port
        from paper_1303_4312_b200.shard import shard_ranges, windows_from_coranks
        port_ = Port()
        rng = np.random.default_rng(42)  # same inputs on every rank
        a = np.sort(rng.integers(0, 50, 100_003)).astype(np.int32)
        b = np.sort(rng.integers(0, 50, 77_777)).astype(np.int32)
        av = np.arange(len(a), dtype=np.uint32)
        bv = np.arange(len(b), dtype=np.uint32) | np.uint32(1 << 31)
        total = len(a) + len(b)
        lo, hi = shard_ranges(total, world)[rank]
        sh = windows_from_coranks(rank, lo, hi, port_.co_rank(lo, a, b)[0],
                                  port_.co_rank(hi, a, b)[0])
        k, v = port_.merge(a[sh.a_begin:sh.a_end], b[sh.b_begin:sh.b_end],
                           av[sh.a_begin:sh.a_end], bv[sh.b_begin:sh.b_end])
        sizes = [None] * world
        dist.all_gather_object(sizes, (lo, hi, k.tobytes(), v.tobytes()))
        if rank == 0:
            ek, ev = port_.merge(a, b, av, bv)
            ok = sizes[0][0] == 0 and sizes[-1][1] == total
            ok &= all(sizes[r][1] == sizes[r + 1][0] for r in range(world - 1))
            lens = [s[1] - s[0] for s in sizes]
            ok &= max(lens) - min(lens) <= 1
            keys = np.concatenate([np.frombuffer(s[2], np.int32) for s in sizes])
            vals = np.concatenate([np.frombuffer(s[3], np.uint32) for s in sizes])
            ok &= np.array_equal(keys, ek) and np.array_equal(vals, ev)
            q.put(bool(ok))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_merge():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
