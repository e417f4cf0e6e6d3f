"""Randomised differential testing of every device entry point against the C
oracle, for a fixed wall-clock budget:  python tools/fuzz.py [seconds] [seed]

Each round draws an entry point (keys / key-value merge, segmented batch,
sort, sort of pairs, pieced range merge, host-buffer merges), a key type, a
size (empty, tiny, around tile multiples, up to a few million), a distribution
(all equal, few distinct, uniform, disjoint ranges, one side tiny) and a
misalignment of the views, runs it on cuda:0 and compares bit-exactly."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1303_4312_b200 as P  # noqa: E402
from oracle.py import Port  # noqa: E402

port = Port()
dev = torch.device("cuda:0")
TILES = [7936, 3840, 2816]


def size(rng):
    r = rng.random()
    if r < 0.1:
        return int(rng.integers(0, 3))
    if r < 0.3:
        return int(rng.integers(0, 5000))
    if r < 0.5:
        t = TILES[int(rng.integers(0, 3))]
        return max(0, t * int(rng.integers(1, 40)) + int(rng.integers(-2, 3)))
    return int(rng.integers(0, 3_000_000))


def draw(rng, dt, n, dist):
    if dist == 0:
        v = np.full(n, 7)
    elif dist == 1:
        v = rng.integers(0, int(rng.integers(1, 20)), n)
    elif dist == 2:
        hi = 2**63 if dt == np.uint64 else 2**31
        v = rng.integers(0, hi, n, dtype=np.uint64 if dt == np.uint64 else np.int64)
    else:
        v = rng.integers(0, 1000, n) + (10_000 if rng.random() < 0.5 else 0)
    v = np.sort(v.astype(dt))
    return v


def view(rng, x):
    """device copy, sometimes at an offset of 1-3 elements (misaligned view)"""
    off = int(rng.integers(0, 4)) if rng.random() < 0.3 else 0
    t = torch.empty(len(x) + off, dtype=P_T[x.dtype], device=dev)
    t[off:] = torch.from_numpy(np.ascontiguousarray(x)).to(dev) if len(x) else t[off:]
    return t[off:]


P_T = {np.dtype(np.int32): torch.int32, np.dtype(np.uint32): torch.uint32,
       np.dtype(np.uint64): torch.uint64}


def one(rng):
    kinds = ["keys", "pairs", "seg", "sort", "sortp", "pieces", "host", "hostp", "rec", "hostrec",
             "recapi"]
    kind = kinds[int(rng.integers(0, len(kinds)))]
    dt = [np.int32, np.uint32, np.uint64][int(rng.integers(0, 3))]
    if kind == "seg" and dt == np.uint64:
        dt = np.int32
    m, n = size(rng), size(rng)
    if rng.random() < 0.15:
        m = int(rng.integers(0, 50))  # one side tiny
    dist = int(rng.integers(0, 4))
    a, b = draw(rng, dt, m, dist), draw(rng, dt, n, dist)
    tag = f"{kind} {np.dtype(dt).name} m={m} n={n} dist={dist}"
    if kind == "keys":
        out = P.stable_merge(view(rng, a), view(rng, b))
        assert np.array_equal(out.cpu().numpy(), port.merge(a, b)), tag
    elif kind == "pairs":
        av = np.arange(m, dtype=np.uint32)
        bv = np.arange(n, dtype=np.uint32) | np.uint32(1 << 31)
        ok, ov = P.merge_pairs(view(rng, a), view(rng, av), view(rng, b), view(rng, bv))
        ek, ev = port.merge(a, b, av, bv)
        assert np.array_equal(ok.cpu().numpy(), ek) and np.array_equal(ov.cpu().numpy(), ev), tag
    elif kind == "seg":
        ns = int(rng.integers(1, 3000))
        la = rng.integers(0, int(rng.integers(1, 5000)), ns)
        lb = rng.integers(0, int(rng.integers(1, 5000)), ns)
        la[rng.random(ns) < 0.1] = 0
        sa = np.concatenate([draw(rng, dt, int(x), dist) for x in la] + [np.empty(0, dt)])
        sb = np.concatenate([draw(rng, dt, int(x), dist) for x in lb] + [np.empty(0, dt)])
        ao = np.concatenate([[0], np.cumsum(la)]).astype(np.uint64)
        bo = np.concatenate([[0], np.cumsum(lb)]).astype(np.uint64)
        out = P.merge_segmented(torch.from_numpy(sa).to(dev), torch.from_numpy(ao).to(dev),
                                torch.from_numpy(sb).to(dev), torch.from_numpy(bo).to(dev))
        assert np.array_equal(out.cpu().numpy(), port.merge_segmented(sa, ao, sb, bo)), \
            f"seg {np.dtype(dt).name} nseg={ns} total={len(sa) + len(sb)}"
    elif kind in ("sort", "sortp"):
        k = rng.permutation(np.concatenate([a, b])) if m + n else np.empty(0, dt)
        if kind == "sort":
            out = P.sort(torch.from_numpy(k).to(dev))
            assert np.array_equal(out.cpu().numpy(), port.merge_sort(k)), tag
        else:
            v = np.arange(len(k), dtype=np.uint32)
            sk, sv = P.sort_pairs(torch.from_numpy(k).to(dev), torch.from_numpy(v).to(dev))
            ek, ev = port.merge_sort_pairs(k, v)
            assert np.array_equal(sk.cpu().numpy(), ek) and np.array_equal(sv.cpu().numpy(), ev), tag
    elif kind == "pieces":
        vece = 16 // np.dtype(dt).itemsize
        def cut(x):
            q = int(rng.integers(1, 5))
            pts = sorted(int(c) // vece * vece for c in rng.integers(0, len(x) + 1, q - 1))
            pts = [0] + pts + [len(x)]
            return [torch.from_numpy(np.ascontiguousarray(x[pts[i]:pts[i + 1]])).to(dev)
                    for i in range(len(pts) - 1)]
        total = m + n
        lo = int(rng.integers(0, total + 1))
        hi = int(rng.integers(lo, total + 1))
        out = P.merge_pieces(cut(a), cut(b), lo, hi)
        assert np.array_equal(out.cpu().numpy(), port.merge(a, b)[lo:hi]), tag + f" [{lo},{hi})"
    elif kind == "host":  # host buffers: keys
        out = np.empty(m + n, dt)
        P.merge_parallel(a, b, out, int(rng.integers(1, 40)))
        assert np.array_equal(out, port.merge(a, b)), tag
    elif kind == "recapi":  # co_rank / plan / full report over records = the key arrays'
        m, n = min(m, 200_000), min(n, 200_000)
        a, b = a[:m], b[:n]
        size_b = 16 if dt == np.uint64 else (12 if rng.random() < 0.5 else 8)
        rd = P.record_dtype(dt, 12 if size_b == 12 else None)
        ra, rb = np.zeros(m, rd), np.zeros(n, rd)
        ra["key"], rb["key"] = a, b
        for i in {0, m + n, int(rng.integers(0, m + n + 1)), int(rng.integers(0, m + n + 1))}:
            st = P.CoRankStats()
            got = P.co_rank_records(i, ra, rb, stats=st)
            assert (got, (st.iterations, st.comparisons)) == port.co_rank(i, a, b, stats=True), tag
        w = int(rng.integers(1, 40))
        synced = bool(rng.integers(0, 2))
        bs, its, cmp = port.merge_report(a, b, w, synced)
        out = np.zeros(m + n, rd)
        rep = P.merge_parallel_records(ra, rb, out, w, synced=synced,
                                       opts=P.MergeOptions(count_comparisons=True))
        assert np.array_equal(out["key"], port.merge(a, b)), tag
        assert rep.block_sizes == [int(x) for x in bs[:w]], tag
        assert rep.corank_iterations == [int(x) for x in its], tag
        assert rep.comparisons == cmp, tag
        pl = P.plan_records(ra, rb, w)
        assert [x.out_end - x.out_begin for x in pl] == rep.block_sizes, tag
        assert all(x.a_end - x.a_begin + x.b_end - x.b_begin == x.out_end - x.out_begin
                   for x in pl), tag
    elif kind in ("rec", "hostrec"):  # records: 8 / 12 / 16 bytes, merged by key
        size_b = 16 if dt == np.uint64 else (12 if rng.random() < 0.5 else 8)
        rd = P.record_dtype(dt, 12 if size_b == 12 else None)
        vname = "index" if size_b == 12 else "val"
        ra, rb = np.zeros(m, rd), np.zeros(n, rd)
        ra["key"], rb["key"] = a, b
        ra[vname] = np.arange(m, dtype=np.uint32)
        rb[vname] = np.arange(n, dtype=np.uint32) | np.uint32(1 << 31)
        ek, ev = port.merge(a, b, ra[vname].copy(), rb[vname].copy())
        if kind == "hostrec":
            out, _ = P.merge_records(ra, rb, workers=int(rng.integers(1, 40)))
        else:  # device, at a random 4-byte offset (8-byte for 16-byte records)
            step = 8 if size_b == 16 else 4
            def dview(r):
                raw = r.view(np.uint8)
                off = step * int(rng.integers(0, 4))
                t = torch.zeros(len(raw) + off + 16, dtype=torch.uint8, device=dev)
                t[off:off + len(raw)] = torch.from_numpy(raw.copy()).to(dev)
                return t[off:off + len(raw)]
            o = dview(np.zeros(m + n, rd))
            P.merge_records(dview(ra), dview(rb), o, key_dtype=dt,
                            record_bytes=12 if size_b == 12 else None)
            out = o.cpu().numpy().view(rd)
        assert np.array_equal(out["key"], ek) and np.array_equal(out[vname], ev), \
            tag + f" record {size_b} B"
    else:  # host buffers: key-value (misaligned host views sometimes)
        sh = int(rng.integers(0, 3))
        av = np.arange(m, dtype=np.uint32)
        bv = np.arange(n, dtype=np.uint32) | np.uint32(1 << 31)
        ok = np.empty(m + n + sh, dt)[sh:]
        ov = np.empty(m + n + sh, np.uint32)[sh:]
        P.merge_pairs(a, av, b, bv, ok, ov)
        ek, ev = port.merge(a, b, av, bv)
        assert np.array_equal(ok, ek) and np.array_equal(ov, ev), tag + f" shift={sh}"
    torch.cuda.synchronize()
    return kind


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rng = np.random.default_rng(seed)
    t0, counts = time.time(), {}
    import paper_1303_4312_b200._native as N
    while time.time() - t0 < budget:
        # sometimes another dynamic-tail anchor unit (pipe_args::tail_unit)
        unit = int(rng.integers(1, 8)) if rng.random() < 0.3 else 0
        N.lib.comerge_cuda_set_tuning(0, unit << 15, 0)
        k = one(rng)
        N.lib.comerge_cuda_set_tuning(0, 0, 0)
        counts[k] = counts.get(k, 0) + 1
    print("fuzz: OK", sum(counts.values()), "rounds", counts, flush=True)


if __name__ == "__main__":
    main()
