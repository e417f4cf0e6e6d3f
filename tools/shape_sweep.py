"""Kernel time and % of the copy peak over adversarial input shapes (no BASELINE
config): all-equal keys, disjoint ranges, perfect interleave, long alternating
runs, one-element sides, 64-bit keys only.  Bench timing (L2 flushed between
steps, events around the merge kernel); every output checked (sorted, and for
key-value merges stable: payloads A-first among equal keys, increasing per
source).

    python tools/shape_sweep.py [--lg 26] [--steps 10]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def shapes(torch, dev, lg):
    n = 1 << lg
    i32, u64 = torch.int32, torch.int64  # uint64 keys as int64 >= 0 (same order)
    ar = lambda k, dt: torch.arange(k, dtype=dt, device=dev)  # noqa: E731
    yield "equal keys", torch.zeros(n, dtype=i32, device=dev), torch.zeros(n, dtype=i32, device=dev)
    yield "disjoint A<B", ar(n, i32), ar(n, i32) + n
    yield "disjoint B<A", ar(n, i32) + n, ar(n, i32)
    yield "interleave", ar(n, i32) * 2, ar(n, i32) * 2 + 1
    run = 1 << 20  # alternating runs of 2^20: A holds even blocks, B odd blocks
    yield "alt runs 2^20", ar(n, i32) + (ar(n, i32) // run) * run, ar(n, i32) + (ar(n, i32) // run + 1) * run
    yield "m=1", torch.tensor([n // 2], dtype=i32, device=dev), ar(2 * n - 1, i32)
    yield "n=1", ar(2 * n - 1, i32), torch.tensor([n // 2], dtype=i32, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    rnd = lambda hi: torch.sort(torch.randint(0, hi, (n,), dtype=u64, device=dev, generator=g))[0]  # noqa: E731
    yield "u64 uniform", rnd(1 << 62).view(torch.uint64), rnd(1 << 62).view(torch.uint64)
    yield "u64 4 distinct", rnd(4).view(torch.uint64), rnd(4).view(torch.uint64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lg", type=int, default=26)
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import bench
    import paper_1303_4312_b200 as P
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    peak = bench.peak_hbm()[0]
    for name, a, b in shapes(torch, dev, args.lg):
        total = a.numel() + b.numel()
        for pairs in (False, True):
            out = torch.empty(total, dtype=a.dtype, device=dev)
            if pairs:
                av = torch.arange(a.numel(), dtype=torch.int32, device=dev).view(torch.uint32)
                bv = (torch.arange(b.numel(), dtype=torch.int32, device=dev) | -2**31).view(torch.uint32)
                ov = torch.empty(total, dtype=torch.uint32, device=dev)
                step = lambda: P.merge_pairs(a, av, b, bv, out, ov)  # noqa: E731
            else:
                step = lambda: P.stable_merge(a, b, out)  # noqa: E731
            r = bench.time_steps(step, args.steps, 3, dev, flush)
            us = statistics.median(r["kern_ms"]) * 1e3
            eb = a.element_size() + (4 if pairs else 0)
            gbs = 2 * total * eb / (us * 1e-6) / 1e9
            # checks: sorted; stable (equal keys: A's payloads (< 2^31) first, each source increasing)
            o = out.view(torch.int64) if a.dtype == torch.uint64 else out
            ok = bool((o[1:] >= o[:-1]).all())
            if pairs:
                v = ov.view(torch.int32).to(torch.int64) & 0xffffffff
                same = o[1:] == o[:-1]
                ok = ok and bool((~same | (v[1:] > v[:-1])).all())
            print(f"{name:16s} {'pairs' if pairs else 'keys ':5s} {str(a.dtype)[6:]:7s} "
                  f"{total / 1e6:7.1f} M  {us:8.1f} us  {gbs:7.0f} GB/s  {100 * gbs / peak:5.1f}%  "
                  f"path {r['path']}  {'ok' if ok else 'WRONG'}", flush=True)
            del out
        del a, b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
