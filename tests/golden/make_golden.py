"""Generate tests/golden/ref_vectors.npz from the UNMODIFIED reference.

Runs the reference library compiled from /root/reference/proj
(oracle/_ref/libcomerge_ref.so, built by `make -C oracle`) on seeded inputs
and stores inputs + outputs as small fixtures.  The GPU box has no
/root/reference, so these committed vectors are how the -m gpu parity tests
and the CPU oracle tests see the reference's own answers.

    python tests/golden/make_golden.py        # rewrites ref_vectors.npz
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.py import Ref, to_aos  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.npz")
DTYPES = {"i32": np.int32, "u32": np.uint32, "u64": np.uint64}


def sorted_keys(rng, dtype, length, alphabet):
    """Sorted keys over [lo, lo+alphabet) (full dtype range when alphabet == 0)."""
    info = np.iinfo(dtype)
    if alphabet == 0:
        if dtype == np.uint64:
            v = rng.integers(0, 2**64, size=length, dtype=np.uint64)
        else:
            v = rng.integers(info.min, int(info.max) + 1, size=length, dtype=np.int64).astype(dtype)
    else:
        lo = -(alphabet // 2) if dtype == np.int32 else 0
        v = (rng.integers(0, alphabet, size=length) + lo).astype(dtype)
    return np.sort(v)


def main():
    ref = Ref()
    rng = np.random.default_rng(20260101)
    fx = {}

    # 1. co_rank: every rank of small dense-duplicate instances, with the
    #    reference's iteration/comparison counts (corank.hpp:89-119).
    for name, dt in DTYPES.items():
        for c in range(6):
            m, n = int(rng.integers(0, 40)), int(rng.integers(0, 40))
            if c == 0:
                m = 0
            if c == 1:
                n = 0
            alphabet = [3, 2, 5, 0, 8, 1][c]
            a, b = sorted_keys(rng, dt, m, alphabet), sorted_keys(rng, dt, n, alphabet)
            res = np.array([ref.co_rank(i, a, b, stats=True) for i in range(m + n + 1)],
                           dtype=object)
            fx[f"corank__{name}__{c}__a"] = a
            fx[f"corank__{name}__{c}__b"] = b
            fx[f"corank__{name}__{c}__j"] = np.array([r[0][0] for r in res], np.uint64)
            fx[f"corank__{name}__{c}__it"] = np.array([r[1][0] for r in res], np.uint32)
            fx[f"corank__{name}__{c}__cmp"] = np.array([r[1][1] for r in res], np.uint32)

    # 2. keys-only merge_parallel (threads mode), ragged and degenerate shapes,
    #    plus the report's block_sizes / corank_iterations for p = 7.
    shapes = [(0, 0), (0, 17), (23, 0), (1, 1), (1000, 3), (3, 1000), (4096, 4096),
              (5000, 1234), (777, 7777)]
    for name, dt in DTYPES.items():
        for c, (m, n) in enumerate(shapes):
            alphabet = [0, 4, 16, 1, 0, 0, 3, 0, 1000][c]
            a, b = sorted_keys(rng, dt, m, alphabet), sorted_keys(rng, dt, n, alphabet)
            out, rep, bs, its = ref.merge_parallel(a, b, 7, simulated=False)
            fx[f"merge__{name}__{c}__a"] = a
            fx[f"merge__{name}__{c}__b"] = b
            fx[f"merge__{name}__{c}__out"] = out
            fx[f"merge__{name}__{c}__bs7"] = bs
            fx[f"merge__{name}__{c}__it7"] = its

    # 3. key-value merges: payload = source-tagged index (A: i, B: i | 1<<31),
    #    massive duplicates, merged by the reference over {key, val} structs.
    for name, dt in DTYPES.items():
        kind = {"i32": 0, "u32": 1, "u64": 2}[name]
        for c, (m, n, alphabet) in enumerate([(3000, 2500, 16), (100, 5000, 2), (4000, 0, 4),
                                              (1, 1, 1), (2048, 2048, 0)]):
            a, b = sorted_keys(rng, dt, m, alphabet), sorted_keys(rng, dt, n, alphabet)
            av = np.arange(m, dtype=np.uint32)
            bv = np.arange(n, dtype=np.uint32) | np.uint32(1 << 31)
            out, _ = ref.merge_parallel_kv(to_aos(a, av), to_aos(b, bv), 5)
            assert kind == {np.int32: 0, np.uint32: 1, np.uint64: 2}[dt]
            fx[f"kv__{name}__{c}__a"] = a
            fx[f"kv__{name}__{c}__b"] = b
            fx[f"kv__{name}__{c}__outk"] = np.ascontiguousarray(out["key"])
            fx[f"kv__{name}__{c}__outv"] = np.ascontiguousarray(out["val"])

    # 4. segmented batches: per-pair stable_merge (merge.hpp:52-68), sizes
    #    including empty pairs.
    for name, dt in (("i32", np.int32), ("u32", np.uint32)):
        for c, (nseg, maxlen) in enumerate([(37, 300), (200, 20), (5, 4096)]):
            ma = rng.integers(0, maxlen + 1, nseg)
            nb = rng.integers(0, maxlen + 1, nseg)
            ma[::7] = 0
            nb[::5] = 0
            a = np.concatenate([sorted_keys(rng, dt, int(x), 64) for x in ma] +
                               [np.empty(0, dt)])
            b = np.concatenate([sorted_keys(rng, dt, int(x), 64) for x in nb] +
                               [np.empty(0, dt)])
            a_off = np.concatenate([[0], np.cumsum(ma)]).astype(np.uint64)
            b_off = np.concatenate([[0], np.cumsum(nb)]).astype(np.uint64)
            out, _ = ref.merge_segmented(a, a_off, b, b_off, threads=2)
            fx[f"seg__{name}__{c}__a"] = a
            fx[f"seg__{name}__{c}__b"] = b
            fx[f"seg__{name}__{c}__aoff"] = a_off
            fx[f"seg__{name}__{c}__boff"] = b_off
            fx[f"seg__{name}__{c}__out"] = out

    # 5. the reference's seeded generator (generate.cpp:69-97), every kind,
    #    pinning the splitmix64 stream recipe used by the GPU generator.
    for dist in range(7):
        a, b = ref.generate(dist, 1000 + dist, [0, 0, 16, 0, 0, 0, 32][dist], 513, 300)
        fx[f"gen__{dist}__a"] = a
        fx[f"gen__{dist}__b"] = b
        fx[f"gen__{dist}__seed"] = np.array([1000 + dist, [0, 0, 16, 0, 0, 0, 32][dist]],
                                            np.uint64)

    # 6. plan() on random instances (parallel.hpp:94-115)
    for c in range(4):
        a = sorted_keys(rng, np.uint64, int(rng.integers(0, 300)), 8)
        b = sorted_keys(rng, np.uint64, int(rng.integers(0, 300)), 8)
        w = int(rng.integers(1, 40))
        fx[f"plan__{c}__a"] = a
        fx[f"plan__{c}__b"] = b
        fx[f"plan__{c}__blocks"] = ref.plan(a, b, w)

    # 7. multiset checksum (keys.hpp:50-55)
    keys = sorted_keys(rng, np.uint64, 1000, 0)
    fx["checksum__keys"] = keys
    fx["checksum__value"] = np.array([ref.checksum(keys)], np.uint64)

    # 8. merge_options::count_comparisons (parallel.hpp:41, :253-280): the
    #    reference's total comparison count for several worker counts, both
    #    modes (simulated, so deterministic), duplicate-heavy and skewed inputs.
    crng = np.random.default_rng(20261019)
    cshapes = [(0, 9, 4), (9, 0, 4), (1, 1, 1), (500, 700, 3), (2000, 37, 0), (37, 2000, 0),
               (1500, 1500, 1), (4096, 4095, 64)]
    workers_set = [1, 2, 3, 7, 16, 100]
    for name, dt in DTYPES.items():
        for c, (m, n, alphabet) in enumerate(cshapes):
            a, b = sorted_keys(crng, dt, m, alphabet), sorted_keys(crng, dt, n, alphabet)
            counts = np.zeros((len(workers_set), 2), np.uint64)
            for wi, w in enumerate(workers_set):
                for synced in (0, 1):
                    _, rep, _, _ = ref.merge_parallel(a, b, w, simulated=True, synced=bool(synced),
                                                      count=True)
                    assert rep.has_comparisons
                    counts[wi, synced] = rep.comparisons
            fx[f"cmp__{name}__{c}__a"] = a
            fx[f"cmp__{name}__{c}__b"] = b
            fx[f"cmp__{name}__{c}__counts"] = counts
    fx["cmp__workers"] = np.array(workers_set, np.uint64)

    # 9. what the reference CLI's `bench` measures (experiment.cpp:49-121):
    #    for every distribution (generate.cpp), seed 5, m = n = 1000, the
    #    comparison count of p = 1, 2, 4 and the generated inputs' checksums.
    dists = [("uniform", 0, 0), ("all-equal", 1, 0), ("few-distinct:16", 2, 16),
             ("disjoint", 3, 0), ("interleaved", 4, 0), ("organ-pipe", 5, 0), ("runs:32", 6, 32)]
    for token, kind, param in dists:
        a, b = ref.generate(kind, 5, param, 1000, 1000)
        counts = []
        for w in (1, 2, 4):
            _, rep, _, _ = ref.merge_parallel(a, b, w, simulated=True, count=True)
            counts.append(rep.comparisons)
        fx[f"clibench__{token}__counts"] = np.array(counts, np.uint64)
        fx[f"clibench__{token}__checksum"] = np.array([ref.checksum(a), ref.checksum(b)],
                                                      np.uint64)

    np.savez_compressed(OUT, **fx)
    print(f"wrote {OUT}: {len(fx)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
