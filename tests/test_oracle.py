"""CPU tests: pin the C oracle (oracle/comerge_oracle.c) to the reference.

1. The reference's own known-answer tests (tests/golden/kat.json).
2. Vectors produced by the unmodified reference (tests/golden/ref_vectors.npz,
   from tests/golden/make_golden.py).
3. When oracle/_ref is built (this container), live comparisons against the
   compiled reference, mirroring its property tests (corank_test.cpp,
   parallel_test.cpp).
"""
import itertools

import numpy as np
import pytest

from conftest import KEY_DTYPES

from oracle.py import available_ref


def arr(v, dt):
    return np.array(v, dtype=dt)


def kinds_for(values):
    """Key kinds able to hold every value of a KAT."""
    out = ["u64", "u32", "i32"]
    if values and max(values) >= 2**31:
        out = ["u64"]
    return out


# ------------------------------------------------------------------ KATs

def test_kat_co_rank(port, kat):
    for case in kat["co_rank"]:
        for k in kinds_for(case["a"] + case["b"]):
            dt = KEY_DTYPES[k]
            (j, kk), (it, cmp) = port.co_rank(case["i"], arr(case["a"], dt), arr(case["b"], dt),
                                              stats=True)
            assert [j, kk] == case["expect"], case["src"]
            if "iterations" in case:
                assert it == case["iterations"], case["src"]
            if "comparisons" in case:
                assert cmp == case["comparisons"], case["src"]
            if "max_comparisons" in case:
                assert cmp <= case["max_comparisons"], case["src"]


def test_kat_co_rank_errors(port, kat):
    for case in kat["co_rank_errors"]:
        with pytest.raises(IndexError, match=case["message"]):
            port.co_rank(case["i"], arr(case["a"], np.uint64), arr(case["b"], np.uint64))


def test_kat_merge(port, kat):
    for case in kat["merge"]:
        for k in kinds_for(case["a"] + case["b"]):
            dt = KEY_DTYPES[k]
            out = port.merge(arr(case["a"], dt), arr(case["b"], dt))
            assert out.tolist() == case["expect"], case["src"]


def test_kat_merge_tagged(port, kat):
    for case in kat["merge_tagged"]:
        a, b = arr(case["a"], np.uint64), arr(case["b"], np.uint64)
        av = np.arange(len(a), dtype=np.uint32)
        bv = np.arange(len(b), dtype=np.uint32) | np.uint32(1 << 31)
        _, vals = port.merge(a, b, av, bv)
        assert [int(v >> 31) for v in vals] == case["expect_origin"], case["src"]
        assert [int(v & 0x7FFFFFFF) for v in vals] == case["expect_index"], case["src"]


def test_kat_partition_output(port, kat):
    for case in kat["partition_output"]:
        if "expect" in case:
            got = [port.partition_output(case["total"], case["workers"], r)
                   for r in range(case["workers"] + 1)]
            assert got == case["expect"], case["src"]
        else:
            assert port.partition_output(case["total"], case["workers"], case["r"]) == \
                case["expect_r"], case["src"]
    for case in kat["partition_output_errors"]:
        with pytest.raises(ValueError):
            port.partition_output(case["total"], case["workers"], case["r"])


def test_kat_plan_and_merge_parallel(port, kat):
    for case in kat["plan"]:
        a, b = arr(case["a"], np.uint64), arr(case["b"], np.uint64)
        w = case["workers"]
        total = len(a) + len(b)
        blocks = []
        for r in range(w):
            lo, hi = port.partition_output(total, w, r), port.partition_output(total, w, r + 1)
            (ja, ka), (jb, kb) = port.co_rank(lo, a, b), port.co_rank(hi, a, b)
            blocks.append([r, lo, hi, ja, jb, ka, kb])
        assert blocks == case["expect"], case["src"]
    for case in kat["merge_parallel"]:
        a, b = arr(case["a"], np.uint64), arr(case["b"], np.uint64)
        out, _, bs, _ = port.merge_parallel(a, b, case["workers"])
        assert out.tolist() == case["expect"], case["src"]
        if "block_sizes" in case:
            assert bs.tolist() == case["block_sizes"], case["src"]


# ------------------------------------------------- reference-made vectors

def _cases(golden, prefix):
    keys = sorted({k.rsplit("__", 1)[0] for k in golden if k.startswith(prefix + "__")})
    return [(k, {f.rsplit("__", 1)[1]: golden[f] for f in golden if f.startswith(k + "__")})
            for k in keys]


def test_golden_co_rank(port, golden):
    cases = _cases(golden, "corank")
    assert len(cases) == 18
    for name, c in cases:
        a, b = c["a"], c["b"]
        for i in range(len(a) + len(b) + 1):
            (j, _), (it, cmp) = port.co_rank(i, a, b, stats=True)
            assert (j, it, cmp) == (int(c["j"][i]), int(c["it"][i]), int(c["cmp"][i])), (name, i)


def test_golden_merge_parallel(port, golden):
    cases = _cases(golden, "merge")
    assert len(cases) == 27
    for name, c in cases:
        out, _, bs, its = port.merge_parallel(c["a"], c["b"], 7)
        assert out.dtype == c["out"].dtype and np.array_equal(out, c["out"]), name
        assert np.array_equal(bs, c["bs7"]) and np.array_equal(its, c["it7"]), name
        for w in (1, 3, 16):
            assert np.array_equal(port.merge_parallel(c["a"], c["b"], w, threads=2)[0],
                                  c["out"]), (name, w)


def test_golden_key_value(port, golden):
    cases = _cases(golden, "kv")
    assert len(cases) == 15
    for name, c in cases:
        a, b = c["a"], c["b"]
        av = np.arange(len(a), dtype=np.uint32)
        bv = np.arange(len(b), dtype=np.uint32) | np.uint32(1 << 31)
        out, outv, _, _ = port.merge_parallel(a, b, 5, av, bv)
        assert np.array_equal(out, c["outk"]) and np.array_equal(outv, c["outv"]), name


def test_golden_segmented(port, golden):
    cases = _cases(golden, "seg")
    assert len(cases) == 6
    for name, c in cases:
        out = port.merge_segmented(c["a"], c["aoff"], c["b"], c["boff"], threads=3)
        assert np.array_equal(out, c["out"]), name


def test_golden_generator_recipe(port, golden):
    # uniform (dist 0: next()) and few-distinct (dist 2: below(param)) pin
    # stream(seed, lane) + below() + sort of generate.cpp:17-29.
    for dist, width in ((0, 0), (2, 16)):
        seed = int(golden[f"gen__{dist}__seed"][0])
        a, b = golden[f"gen__{dist}__a"], golden[f"gen__{dist}__b"]
        assert np.array_equal(port.generate_sorted(np.uint64, seed, 0, len(a), width), a)
        assert np.array_equal(port.generate_sorted(np.uint64, seed, 1, len(b), width), b)


def test_golden_checksum(port, golden):
    assert port.checksum(golden["checksum__keys"]) == int(golden["checksum__value"][0])


def test_golden_plan(port, golden):
    for name, c in _cases(golden, "plan"):
        a, b, blocks = c["a"], c["b"], c["blocks"]
        w = len(blocks)
        total = len(a) + len(b)
        for r in range(w):
            lo, hi = port.partition_output(total, w, r), port.partition_output(total, w, r + 1)
            ja, jb = port.co_rank(lo, a, b)[0], port.co_rank(hi, a, b)[0]
            assert [r, lo, hi, ja, jb, lo - ja, hi - jb] == blocks[r].tolist(), name


# -------------------------------------------- properties (reference tests)

def brute_force(i, a, b):
    """testutil::brute_force_co_ranks (tests/oracles.hpp:23-37)."""
    m, n = len(a), len(b)
    found = []
    for j in range(max(0, i - n), min(i, m) + 1):
        k = i - j
        first = j == 0 or k == n or not (b[k] < a[j - 1])
        second = k == 0 or j == m or b[k - 1] < a[j]
        if first and second:
            found.append((j, k))
    return found


def ceil_log2(x):
    return 0 if x <= 1 else int(x - 1).bit_length()


def test_exhaustive_uniqueness_and_bound(port):
    """Acceptance criterion 1 + corrected bound (acceptance_test.cpp:56-159)."""
    rng = np.random.default_rng(10101)
    for m, n in itertools.product(range(0, 13), range(0, 13)):
        a = np.sort(rng.integers(0, 3, m)).astype(np.uint64)
        b = np.sort(rng.integers(0, 3, n)).astype(np.uint64)
        for i in range(m + n + 1):
            sat = brute_force(i, a, b)
            assert len(sat) == 1
            (j, k), (it, cmp) = port.co_rank(i, a, b, stats=True)
            assert (j, k) == sat[0]
            bound = ceil_log2(max(1, min(m, n, i, m + n - i))) + 1
            assert it <= bound and cmp <= 2 * bound


@pytest.mark.skipif(not available_ref(), reason="oracle/_ref not built")
def test_port_equals_reference_live(port):
    from oracle.py import Ref
    ref = Ref()
    rng = np.random.default_rng(34)
    for round_ in range(120):
        dt = [np.int32, np.uint32, np.uint64][round_ % 3]
        m, n = int(rng.integers(0, 400)), int(rng.integers(0, 400))
        alphabet = [4, 0, 1, 50][round_ % 4]
        def draw(sz):
            if alphabet == 0:
                v = rng.integers(0, 2**31, sz)
            else:
                v = rng.integers(0, alphabet, sz) - (alphabet // 2 if dt == np.int32 else 0)
            return np.sort(v.astype(dt))
        a, b = draw(m), draw(n)
        for i in rng.integers(0, m + n + 1, 10):
            assert port.co_rank(int(i), a, b, stats=True) == ref.co_rank(int(i), a, b, stats=True)
        for w in (1, 2, 3, 4, 7, 16):
            o1, _, bs1, it1 = port.merge_parallel(a, b, w)
            o2, _, bs2, it2 = ref.merge_parallel(a, b, w, simulated=True)
            assert np.array_equal(o1, o2) and np.array_equal(bs1, bs2) and np.array_equal(it1, it2)


@pytest.mark.skipif(not available_ref(), reason="oracle/_ref not built")
def test_reference_errors_match_port(port):
    from oracle.py import Ref
    ref = Ref()
    a, b = np.array([1, 2], np.uint64), np.array([3], np.uint64)
    with pytest.raises(IndexError, match="rank out of range"):
        ref.co_rank(4, a, b)
    with pytest.raises(ValueError, match="output length must equal"):
        ref.merge_parallel(a, b, 2, out=np.zeros(2, np.uint64))
    with pytest.raises(ValueError, match="worker count must be positive"):
        ref.merge_parallel(a, b, 0)


def test_oracle_merge_sort_is_stable_sort(port):
    """oracle_merge_sort (the GPU sort's checker) equals numpy's stable sort."""
    rng = np.random.default_rng(2)
    for dt in (np.int32, np.uint32, np.uint64):
        for n in (0, 1, 2, 3, 31, 1000, 4097):
            k = rng.integers(0, 40, n).astype(dt)
            assert np.array_equal(port.merge_sort(k), np.sort(k, kind="stable"))


def test_oracle_comparison_counts_match_reference(port, golden):
    """merge_options::count_comparisons totals (reference, tests/golden, section 8)."""
    ws = [int(x) for x in golden["cmp__workers"]]
    for name in ("i32", "u32", "u64"):
        for c in range(8):
            a, b = golden[f"cmp__{name}__{c}__a"], golden[f"cmp__{name}__{c}__b"]
            counts = golden[f"cmp__{name}__{c}__counts"]
            for wi, w in enumerate(ws):
                for synced in (0, 1):
                    _, _, total = port.merge_report(a, b, w, bool(synced))
                    assert total == int(counts[wi, synced]), (name, c, w, synced)


def test_oracle_merge_sort_pairs_is_stable(port):
    rng = np.random.default_rng(3)
    for dt in (np.int32, np.uint64):
        for n in (0, 1, 7, 1000, 4097):
            k = rng.integers(0, 9, n).astype(dt)
            v = np.arange(n, dtype=np.uint32)
            ok, ov = port.merge_sort_pairs(k, v)
            idx = np.argsort(k, kind="stable")
            assert np.array_equal(ok, k[idx]) and np.array_equal(ov, v[idx])
