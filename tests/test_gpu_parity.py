"""GPU parity: the sm_100a path (through the C ABI) against the reference.

Every check is bit-exact (integer work):
  * the reference's KATs (tests/golden/kat.json),
  * vectors produced by the unmodified reference (tests/golden/ref_vectors.npz),
  * seeded random sweeps against the C oracle (oracle/comerge_oracle.c) over
    ragged / empty / tile-boundary / misaligned shapes and duplicate-heavy keys,
  * the five BASELINE configs at full size: exact comparison with the oracle
    where the host finishes in seconds, and size-independent properties
    (sortedness, multiset checksum, tagged stability) everywhere.
"""
import numpy as np
import pytest

from conftest import KEY_DTYPES

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

TDT = {np.dtype(np.int32): torch.int32, np.dtype(np.uint32): torch.uint32,
       np.dtype(np.uint64): torch.uint64}


def dev(x, cuda):
    return torch.from_numpy(np.ascontiguousarray(x)).to(cuda)


def host(t):
    return t.cpu().numpy()


def P():
    import paper_1303_4312_b200 as mod
    return mod


@pytest.fixture(params=["tile", "pipe", "small"])
def path(request):
    """Run a test through each device kernel (v1 tile, the tile pipeline, the small-merge kernel)."""
    P().set_kernel_path(request.param)
    yield request.param
    P().set_kernel_path("auto")


def tagged(m, n):
    return (np.arange(m, dtype=np.uint32),
            np.arange(n, dtype=np.uint32) | np.uint32(1 << 31))


# ------------------------------------------------------------------ KATs

def test_kat_co_rank(cuda, kat):
    from test_oracle import kinds_for
    for case in kat["co_rank"]:
        for k in kinds_for(case["a"] + case["b"]):
            dt = KEY_DTYPES[k]
            a, b = dev(np.array(case["a"], dt), cuda), dev(np.array(case["b"], dt), cuda)
            st = P().CoRankStats()
            assert list(P().co_rank(case["i"], a, b, st)) == case["expect"], case["src"]
            if "iterations" in case:
                assert st.iterations == case["iterations"]
            if "comparisons" in case:
                assert st.comparisons == case["comparisons"]
            if "max_comparisons" in case:
                assert st.comparisons <= case["max_comparisons"]
    for case in kat["co_rank_errors"]:
        a = dev(np.array(case["a"], np.uint64), cuda)
        b = dev(np.array(case["b"], np.uint64), cuda)
        with pytest.raises(IndexError, match=case["message"]):
            P().co_rank(case["i"], a, b)


def test_kat_merge(cuda, kat):
    from test_oracle import kinds_for
    for case in kat["merge"]:
        for k in kinds_for(case["a"] + case["b"]):
            dt = KEY_DTYPES[k]
            out = P().stable_merge(dev(np.array(case["a"], dt), cuda),
                                   dev(np.array(case["b"], dt), cuda))
            torch.cuda.synchronize()
            assert host(out).tolist() == case["expect"], case["src"]
    for case in kat["merge_tagged"]:
        for k in ("i32", "u32", "u64"):
            dt = KEY_DTYPES[k]
            av, bv = tagged(len(case["a"]), len(case["b"]))
            _, vals = P().merge_pairs(dev(np.array(case["a"], dt), cuda), dev(av, cuda),
                                      dev(np.array(case["b"], dt), cuda), dev(bv, cuda))
            vals = host(vals)
            assert [int(v >> 31) for v in vals] == case["expect_origin"], case["src"]
            assert [int(v & 0x7FFFFFFF) for v in vals] == case["expect_index"], case["src"]
    for case in kat["merge_errors"]:
        a = dev(np.array(case["a"], np.uint64), cuda)
        b = dev(np.array(case["b"], np.uint64), cuda)
        with pytest.raises(ValueError, match=case["message"]):
            P().stable_merge(a, b, torch.zeros(case["out_len"], dtype=torch.uint64, device=cuda))


def test_kat_plan_and_merge_parallel(cuda, kat):
    for case in kat["plan"]:
        a = dev(np.array(case["a"], np.uint64), cuda)
        b = dev(np.array(case["b"], np.uint64), cuda)
        got = [list(x.as_tuple()) for x in P().plan(a, b, case["workers"])]
        assert got == case["expect"], case["src"]
    for case in kat["merge_parallel"]:
        a, b = np.array(case["a"], np.uint64), np.array(case["b"], np.uint64)
        out = np.zeros(len(a) + len(b), np.uint64)
        rep = P().merge_parallel(a, b, out, case["workers"])
        assert out.tolist() == case["expect"], case["src"]
        if "block_sizes" in case:
            assert rep.block_sizes == case["block_sizes"]
    for case in kat["merge_parallel_errors"]:
        a, b = np.array(case["a"], np.uint64), np.array(case["b"], np.uint64)
        with pytest.raises(ValueError, match=case["message"]):
            P().merge_parallel(a, b, np.zeros(case["out_len"], np.uint64), case["workers"])


# ------------------------------------------------- reference-made vectors

def _cases(golden, prefix):
    from test_oracle import _cases as c
    return c(golden, prefix)


def test_golden_co_rank_batch_exact_stats(cuda, golden):
    """Device Algorithm 1 reproduces the reference's j, iterations and comparisons."""
    for name, c in _cases(golden, "corank"):
        a, b = dev(c["a"], cuda), dev(c["b"], cuda)
        ranks = torch.arange(len(c["a"]) + len(c["b"]) + 1, device=cuda).to(torch.uint64)
        j, it, cmp = P().co_rank_batch(ranks, a, b, with_stats=True)
        assert np.array_equal(host(j), c["j"]), name
        assert np.array_equal(host(it), c["it"]), name
        assert np.array_equal(host(cmp), c["cmp"]), name


def test_golden_merges_device_and_host_paths(cuda, path, golden):
    for name, c in _cases(golden, "merge"):
        out = P().stable_merge(dev(c["a"], cuda), dev(c["b"], cuda))
        torch.cuda.synchronize()
        assert np.array_equal(host(out), c["out"]), name
        hout = np.full(len(c["out"]), 0x5A, dtype=c["out"].dtype)  # poisoned output
        rep = P().merge_parallel(c["a"], c["b"], hout, 7)
        assert np.array_equal(hout, c["out"]), name
        assert rep.block_sizes == c["bs7"].tolist(), name
        assert rep.corank_iterations == c["it7"].tolist(), name
        rep_s = P().merge_parallel_synced(c["a"], c["b"], hout, 7)
        assert np.array_equal(hout, c["out"]) and len(rep_s.corank_iterations) == 7


def test_golden_key_value(cuda, path, golden):
    for name, c in _cases(golden, "kv"):
        av, bv = tagged(len(c["a"]), len(c["b"]))
        ok, ov = P().merge_pairs(dev(c["a"], cuda), dev(av, cuda), dev(c["b"], cuda), dev(bv, cuda))
        torch.cuda.synchronize()
        assert np.array_equal(host(ok), c["outk"]) and np.array_equal(host(ov), c["outv"]), name
        hk = np.empty_like(c["outk"])
        hv = np.empty_like(c["outv"])
        P().merge_pairs(c["a"], av, c["b"], bv, hk, hv)  # host buffers through the C ABI
        assert np.array_equal(hk, c["outk"]) and np.array_equal(hv, c["outv"]), name


def test_golden_segmented(cuda, path, golden):
    for name, c in _cases(golden, "seg"):
        out = P().merge_segmented(dev(c["a"], cuda), dev(c["aoff"], cuda), dev(c["b"], cuda),
                                  dev(c["boff"], cuda))
        torch.cuda.synchronize()
        assert np.array_equal(host(out), c["out"]), name


def test_golden_plan(cuda, golden):
    for name, c in _cases(golden, "plan"):
        got = [list(x.as_tuple()) for x in P().plan(dev(c["a"], cuda), dev(c["b"], cuda),
                                                    len(c["blocks"]))]
        assert got == c["blocks"].tolist(), name


# ------------------------------------------------------ random sweeps

def _draw(rng, dt, size, alphabet):
    if alphabet == 0:
        hi = 2**64 if dt == np.uint64 else 2**31
        v = rng.integers(0, hi, size, dtype=np.uint64 if dt == np.uint64 else np.int64)
        if dt == np.int32:
            v = v - 2**30
    else:
        v = rng.integers(0, alphabet, size) - (alphabet // 2 if dt == np.int32 else 0)
    return np.sort(v.astype(dt))


# tile sizes of the pipeline (keys-only) and tile kernels: shapes straddle both
TILES = {np.int32: 256 * 31, np.uint32: 256 * 31, np.uint64: 256 * 15}
PAIR_TILES = {np.int32: 256 * 15, np.uint32: 256 * 15, np.uint64: 256 * 11}


@pytest.mark.parametrize("dt", [np.int32, np.uint32, np.uint64])
def test_random_sweep_keys_and_pairs(cuda, path, port, dt):
    rng = np.random.default_rng(int(np.dtype(dt).itemsize) * 7 + (dt == np.int32))
    T = TILES[dt]
    shapes = [(0, 0), (0, 1), (1, 0), (T - 1, 0), (0, T + 1), (T, T), (T - 1, 1), (1, T - 1),
              (2 * T + 3, 5), (5, 3 * T - 2), (3, 50000), (50000, 3), (70001, 69999)]
    T2 = PAIR_TILES[dt]  # the key-value tile
    shapes += [(T2 - 1, 0), (0, T2 + 1), (T2, T2), (T2 - 1, 1), (2 * T2 + 3, 5), (5, 3 * T2 - 2)]
    shapes += [(int(rng.integers(0, 20000)), int(rng.integers(0, 20000))) for _ in range(12)]
    for idx, (m, n) in enumerate(shapes):
        alphabet = [0, 1, 2, 16, 1000][idx % 5]
        a, b = _draw(rng, dt, m, alphabet), _draw(rng, dt, n, alphabet)
        expect = port.merge(a, b)
        out = P().stable_merge(dev(a, cuda), dev(b, cuda))
        torch.cuda.synchronize()
        assert np.array_equal(host(out), expect), (m, n, alphabet)
        av, bv = tagged(m, n)
        ek, ev = port.merge(a, b, av, bv)
        ok, ov = P().merge_pairs(dev(a, cuda), dev(av, cuda), dev(b, cuda), dev(bv, cuda))
        torch.cuda.synchronize()
        assert np.array_equal(host(ok), ek) and np.array_equal(host(ov), ev), (m, n, alphabet)


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_misaligned_views(cuda, path, port, dt):
    """Inputs / outputs that are not 16-byte aligned take the scalar edges."""
    rng = np.random.default_rng(5)
    for shift_a, shift_b, shift_o in [(1, 0, 0), (0, 3, 1), (2, 1, 3), (3, 3, 2)]:
        m, n = 9001 + shift_a, 7777 + shift_b
        a, b = _draw(rng, dt, m, 64), _draw(rng, dt, n, 64)
        ta = torch.zeros(m + 8, dtype=TDT[np.dtype(dt)], device=cuda)
        tb = torch.zeros(n + 8, dtype=TDT[np.dtype(dt)], device=cuda)
        to = torch.zeros(m + n + 8, dtype=TDT[np.dtype(dt)], device=cuda)
        va, vb = ta[shift_a:shift_a + m], tb[shift_b:shift_b + n]
        va.copy_(dev(a, cuda))
        vb.copy_(dev(b, cuda))
        vo = to[shift_o:shift_o + m + n]
        P().stable_merge(va, vb, vo)
        torch.cuda.synchronize()
        assert np.array_equal(host(vo), port.merge(a, b)), (shift_a, shift_b, shift_o)


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_misaligned_pairs_and_segmented_pipeline(cuda, port, dt):
    """The tile pipeline at every element offset mod 16 bytes of keys,
    payloads and outputs (byte-space windows and stores: no alignment cliff),
    large enough for the persistent grid and its dynamic tail."""
    rng = np.random.default_rng(8)
    tdt = TDT[np.dtype(dt)]
    vece = 16 // np.dtype(dt).itemsize
    m, n = 300_001, 250_003
    a, b = _draw(rng, dt, m, 20), _draw(rng, dt, n, 20)
    av, bv = tagged(m, n)
    ek, ev = port.merge(a, b, av, bv)

    def view(x, t, shift):
        buf = torch.zeros(len(x) + 8, dtype=t, device=cuda)
        v = buf[shift:shift + len(x)]
        v.copy_(dev(x, cuda))
        return v

    P().set_kernel_path("pipe")
    for sh in [(1, 0, 0, 0, 0, 0), (0, 1, 2, 3, 1, 2), (vece - 1, 1, 0, 1, 3, 1),
               (1, vece - 1, 3, 0, 2, 3), (0, 0, 0, 0, 0, 1)]:
        va, vb = view(a, tdt, sh[0] % vece), view(b, tdt, sh[1] % vece)
        vav, vbv = view(av, torch.uint32, sh[2]), view(bv, torch.uint32, sh[3])
        ok = torch.zeros(m + n + 8, dtype=tdt, device=cuda)[sh[4] % vece:][:m + n]
        ov = torch.zeros(m + n + 8, dtype=torch.uint32, device=cuda)[sh[5]:][:m + n]
        P().merge_pairs(va, vav, vb, vbv, ok, ov)
        P().stable_merge(va, vb, ok2 := torch.zeros(m + n + 3, dtype=tdt, device=cuda)[3 % vece:][:m + n])
        torch.cuda.synchronize()
        assert P()._native.lib.comerge_cuda_last_path() == 3
        assert np.array_equal(host(ok), ek) and np.array_equal(host(ov), ev), sh
        assert np.array_equal(host(ok2), ek), sh
    P().set_kernel_path("auto")
    if dt == np.int32:  # segmented batch, misaligned runs and output
        la, lb = rng.integers(0, 3000, 500), rng.integers(0, 3000, 500)
        sa = np.concatenate([np.sort(rng.integers(0, 99, x)) for x in la]).astype(np.int32)
        sb = np.concatenate([np.sort(rng.integers(0, 99, x)) for x in lb]).astype(np.int32)
        ao = np.concatenate([[0], np.cumsum(la)]).astype(np.uint64)
        bo = np.concatenate([[0], np.cumsum(lb)]).astype(np.uint64)
        expect = port.merge_segmented(sa, ao, sb, bo)
        for s0, s1, s2 in [(1, 2, 3), (3, 0, 1), (0, 0, 2)]:
            out = torch.zeros(len(sa) + len(sb) + 4, dtype=torch.int32, device=cuda)[s2:]
            out = out[:len(sa) + len(sb)]
            P().merge_segmented(view(sa, torch.int32, s0), dev(ao, cuda), view(sb, torch.int32, s1),
                                dev(bo, cuda), out)
            torch.cuda.synchronize()
            assert P()._native.lib.comerge_cuda_last_path() == 5
            assert np.array_equal(host(out), expect), (s0, s1, s2)


def _seg_batch(rng, nseg, lo, hi, alphabet, empty_every=0):
    la, lb = rng.integers(lo, hi + 1, nseg), rng.integers(lo, hi + 1, nseg)
    if empty_every:
        la[::empty_every] = 0
        lb[1::empty_every] = 0
    sa = np.concatenate([np.sort(rng.integers(0, alphabet, x)) for x in la] +
                        [np.zeros(0, np.int64)]).astype(np.int32)
    sb = np.concatenate([np.sort(rng.integers(0, alphabet, x)) for x in lb] +
                        [np.zeros(0, np.int64)]).astype(np.int32)
    ao = np.concatenate([[0], np.cumsum(la)]).astype(np.uint64)
    bo = np.concatenate([[0], np.cumsum(lb)]).astype(np.uint64)
    return sa, ao, sb, bo


def test_segmented_host_buffers(cuda, port):
    """Host segmented batches (comerge_merge_segmented_host_*): >= 2^20
    elements through the chunked H2D / merge / D2H pipeline (cuts co-ranked
    in (segment, key) order, chunk segments rebased on the device), smaller
    ones staged; pageable and pinned buffers; bit-exact vs the oracle."""
    rng = np.random.default_rng(31)
    cases = [_seg_batch(rng, 2000, 1, 4096, 1 << 20),          # C5 shape, 8 M elements
             _seg_batch(rng, 60000, 0, 40, 50, empty_every=7),  # tiny pairs, empty ones
             _seg_batch(rng, 1, 1_500_000, 1_500_000, 1000),    # one huge pair
             _seg_batch(rng, 3, 400_000, 700_000, 3),           # few pairs, heavy ties
             _seg_batch(rng, 300, 0, 2000, 100)]                # small: staged
    for sa, ao, sb, bo in cases:
        expect = port.merge_segmented(sa, ao, sb, bo)
        out, rep = P().merge_segmented(sa, ao, sb, bo, report=True)
        assert np.array_equal(out, expect), (len(sa), len(ao))
        total = len(sa) + len(sb)
        assert rep.h2d_bytes >= total * 4 and rep.d2h_bytes == total * 4
    # pinned buffers (page-locked host memory)
    sa, ao, sb, bo = cases[0]
    pa = torch.from_numpy(sa).pin_memory().numpy()
    pb = torch.from_numpy(sb).pin_memory().numpy()
    po = torch.empty(len(sa) + len(sb), dtype=torch.int32).pin_memory().numpy()
    P().merge_segmented(pa, ao, pb, bo, out=po)
    assert np.array_equal(po, port.merge_segmented(sa, ao, sb, bo))
    # contract
    with pytest.raises(ValueError, match="nondecreasing"):
        P().merge_segmented(sa, ao[::-1].copy(), sb, bo)
    bad = ao.copy()
    bad[0] = 1
    with pytest.raises(ValueError, match="start at 0"):
        P().merge_segmented(sa, bad, sb, bo)


def test_random_segmented(cuda, path, port):
    rng = np.random.default_rng(99)
    for dt in (np.int32, np.uint32):
        for nseg, maxlen in [(1, 10000), (3000, 8), (500, 600), (64, 4096), (7, 30000)]:
            ma = rng.integers(0, maxlen + 1, nseg)
            nb = rng.integers(0, maxlen + 1, nseg)
            ma[rng.integers(0, nseg, nseg // 4)] = 0
            nb[rng.integers(0, nseg, nseg // 5)] = 0
            both = rng.integers(0, nseg, nseg // 10)
            ma[both] = 0
            nb[both] = 0
            a = np.concatenate([_draw(rng, dt, int(x), 100) for x in ma] + [np.empty(0, dt)])
            b = np.concatenate([_draw(rng, dt, int(x), 100) for x in nb] + [np.empty(0, dt)])
            ao = np.concatenate([[0], np.cumsum(ma)]).astype(np.uint64)
            bo = np.concatenate([[0], np.cumsum(nb)]).astype(np.uint64)
            out = P().merge_segmented(dev(a, cuda), dev(ao, cuda), dev(b, cuda), dev(bo, cuda))
            torch.cuda.synchronize()
            assert np.array_equal(host(out), port.merge_segmented(a, ao, b, bo)), (nseg, maxlen)


def test_segmented_short_segments_inside_long(cuda, path, port):
    """Tiles of few segments where some threads' outputs still cross one, two
    or many segment ends (clusters of 0-6 element pairs between long pairs):
    the consumers' lean loop, its one-switch form and the rolled fallback."""
    rng = np.random.default_rng(4242)
    for dt in (np.int32, np.uint32):
        ma, nb = [], []
        for _ in range(60):
            ma.append(int(rng.integers(1000, 9000)))
            nb.append(int(rng.integers(0, 9000)))
            for _ in range(int(rng.integers(0, 12))):
                ma.append(int(rng.integers(0, 4)))
                nb.append(int(rng.integers(0, 4)))
        ma, nb = np.array(ma), np.array(nb)
        a = np.concatenate([_draw(rng, dt, int(x), 50) for x in ma])
        b = np.concatenate([_draw(rng, dt, int(x), 50) for x in nb])
        ao = np.concatenate([[0], np.cumsum(ma)]).astype(np.uint64)
        bo = np.concatenate([[0], np.cumsum(nb)]).astype(np.uint64)
        out = P().merge_segmented(dev(a, cuda), dev(ao, cuda), dev(b, cuda), dev(bo, cuda))
        torch.cuda.synchronize()
        assert np.array_equal(host(out), port.merge_segmented(a, ao, b, bo)), dt


def test_co_rank_split_equals_reference_search(cuda, path, port):
    """The partition's one-sided search returns Algorithm 1's split (Lemma 1)."""
    rng = np.random.default_rng(3)
    for dt in (np.int32, np.uint64):
        a, b = _draw(rng, dt, 100000, 7), _draw(rng, dt, 80000, 7)
        ranks = np.unique(rng.integers(0, 180001, 2000)).astype(np.uint64)
        j = host(P().co_rank_batch(dev(ranks, cuda), dev(a, cuda), dev(b, cuda)))
        for i, jj in zip(ranks[:200], j[:200]):
            assert port.co_rank(int(i), a, b)[0] == int(jj)
        out = host(P().stable_merge(dev(a, cuda), dev(b, cuda)))
        assert np.array_equal(out, port.merge(a, b))


def test_worker_count_independence(cuda, path, port):
    """Acceptance criterion 6 at GPU scale: outputs identical for any p."""
    rng = np.random.default_rng(2026)
    a, b = _draw(rng, np.uint64, 300000, 0), _draw(rng, np.uint64, 300000, 0)
    expect = port.merge(a, b)
    for p in (1, 2, 4, 8, 33):
        out = np.zeros(600000, np.uint64)
        rep = P().merge_parallel(a, b, out, p)
        assert np.array_equal(out, expect) and len(rep.block_sizes) == p
        assert max(rep.block_sizes) - min(rep.block_sizes) <= 1


# ------------------------------------------------------ generator pin

def test_gpu_generator_matches_reference_recipe(cuda, port, golden):
    from paper_1303_4312_b200 import testkit as tk
    for dist, width in ((0, 0), (2, 16)):
        seed = int(golden[f"gen__{dist}__seed"][0])
        a = golden[f"gen__{dist}__a"]
        got = tk.generate_sorted(torch.uint64, seed, 0, len(a), width)
        assert np.array_equal(host(got), a)
    for dt, width in ((torch.int32, 2**31), (torch.int32, 16), (torch.uint32, 2**20),
                      (torch.uint64, 0), (torch.uint64, 3 * 2**62)):
        for seed, length in ((5, 1), (5, 1000), (77, 123457)):
            got = tk.generate_sorted(dt, seed, 1, length, width)
            npdt = {torch.int32: np.int32, torch.uint32: np.uint32, torch.uint64: np.uint64}[dt]
            assert np.array_equal(host(got), port.generate_sorted(npdt, seed, 1, length, width))


# ------------------------------------------- BASELINE configs, full size

def _config_inputs(cfg, cuda):
    import bench
    return bench.make_inputs(cfg, seed=5, device=cuda)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C3s", "C4", "C5"])
def test_baseline_config_full_size(cuda, port, cfg):
    """Every BASELINE config at full size, byte-for-byte against the REFERENCE
    itself (oracle/_ref: comerge::merge_parallel at hardware_concurrency
    workers, parallel.hpp:304-317; key-value configs in its own call shape,
    {key, val} structs with a key-only less, oracle.hpp:22-37; C5 as
    comerge::stable_merge per pair, merge.hpp:52-68), plus the size-independent
    properties as extra guards."""
    from oracle.py import Ref, available_ref, to_aos
    assert available_ref(), "oracle/_ref/libcomerge_ref.so (the compiled reference) is missing"
    ref = Ref()
    threads = ref.hardware_concurrency()
    P().set_kernel_path("auto")
    import bench
    from paper_1303_4312_b200 import testkit as tk
    inp = _config_inputs(cfg, cuda)
    out = bench.run_config(cfg, inp)
    torch.cuda.synchronize()
    a, b = inp["a"], inp["b"]
    # size-independent properties (C5 is sorted per pair only)
    if cfg != "C5":
        assert tk.count_unsorted(out["keys"]) == 0
    assert tk.checksum(out["keys"]) == (tk.checksum(a) + tk.checksum(b)) % 2**64
    if "vals" in out:
        assert tk.verify_pairs(a, b, out["keys"], out["vals"]) == [0, 0, 0, 0]
    # the reference's own output on the same inputs, compared byte for byte
    ha, hb = host(a), host(b)
    got = host(out["keys"])
    if cfg == "C5":
        expect, _ = ref.merge_segmented(ha, host(inp["a_off"]), hb, host(inp["b_off"]),
                                        threads=threads)
        assert got.tobytes() == expect.tobytes()
    elif "vals" in out:
        a_aos, b_aos = to_aos(ha, host(inp["av"])), to_aos(hb, host(inp["bv"]))
        del ha, hb
        expect, rep = ref.merge_parallel_kv(a_aos, b_aos, threads)
        del a_aos, b_aos
        assert rep.m + rep.n == len(got)
        assert got.tobytes() == np.ascontiguousarray(expect["key"]).tobytes()
        assert host(out["vals"]).tobytes() == np.ascontiguousarray(expect["val"]).tobytes()
    else:
        expect, rep, _, _ = ref.merge_parallel(ha, hb, threads)
        assert got.tobytes() == expect.tobytes()


def test_host_buffers_pipelined(cuda, port):
    """Host inputs >= 1M elements take the chunked H2D/merge/D2H pipeline
    (host co-ranks of the chunk boundaries); pinned and pageable buffers."""
    rng = np.random.default_rng(77)
    for dt, (m, n), alphabet in [(np.int32, (1_500_000, 2_100_000), 1000),
                                 (np.uint64, (3_000_001, 17), 0), (np.int32, (2_000_000, 0), 5)]:
        a, b = _draw(rng, dt, m, alphabet), _draw(rng, dt, n, alphabet)
        expect = port.merge(a, b)
        out = np.zeros(m + n, dt)
        rep = P().merge_parallel(a, b, out, 7)
        assert np.array_equal(out, expect)
        assert rep.h2d_bytes == (m + n) * out.itemsize and rep.d2h_bytes == (m + n) * out.itemsize
        ra = P().merge_parallel(a, b, out, 7)  # repeatable
        assert np.array_equal(out, expect) and ra.block_sizes == rep.block_sizes
        # pinned host memory
        tdt = TDT[np.dtype(dt)]
        pa = torch.from_numpy(a).pin_memory()
        pb = torch.from_numpy(b).pin_memory()
        po = torch.zeros(m + n, dtype=tdt).pin_memory()
        P().merge_parallel(pa.numpy(), pb.numpy(), po.numpy(), 3)
        assert np.array_equal(po.numpy(), expect)
        from paper_1303_4312_b200 import _native as N
        for mode in (1, 2):  # zero-copy, plain staging
            N.lib.comerge_cuda_set_host_mode(mode)
            try:
                po.zero_()
                P().merge_parallel(pa.numpy(), pb.numpy(), po.numpy(), 3)
                assert np.array_equal(po.numpy(), expect), mode
            finally:
                N.lib.comerge_cuda_set_host_mode(0)
        av, bv = tagged(m, n)
        ek, ev = port.merge(a, b, av, bv)
        ok, ov = np.empty_like(ek), np.empty_like(ev)
        P().merge_pairs(a, av, b, bv, ok, ov)
        assert np.array_equal(ok, ek) and np.array_equal(ov, ev)
        # mixed page-locked and pageable arrays: only the pageable ones go
        # through the page-locked staging slots
        pav = torch.from_numpy(av).pin_memory()
        pbv = torch.from_numpy(bv).pin_memory()
        pov = torch.zeros(m + n, dtype=torch.uint32).pin_memory()
        ok2 = np.zeros_like(ek)
        P().merge_pairs(pa.numpy(), av, b, pbv.numpy(), ok2, pov.numpy())
        assert np.array_equal(ok2, ek) and np.array_equal(pov.numpy(), ev)
        po.zero_()
        ov2 = np.zeros_like(ev)
        P().merge_pairs(a, pav.numpy(), pb.numpy(), bv, po.numpy(), ov2)
        assert np.array_equal(po.numpy(), ek) and np.array_equal(ov2, ev)


def test_host_pipeline_aligned_windows(cuda, port):
    """The host pipeline copies 256-byte aligned supersets of each chunk's
    windows and merges the chunk as an output range: chunk boundaries in the
    middle of duplicate runs, empty windows, skewed sides, 64-bit keys with
    payloads, and host arrays that are not 256-byte aligned (offset views)."""
    rng = np.random.default_rng(2024)
    cases = [(np.int32, 2_500_003, 1_700_001, 3), (np.int32, 4_000_000, 9, 0),
             (np.int32, 5, 3_000_000, 1 << 20), (np.uint64, 1_100_000, 1_300_007, 2),
             (np.uint64, 2_000_000, 2_000_000, 0)]
    for dt, m, n, alphabet in cases:
        for shift in (0, 1, 3):
            a = _draw(rng, dt, m + shift, alphabet)[shift:]
            b = _draw(rng, dt, n + 1, alphabet)[1:] if shift else _draw(rng, dt, n, alphabet)
            av, bv = tagged(m, n)
            ek, ev = port.merge(a, b, av, bv)
            ok = np.empty(m + n + shift, dt)[shift:]
            ov = np.empty(m + n + 2, np.uint32)[2:] if shift else np.empty(m + n, np.uint32)
            P().merge_pairs(a, av, b, bv, ok, ov)
            assert np.array_equal(ok, ek) and np.array_equal(ov, ev), (dt, m, n, shift)
            out = np.empty(m + n, dt)
            P().merge_parallel(a, b, out, 4)
            assert np.array_equal(out, ek), (dt, m, n, shift)


def test_host_pipeline_report_matches_reference_stats(cuda, port):
    """merge_report.corank_iterations of the host pipeline = Algorithm 1's."""
    rng = np.random.default_rng(5)
    a, b = _draw(rng, np.uint64, 1_200_000, 64), _draw(rng, np.uint64, 900_000, 64)
    out = np.empty(len(a) + len(b), np.uint64)
    rep = P().merge_parallel(a, b, out, 5)
    total = len(a) + len(b)
    bounds = [port.partition_output(total, 5, r) for r in range(6)]
    its = [port.co_rank(i, a, b, stats=True)[1][0] for i in bounds]
    assert rep.corank_iterations == [x for r in range(5) for x in (its[r], its[r + 1])]
    rep_s = P().merge_parallel_synced(a, b, out, 5)
    assert rep_s.corank_iterations == its[:5]


def test_rank_shards_concatenate(cuda, port):
    """Algorithm 2 across ranks (paper_1303_4312_b200.shard): each rank merges
    only its co-ranked windows; the shards concatenate to the full merge."""
    from paper_1303_4312_b200.shard import merge_shard
    rng = np.random.default_rng(8)
    a, b = _draw(rng, np.int32, 300_001, 40), _draw(rng, np.int32, 200_003, 40)
    expect = port.merge(a, b)
    ta, tb = dev(a, cuda), dev(b, cuda)
    for world in (1, 2, 3, 8):
        parts = [merge_shard(ta, tb, r, world)[1] for r in range(world)]
        torch.cuda.synchronize()
        assert np.array_equal(np.concatenate([host(p) for p in parts]), expect), world


# ------------------------------------------------------------ merge sort
# block-sorted runs + merge passes of the pipeline in
# merge-pass mode.  Oracle: oracle_merge_sort (repeated stable_merge of
# adjacent runs, merge.hpp:52-68), bit-exact.

SORT_RUN = {np.dtype(np.int32): 16384, np.dtype(np.uint32): 16384, np.dtype(np.uint64): 8192}


@pytest.mark.parametrize("dt", [np.int32, np.uint32, np.uint64])
def test_sort_sizes_against_oracle(cuda, port, dt):
    R = SORT_RUN[np.dtype(dt)]
    rng = np.random.default_rng(7)
    sizes = [0, 1, 2, 7, R - 1, R, R + 1, 2 * R, 2 * R + 3, 3 * R + 17, 8 * R, 8 * R + 5,
             100_003, 1 << 20]
    for n in sizes:
        for alphabet in (3, 1 << 20, None):
            if alphabet is None:
                info = np.iinfo(dt)
                k = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
            else:
                k = rng.integers(0, alphabet, n).astype(dt)
            got = host(P().sort(dev(k, cuda)))
            assert np.array_equal(got, port.merge_sort(k)), (dt, n, alphabet)


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_sort_presorted_reversed_and_in_place(cuda, port, dt):
    n = 300_001
    rng = np.random.default_rng(3)
    base = np.sort(rng.integers(0, 1 << 30, n).astype(dt))
    for k in (base, base[::-1].copy(), np.full(n, 5, dtype=dt)):
        t = dev(k, cuda)
        P().sort(t, out=t)  # in place
        assert np.array_equal(host(t), port.merge_sort(k))


def test_sort_misaligned_output_and_workspace(cuda, port):
    n = 70_001
    k = np.random.default_rng(5).integers(-1000, 1000, n).astype(np.int32)
    buf = torch.empty(n + 1, dtype=torch.int32, device=cuda)
    out = buf[1:]  # 4-byte offset: the last pass goes through scratch + a copy
    ws = torch.empty(P().sort_workspace_bytes(n, torch.int32), dtype=torch.uint8, device=cuda)
    P().sort(dev(k, cuda), out=out, workspace=ws)
    assert np.array_equal(host(out), port.merge_sort(k))
    with pytest.raises(ValueError):
        P().sort(dev(k, cuda), out=torch.empty(n - 1, dtype=torch.int32, device=cuda))


def test_sort_large_properties(cuda):
    """2^26 int32 keys (the C5 total): sorted, same multiset (size-independent)."""
    from paper_1303_4312_b200 import testkit as tk
    n = 1 << 26
    import paper_1303_4312_b200._native as N
    raw = torch.empty(n, dtype=torch.int64, device=cuda)
    N.check(N.tk().comerge_testkit_generate_raw(11, 0, n, 1 << 31, raw.data_ptr(), None), True)
    keys = raw.to(torch.int32)  # draws below 2^31
    out = P().sort(keys)
    torch.cuda.synchronize()
    assert tk.count_unsorted(out) == 0
    assert tk.checksum(out) == tk.checksum(keys)


# ------------------------------------------- merge report: comparisons
# merge_options::count_comparisons (parallel.hpp:41, :253-280) against the
# reference's own totals (tests/golden section 8) and the oracle's report.

@pytest.mark.parametrize("where", ["host", "device"])
def test_comparison_counts_match_reference(cuda, port, golden, where):
    from paper_1303_4312_b200.comerge import MergeOptions
    ws = [int(x) for x in golden["cmp__workers"]]
    opts = MergeOptions(count_comparisons=True)
    for name in ("i32", "u32", "u64"):
        for c in range(8):
            a, b = golden[f"cmp__{name}__{c}__a"], golden[f"cmp__{name}__{c}__b"]
            counts = golden[f"cmp__{name}__{c}__counts"]
            for wi, w in enumerate(ws):
                for synced in (False, True):
                    if where == "host":
                        aa, bb = a, b
                        out = np.empty(len(a) + len(b), a.dtype)
                    else:
                        aa, bb = dev(a, cuda), dev(b, cuda)
                        out = torch.empty(len(a) + len(b), dtype=TDT[a.dtype], device=cuda)
                    fn = P().merge_parallel_synced if synced else P().merge_parallel
                    rep = fn(aa, bb, out, w, opts=opts)
                    assert rep.comparisons == int(counts[wi, int(synced)]), (name, c, w, synced)
                    bs, its, _ = port.merge_report(a, b, w, synced)
                    assert rep.block_sizes == [int(x) for x in bs[:w]]
                    assert rep.corank_iterations == [int(x) for x in its]
                    got = out if where == "host" else host(out)
                    assert np.array_equal(got, port.merge(a, b))


def test_comparison_counts_large_host_pipeline(cuda, port):
    """The chunked host pipeline (>= 2^20 elements) reports the same counts."""
    from paper_1303_4312_b200.comerge import MergeOptions
    rng = np.random.default_rng(9)
    a = np.sort(rng.integers(0, 64, 700_000).astype(np.int32))
    b = np.sort(rng.integers(0, 64, 600_000).astype(np.int32))
    out = np.empty(len(a) + len(b), np.int32)
    for w, synced in ((1, False), (16, False), (16, True), (1000, True)):
        fn = P().merge_parallel_synced if synced else P().merge_parallel
        rep = fn(a, b, out, w, opts=MergeOptions(count_comparisons=True))
        _, _, total = port.merge_report(a, b, w, synced)
        assert rep.comparisons == total
    assert np.array_equal(out, port.merge(a, b))


@pytest.mark.parametrize("dt", [np.int32, np.uint32, np.uint64])
def test_sort_pairs_stability_against_oracle(cuda, port, dt):
    """Key-value sort: payload = input index, so stability is visible."""
    R = 8192 if np.dtype(dt).itemsize == 4 else 4096
    rng = np.random.default_rng(8)
    for n in (0, 1, 9, R - 1, R, R + 1, 2 * R + 3, 5 * R + 7, 100_003, 1 << 20):
        for alphabet in (2, 1000, None):
            if alphabet is None:
                info = np.iinfo(dt)
                k = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
            else:
                k = rng.integers(0, alphabet, n).astype(dt)
            v = rng.permutation(n).astype(np.uint32)
            ok, ov = P().sort_pairs(dev(k, cuda), dev(v, cuda))
            ek, ev = port.merge_sort_pairs(k, v)
            assert np.array_equal(host(ok), ek) and np.array_equal(host(ov), ev), (dt, n, alphabet)


def test_sort_pairs_in_place_and_misaligned(cuda, port):
    n = 123_457
    rng = np.random.default_rng(10)
    k = rng.integers(0, 50, n).astype(np.int32)
    v = np.arange(n, dtype=np.uint32)
    tk, tv = dev(k, cuda), dev(v, cuda)
    P().sort_pairs(tk, tv, out_keys=tk, out_vals=tv)
    ek, ev = port.merge_sort_pairs(k, v)
    assert np.array_equal(host(tk), ek) and np.array_equal(host(tv), ev)
    bk = torch.empty(n + 1, dtype=torch.int32, device=cuda)
    bv = torch.empty(n + 3, dtype=torch.uint32, device=cuda)
    ok, ov = P().sort_pairs(dev(k, cuda), dev(v, cuda), out_keys=bk[1:], out_vals=bv[3:])
    assert np.array_equal(host(ok), ek) and np.array_equal(host(ov), ev)


# ------------------------------------------- 64-bit sizes (> 2^32 elements)
# The API indexes with size_t (up to 2^40); these runs cross 2^32 in the
# output (and in one input) so every 32-bit truncation would show.  Inputs are
# sorted runs of equal keys made on the device; properties are size-independent
# (sortedness + multiset checksum fix a keys-only merge / sort uniquely; the
# tagged check fixes a key-value merge).

def _free_gb():
    free, _ = torch.cuda.mem_get_info()
    return free / 2**30


def test_max_size_keys_merge_crosses_2_32(cuda):
    from paper_1303_4312_b200 import testkit as tk
    m, n = (1 << 32) + 5, (1 << 31) + 3
    if _free_gb() < 60:
        pytest.skip("needs ~52 GB of device memory")
    a = tk.fill_runs(m, 3, torch.int32)
    b = tk.fill_runs(n, 2, torch.int32, offset=1)
    out = P().stable_merge(a, b)
    torch.cuda.synchronize()
    assert tk.count_unsorted(out) == 0
    assert tk.checksum(out) == (tk.checksum(a) + tk.checksum(b)) % 2**64
    # the boundary at output rank 2^32 + 1: Algorithm 1 on the device agrees with
    # the closed form (A run of 3 equal keys, B run of 2, B offset by 1)
    i = (1 << 32) + 1
    j, k = P().co_rank(i, a, b)
    assert j + k == i and 0 <= j <= m and 0 <= k <= n
    if j > 0 and k < n:
        assert not (int(b[k]) < int(a[j - 1]))
    if k > 0 and j < m:
        assert int(b[k - 1]) < int(a[j])
    del a, b, out
    torch.cuda.empty_cache()


def test_max_size_pairs_merge_crosses_2_32(cuda):
    """A = K runs of 3 equal keys, B = K runs of 5 (same key range), payloads
    = raw input indices: the stable merge is known in closed form -- output
    8k..8k+2 are A's 3k..3k+2, 8k+3..8k+7 are B's 5k..5k+4 -- and is checked
    position by position (in chunks) across 2^32."""
    from paper_1303_4312_b200 import testkit as tk
    K = (1 << 29) + 8
    m, n = 3 * K, 5 * K  # total 8K > 2^32; payload indices < 2^32
    if _free_gb() < 80:
        pytest.skip("needs ~70 GB of device memory")
    a = tk.fill_runs(m, 3, torch.int32)
    b = tk.fill_runs(n, 5, torch.int32)
    av, bv = tk.iota(m, 0), tk.iota(n, 0)
    ok, ov = P().merge_pairs(a, av, b, bv)
    torch.cuda.synchronize()
    del a, b, av, bv
    total = m + n
    step = 1 << 28
    for p0 in range(0, total, step):
        p = torch.arange(p0, min(p0 + step, total), dtype=torch.int64, device=cuda)
        k, r = p // 8, p % 8
        exp_pay = torch.where(r < 3, 3 * k + r, 5 * k + r - 3)
        assert torch.equal(ok[p0:p0 + len(p)].to(torch.int64), k), p0
        got = ov[p0:p0 + len(p)].view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        assert torch.equal(got, exp_pay), p0
    del ok, ov
    torch.cuda.empty_cache()


def test_max_size_sort_crosses_2_32(cuda):
    from paper_1303_4312_b200 import testkit as tk
    n = (1 << 32) + 17
    if _free_gb() < 80:
        pytest.skip("needs ~70 GB of device memory")
    # scrambled keys (a multiplicative hash of the index; the testkit's
    # generator draws at most 2^31 per call)
    keys = torch.empty(n, dtype=torch.int32, device=cuda)
    step = 1 << 28
    for p0 in range(0, n, step):
        p = torch.arange(p0, min(p0 + step, n), dtype=torch.int64, device=cuda)
        keys[p0:p0 + len(p)] = ((p * 0x9E3779B1) >> 7 & 0x7FFFFFFF).to(torch.int32)
    del p
    torch.cuda.empty_cache()
    out = P().sort(keys)
    torch.cuda.synchronize()
    assert tk.count_unsorted(out) == 0
    assert tk.checksum(out) == tk.checksum(keys)
    del keys, out
    torch.cuda.empty_cache()


# ------------------------------------- pieced inputs / multi-GPU split (8f-4)

@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_merge_pieces_ranges_against_oracle(cuda, port, dt):
    """A and B cut into pieces (no concatenation), any output range."""
    rng = np.random.default_rng(12)
    a, b = _draw(rng, dt, 400_004, 60), _draw(rng, dt, 333_332, 60)
    expect = port.merge(a, b)
    total = len(a) + len(b)
    vece = 16 // np.dtype(dt).itemsize
    for cuts_a, cuts_b in (([], []), ([100_000], [4 * vece]), ([0, 200_000, 200_000 + vece], [333_328]),
                           ([40_000 * k for k in range(1, 8)], [47_616 * k for k in range(1, 7)])):
        pa = [dev(x, cuda) for x in np.split(a, cuts_a)]
        pb = [dev(x, cuda) for x in np.split(b, cuts_b)]
        for lo, hi in ((0, total), (0, 0), (12345, 500_000), (total - 7, total), (1, total - 1)):
            out = P().merge_pieces(pa, pb, lo, hi)
            torch.cuda.synchronize()
            assert np.array_equal(host(out), expect[lo:hi]), (len(pa), len(pb), lo, hi)
    # a piece that is not a 16-byte multiple (and not last) is rejected
    with pytest.raises(ValueError):
        P().merge_pieces([dev(a[:3], cuda), dev(a[3:], cuda)], [dev(b, cuda)], 0, total)


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_merge_pairs_pieces_stability(cuda, port, dt):
    """Key-value pieces: payload pieces cut like their keys; tagged payloads
    prove the A-before-B order across piece and range boundaries."""
    rng = np.random.default_rng(13)
    a, b = _draw(rng, dt, 300_008, 20), _draw(rng, dt, 250_004, 20)
    av, bv = tagged(len(a), len(b))
    ek, ev = port.merge(a, b, av, bv)
    total = len(a) + len(b)
    for cuts_a, cuts_b in (([], []), ([100_000, 200_000], [4]), ([8 * k for k in range(1, 8)], [])):
        pa = [dev(x, cuda) for x in np.split(a, cuts_a)]
        pav = [dev(x, cuda) for x in np.split(av, cuts_a)]
        pb = [dev(x, cuda) for x in np.split(b, cuts_b)]
        pbv = [dev(x, cuda) for x in np.split(bv, cuts_b)]
        for lo, hi in ((0, total), (99_999, 400_001), (total - 5, total)):
            ok, ov = P().merge_pieces(pa, pb, lo, hi, a_val_pieces=pav, b_val_pieces=pbv)
            torch.cuda.synchronize()
            assert np.array_equal(host(ok), ek[lo:hi]) and np.array_equal(host(ov), ev[lo:hi])


def _ipc_worker(rank, world, port, q):
    import os
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)  # one GPU here: the ranks share it (IPC works the same)
        from paper_1303_4312_b200.shard import merge_distributed
        rng = np.random.default_rng(99)  # every rank draws the same full inputs...
        a = np.sort(rng.integers(0, 1000, 600_000)).astype(np.int32)
        b = np.sort(rng.integers(0, 1000, 500_008)).astype(np.int32)
        ca = [0, 250_000, 600_000] if world == 2 else None
        cb = [0, 300_000, 500_008] if world == 2 else None
        # ...and keeps only its own piece on the device
        la = torch.from_numpy(a[ca[rank]:ca[rank + 1]]).cuda()
        lb = torch.from_numpy(b[cb[rank]:cb[rank + 1]]).cuda()
        lo, out = merge_distributed(la, lb)
        av = np.arange(len(a), dtype=np.uint32)
        bv = np.arange(len(b), dtype=np.uint32) | np.uint32(1 << 31)
        lav = torch.from_numpy(av[ca[rank]:ca[rank + 1]]).cuda()
        lbv = torch.from_numpy(bv[cb[rank]:cb[rank + 1]]).cuda()
        lo2, ok, ov = merge_distributed(la, lb, a_vals=lav, b_vals=lbv)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, out.cpu().numpy().tobytes(), ok.cpu().numpy().tobytes(),
                                       ov.cpu().numpy().tobytes()))
        if rank == 0:
            from oracle.py import Port
            parts.sort(key=lambda p: p[0])
            got = np.concatenate([np.frombuffer(p[1], np.int32) for p in parts])
            gk = np.concatenate([np.frombuffer(p[2], np.int32) for p in parts])
            gv = np.concatenate([np.frombuffer(p[3], np.uint32) for p in parts])
            ek, ev = Port().merge(a, b, av, bv)
            q.put(bool(np.array_equal(got, Port().merge(a, b)) and np.array_equal(gk, ek)
                       and np.array_equal(gv, ev)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_merge_distributed_ipc_world2(cuda):
    """Two processes, each holding one piece of A and of B; each merges its
    output range reading the other's piece through a CUDA IPC mapping."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True


# ------------------------------------------------- write-once coverage
# the outputs sit inside a poisoned device buffer; every path must
# write exactly its output range (guards untouched) and every position in it
# (the oracle comparison), for keys, payloads, segmented batches, pieced
# ranges and the sorts.

def _guarded(n, dtype, cuda, guard=4099, poison=0x5A):
    buf = torch.full((n + 2 * guard,), poison, dtype=torch.int64, device=cuda).to(dtype)
    return buf, buf[guard:guard + n], guard


def _guards_intact(buf, n, guard, poison=0x5A):
    h = host(buf.view(torch.uint8) if buf.dtype == torch.uint64 else buf)
    if buf.dtype == torch.uint64:
        h = host(buf.view(torch.int64))
    return bool((h[:guard] == poison).all() and (h[guard + n:] == poison).all())


@pytest.mark.parametrize("guard", [4096, 4099])  # aligned (pipeline) and misaligned output
def test_outputs_written_exactly_once(cuda, path, port, guard):
    rng = np.random.default_rng(21)
    for dt in (np.int32, np.uint64):
        a, b = _draw(rng, dt, 123_457, 30), _draw(rng, dt, 98_765, 30)
        av, bv = tagged(len(a), len(b))
        total = len(a) + len(b)
        # keys
        buf, out, g = _guarded(total, TDT[np.dtype(dt)], cuda, guard)
        P().stable_merge(dev(a, cuda), dev(b, cuda), out)
        torch.cuda.synchronize()
        assert _guards_intact(buf, total, g) and np.array_equal(host(out), port.merge(a, b))
        # key-value
        kbuf, ok, g = _guarded(total, TDT[np.dtype(dt)], cuda, guard)
        vbuf, ov, _ = _guarded(total, torch.uint32, cuda, guard)
        P().merge_pairs(dev(a, cuda), dev(av, cuda), dev(b, cuda), dev(bv, cuda), ok, ov)
        torch.cuda.synchronize()
        ek, ev = port.merge(a, b, av, bv)
        assert _guards_intact(kbuf, total, g) and _guards_intact(vbuf, total, g)
        assert np.array_equal(host(ok), ek) and np.array_equal(host(ov), ev)


@pytest.mark.parametrize("guard", [4096, 4099])
def test_outputs_written_exactly_once_other_modes(cuda, port, guard):
    rng = np.random.default_rng(22)
    # segmented batch (ragged, empty pairs)
    la, lb = rng.integers(0, 700, 400), rng.integers(0, 700, 400)
    la[::9] = 0
    sa = np.concatenate([np.sort(rng.integers(0, 99, x)) for x in la]).astype(np.int32)
    sb = np.concatenate([np.sort(rng.integers(0, 99, x)) for x in lb]).astype(np.int32)
    ao = np.concatenate([[0], np.cumsum(la)]).astype(np.uint64)
    bo = np.concatenate([[0], np.cumsum(lb)]).astype(np.uint64)
    total = len(sa) + len(sb)
    buf, out, g = _guarded(total, torch.int32, cuda, guard)
    P().merge_segmented(dev(sa, cuda), dev(ao, cuda), dev(sb, cuda), dev(bo, cuda), out)
    torch.cuda.synchronize()
    assert _guards_intact(buf, total, g)
    assert np.array_equal(host(out), port.merge_segmented(sa, ao, sb, bo))
    # pieced range merge
    a, b = _draw(rng, np.int32, 200_000, 50), _draw(rng, np.int32, 180_004, 50)
    lo, hi = 77_777, 300_001
    buf, out, g = _guarded(hi - lo, torch.int32, cuda, 4096)
    P().merge_pieces([dev(a[:100_000], cuda), dev(a[100_000:], cuda)], [dev(b, cuda)], lo, hi,
                     out=out)
    torch.cuda.synchronize()
    assert _guards_intact(buf, hi - lo, g) and np.array_equal(host(out), port.merge(a, b)[lo:hi])
    # sorts (keys, pairs) into guarded outputs
    k = rng.integers(-5000, 5000, 150_001).astype(np.int32)
    v = np.arange(len(k), dtype=np.uint32)
    buf, out, g = _guarded(len(k), torch.int32, cuda, guard)
    P().sort(dev(k, cuda), out=out)
    torch.cuda.synchronize()
    assert _guards_intact(buf, len(k), g) and np.array_equal(host(out), port.merge_sort(k))
    kbuf, ok, g = _guarded(len(k), torch.int32, cuda, guard)
    vbuf, ov, _ = _guarded(len(k), torch.uint32, cuda, guard)
    P().sort_pairs(dev(k, cuda), dev(v, cuda), out_keys=ok, out_vals=ov)
    torch.cuda.synchronize()
    ek, ev = port.merge_sort_pairs(k, v)
    assert _guards_intact(kbuf, len(k), g) and _guards_intact(vbuf, len(k), g)
    assert np.array_equal(host(ok), ek) and np.array_equal(host(ov), ev)


# ------------------------------------------------------- CUDA graph replay
def test_cuda_graph_replay_new_inputs(cuda, port):
    """A merge captured in a CUDA graph and replayed on new contents of the same
    buffers: the dynamic tail's per-launch epoch comes from a device-side
    launch counter, so identical kernel arguments never reuse stale state."""
    rng = np.random.default_rng(31)
    m, n = 1 << 21, (1 << 21) + 12345
    ta = torch.empty(m, dtype=torch.int32, device=cuda)
    tb = torch.empty(n, dtype=torch.int32, device=cuda)
    tav = torch.arange(m, dtype=torch.int32, device=cuda).view(torch.uint32)
    tbv = (torch.arange(n, dtype=torch.int64, device=cuda) | (1 << 31)).to(torch.int32).view(torch.uint32)
    ok = torch.empty(m + n, dtype=torch.int32, device=cuda)
    ov = torch.empty(m + n, dtype=torch.uint32, device=cuda)
    ws = torch.empty(P().workspace_bytes(m, n, torch.int32, True), dtype=torch.uint8, device=cuda)

    def fill(seed):
        r = np.random.default_rng(seed)
        a = np.sort(r.integers(0, 1 << 20, m)).astype(np.int32)
        b = np.sort(r.integers(0, 1 << 20, n)).astype(np.int32)
        ta.copy_(torch.from_numpy(a))
        tb.copy_(torch.from_numpy(b))
        return a, b

    fill(0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside capture (occupancy, attributes)
        P().merge_pairs(ta, tav, tb, tbv, ok, ov, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        P().merge_pairs(ta, tav, tb, tbv, ok, ov, workspace=ws)
    av, bv = host(tav), host(tbv)
    for seed in (1, 2, 3, 4):
        a, b = fill(seed)
        g.replay()
        torch.cuda.synchronize()
        ek, ev = port.merge(a, b, av, bv)
        assert np.array_equal(host(ok), ek) and np.array_equal(host(ov), ev), seed


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_merge_pieces_large_range_with_dynamic_tail(cuda, port, dt):
    """Ranges long enough for the pipeline's dynamic tail (>= 4 tiles per CTA),
    ending before m + n: the tail's last boundary is co-ranked, not (m, n)."""
    rng = np.random.default_rng(41)
    m, n = 6_000_000, 5_000_004
    a, b = _draw(rng, dt, m, 1 << 16), _draw(rng, dt, n, 1 << 16)
    expect = port.merge_parallel(a, b, 16, threads=8)[0]
    pa = [dev(a[:2_000_000], cuda), dev(a[2_000_000:], cuda)]
    pb = [dev(b[:3_000_000], cuda), dev(b[3_000_000:], cuda)]
    for lo, hi in ((1_234_567, m + n - 7), (0, m + n), (3, 10_000_001)):
        out = P().merge_pieces(pa, pb, lo, hi)
        torch.cuda.synchronize()
        assert np.array_equal(host(out), expect[lo:hi]), (lo, hi)


@pytest.mark.parametrize("unit", [1, 2, 3, 4, 7])
def test_tail_anchor_units(cuda, port, unit):
    """Dynamic-tail anchors (merge_pipe.cuh, pipe_args::tail_unit): every
    unit-th tail boundary co-ranked over the whole diagonal, the ones between
    bracketed by it, the last 2 x grid single.  Sizes where the anchored part
    is not a multiple of the unit; keys-only int32 (duplicate-heavy), key-value
    int32, and an output range (range merges co-rank the end boundary too)."""
    import paper_1303_4312_b200._native as N
    rng = np.random.default_rng(100 + unit)
    m, n = 11_000_003, 9_500_001  # 2583 int32 tiles: tail 775 (> 2 x 296 singles)
    a, b = _draw(rng, np.int32, m, 1 << 12), _draw(rng, np.int32, n, 1 << 12)
    av, bv = tagged(m, n)
    ek, ev = port.merge(a, b, av, bv)
    da, db, dav, dbv = dev(a, cuda), dev(b, cuda), dev(av, cuda), dev(bv, cuda)
    N.lib.comerge_cuda_set_tuning(0, unit << 15, 0)
    try:
        P().set_kernel_path("pipe")
        keys = P().stable_merge(da, db)
        ok, ov = P().merge_pairs(da, dav, db, dbv)
        lo, hi = 1_000_001, m + n - 12_345
        rk = P().merge_pieces([da], [db], lo, hi)
        torch.cuda.synchronize()
    finally:
        N.lib.comerge_cuda_set_tuning(0, 0, 0)
        P().set_kernel_path("auto")
    assert np.array_equal(host(keys), ek)
    assert np.array_equal(host(ok), ek) and np.array_equal(host(ov), ev)
    assert np.array_equal(host(rk), ek[lo:hi])


def test_concurrent_streams_and_host_threads(cuda, port):
    """Reentrancy (async on the caller's stream, reentrant across
    streams, no global mutable state): 4 host threads, each on its own CUDA
    stream, interleave device key-value merges (tile pipeline with dynamic
    tails running concurrently, scratch from the private pool), segmented
    batches and host-buffer merges (the chunked H2D/merge/D2H pipeline);
    every result bit-exact against the oracle."""
    import threading
    rng = np.random.default_rng(777)
    cases = []
    for t in range(4):
        m, n = int(rng.integers(300_000, 2_500_000)), int(rng.integers(300_000, 2_500_000))
        a = _draw(rng, np.int32, m, 1000 if t % 2 else 0)
        b = _draw(rng, np.int32, n, 1000 if t % 2 else 0)
        av, bv = tagged(m, n)
        la, lb = rng.integers(0, 3000, 200), rng.integers(0, 3000, 200)
        sa = np.concatenate([_draw(rng, np.int32, int(x), 1 << 20) for x in la])
        sb = np.concatenate([_draw(rng, np.int32, int(x), 1 << 20) for x in lb])
        ao = np.concatenate([[0], np.cumsum(la)]).astype(np.uint64)
        bo = np.concatenate([[0], np.cumsum(lb)]).astype(np.uint64)
        cases.append(dict(a=a, b=b, av=av, bv=bv, sa=sa, sb=sb, ao=ao, bo=bo,
                          ek=port.merge(a, b, av, bv), es=port.merge_segmented(sa, ao, sb, bo)))
    errors = []

    def worker(t):
        try:
            c = cases[t]
            s = torch.cuda.Stream(device=cuda)
            with torch.cuda.stream(s):
                ta, tb = dev(c["a"], cuda), dev(c["b"], cuda)
                tav, tbv = dev(c["av"], cuda), dev(c["bv"], cuda)
                ts = [dev(c[k], cuda) for k in ("sa", "ao", "sb", "bo")]
                for _ in range(5):
                    ok, ov = P().merge_pairs(ta, tav, tb, tbv)
                    so = P().merge_segmented(*ts)
                    hk = np.empty(len(c["a"]) + len(c["b"]), np.int32)
                    P().merge_parallel(c["a"], c["b"], hk, 3)  # host buffers
                    s.synchronize()
                    assert np.array_equal(host(ok), c["ek"][0]), t
                    assert np.array_equal(host(ov), c["ek"][1]), t
                    assert np.array_equal(host(so), c["es"]), t
                    assert np.array_equal(hk, c["ek"][0]), t
        except Exception as e:  # noqa: BLE001 -- reported below
            errors.append((t, repr(e)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
