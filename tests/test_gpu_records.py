"""GPU parity of the key-value RECORD merge -- the reference's own key-value
call shape: merge_parallel<T>(a, b, out, workers, less) over a {key, val}
struct with a key-only less (tagged<K> / tagged_key_less,
/root/reference/proj/include/comerge/oracle.hpp:22-37; parallel.hpp:304-317).

Expected outputs come from the reference itself (oracle/_ref:
comerge::merge_parallel over its {key, val} structs), compared field by field
(keys and payloads bit-exact); the padding word of 16-byte records must
travel with its record (it is set to a function of the payload).  Device and
host buffers, every alignment class of the arrays (16 / 8 / 4-byte record
positions), tile-boundary, empty and ragged shapes, duplicate-heavy keys.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

T_REC = {np.int32: 256 * 15, np.uint32: 256 * 15, np.uint64: 256 * 7}  # pipeline tile sizes
PAD_MIX = np.uint32(0x5BD1E995)


def P():
    import paper_1303_4312_b200 as mod
    return mod


def _keys(rng, dt, size, alphabet):
    if alphabet == 0:
        hi = 2**64 if dt == np.uint64 else 2**31
        v = rng.integers(0, hi, size, dtype=np.uint64 if dt == np.uint64 else np.int64)
        if dt == np.int32:
            v = v - 2**30
    else:
        v = rng.integers(0, alphabet, size) - (alphabet // 2 if dt == np.int32 else 0)
    return np.sort(v.astype(dt))


def records(keys, tag):
    r = np.zeros(len(keys), P().record_dtype(keys.dtype))
    r["key"] = keys
    r["val"] = np.arange(len(keys), dtype=np.uint32) | np.uint32(tag)
    if "pad" in r.dtype.names:
        r["pad"] = r["val"] ^ PAD_MIX
    return r


def reference_merge(a, b):
    """comerge::merge_parallel over the reference's {key, val} structs."""
    from oracle.py import KIND, Ref, kv_dtype
    ref = Ref()
    kind = KIND[np.dtype(a["key"].dtype)]
    ra = np.zeros(len(a), kv_dtype(kind))
    rb = np.zeros(len(b), kv_dtype(kind))
    ra["key"], ra["val"] = a["key"], a["val"]
    rb["key"], rb["val"] = b["key"], b["val"]
    out, _ = ref.merge_parallel_kv(ra, rb, max(1, ref.hardware_concurrency()))
    return np.ascontiguousarray(out["key"]), np.ascontiguousarray(out["val"])


def check(got, a, b):
    ek, ev = reference_merge(a, b)
    assert np.array_equal(got["key"], ek)
    assert np.array_equal(got["val"], ev)
    if "pad" in got.dtype.names:  # the whole record moved, padding included
        assert np.array_equal(got["pad"], got["val"] ^ PAD_MIX)


def on_device(r, cuda, offset=0):
    """Record bytes in a device buffer starting `offset` bytes past a 256-byte
    aligned allocation (alignment classes of the record positions)."""
    raw = r.view(np.uint8)
    buf = torch.zeros(len(raw) + offset + 64, dtype=torch.uint8, device=cuda)
    view = buf[offset:offset + len(raw)]
    view.copy_(torch.from_numpy(raw.copy()).to(cuda))
    return view


def device_merge(a, b, cuda, offs=(0, 0, 0)):
    kd = a["key"].dtype
    ta, tb = on_device(a, cuda, offs[0]), on_device(b, cuda, offs[1])
    size = a.dtype.itemsize
    obuf = torch.full(((len(a) + len(b)) * size + offs[2] + 64,), 0x77, dtype=torch.uint8,
                      device=cuda)
    out = obuf[offs[2]:offs[2] + (len(a) + len(b)) * size]
    P().merge_records(ta, tb, out, key_dtype=kd)
    torch.cuda.synchronize()
    h = obuf.cpu().numpy()
    # nothing written outside the output range
    assert (h[:offs[2]] == 0x77).all() and (h[offs[2] + len(out):] == 0x77).all()
    return out.cpu().numpy().view(a.dtype)


@pytest.mark.parametrize("dt", [np.int32, np.uint32, np.uint64])
def test_records_device_against_reference(cuda, dt):
    rng = np.random.default_rng(17 + np.dtype(dt).itemsize)
    T = T_REC[dt]
    shapes = [(0, 0), (0, 1), (1, 0), (T - 1, 0), (0, T + 1), (T, T), (T - 1, 1), (1, T - 1),
              (2 * T + 3, 5), (5, 3 * T - 2), (3, 50000), (50000, 3), (70001, 69999),
              (1 << 20, (1 << 20) + 7)]
    shapes += [(int(rng.integers(0, 20000)), int(rng.integers(0, 20000))) for _ in range(6)]
    for idx, (m, n) in enumerate(shapes):
        alphabet = [0, 1, 2, 16, 1000][idx % 5]
        a = records(_keys(rng, dt, m, alphabet), 0)
        b = records(_keys(rng, dt, n, alphabet), 1 << 31)
        check(device_merge(a, b, cuda), a, b)


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_records_alignment_classes(cuda, dt):
    """Arrays at any record offset: 16-, 8- and (8-byte records) 4-byte
    aligned positions pick different vector widths; outputs identical."""
    rng = np.random.default_rng(3)
    offsets = [(0, 0, 0), (8, 0, 8), (0, 8, 0), (8, 8, 8)]
    if dt == np.int32:
        offsets += [(4, 0, 0), (0, 4, 12), (12, 4, 4)]
    for m, n in [(100_003, 77_777), (5000, 3)]:
        a = records(_keys(rng, dt, m, 40), 0)
        b = records(_keys(rng, dt, n, 40), 1 << 31)
        for offs in offsets:
            check(device_merge(a, b, cuda, offs), a, b)


def test_records_misaligned_to_record_type_rejected(cuda):
    a = records(np.arange(10, dtype=np.uint64), 0)
    ta = on_device(a, cuda, 4)  # 16-byte records need 8-byte alignment
    with pytest.raises(ValueError, match="aligned"):
        P().merge_records(ta, ta, key_dtype=np.uint64)


@pytest.mark.parametrize("dt", [np.int32, np.uint64])
def test_records_host_buffers(cuda, dt):
    """Host arrays: small ones staged, >= 2^20 records through the chunked
    H2D / merge / D2H pipeline; the report's block sizes are the reference's."""
    rng = np.random.default_rng(11)
    for m, n, alphabet in [(1000, 999, 7), (1_500_000, 2_100_003, 1000), (3_000_001, 17, 0)]:
        a = records(_keys(rng, dt, m, alphabet), 0)
        b = records(_keys(rng, dt, n, alphabet), 1 << 31)
        out, rep = P().merge_records(a, b, workers=7)
        check(out, a, b)
        total = m + n
        assert rep.block_sizes == [P().partition_output(total, 7, r + 1) -
                                   P().partition_output(total, 7, r) for r in range(7)]
        if total >= 1 << 20:
            assert rep.h2d_bytes == total * a.dtype.itemsize == rep.d2h_bytes


def test_records_c2_c4_shapes_full_size(cuda):
    """C2 and C4 in the reference's record form at full size, byte for byte
    against the reference (bench.py's seeded inputs)."""
    import bench
    for cfg in ("C2", "C4"):
        inp = bench.make_inputs(cfg, seed=5, device=cuda)
        a = records(inp["a"].cpu().numpy(), 0)
        b = records(inp["b"].cpu().numpy(), 1 << 31)
        del inp
        got = device_merge(a, b, cuda)
        check(got, a, b)
        del a, b, got
        torch.cuda.empty_cache()


# ---- 12-byte records: the reference's OWN tagged<int32_t> / tagged<uint32_t>
# (oracle.hpp:22-27: key, origin byte + 3 padding bytes, uint32 index),
# merged by comerge::merge_parallel(..., tagged_key_less{}) in oracle/_ref.

T_REC12 = 256 * 11  # pipeline tile of 12-byte records


def tagged(keys, origin):
    """Records in the reference's tagged<K> layout; the padding bytes carry a
    pattern of the index (they must travel with their record)."""
    from oracle.py import KIND, tagged_dtype
    r = np.zeros(len(keys), tagged_dtype(KIND[np.dtype(keys.dtype)]))
    r["key"] = keys
    r["origin"] = origin
    r["index"] = np.arange(len(keys), dtype=np.uint32)
    raw = r.view(np.uint8).reshape(len(keys), 12)
    raw[:, 5:8] = (r["index"][:, None] >> np.array([0, 8, 16], np.uint32)).astype(np.uint8) ^ 0xA5
    return r


def check_tagged(got, a, b):
    """Byte for byte against comerge::merge_parallel over tagged<K> with
    tagged_key_less (the reference, hardware_concurrency workers)."""
    from oracle.py import Ref
    ref = Ref()
    expect, rep = ref.merge_parallel_tagged(a, b, max(1, ref.hardware_concurrency()))
    assert rep.m == len(a) and rep.n == len(b)
    assert got.tobytes() == expect.tobytes()


def device_merge12(a, b, cuda, offs=(0, 0, 0)):
    kd = a["key"].dtype
    ta, tb = on_device(a, cuda, offs[0]), on_device(b, cuda, offs[1])
    obuf = torch.full(((len(a) + len(b)) * 12 + offs[2] + 64,), 0x77, dtype=torch.uint8,
                      device=cuda)
    out = obuf[offs[2]:offs[2] + (len(a) + len(b)) * 12]
    P().merge_records(ta, tb, out, key_dtype=kd, record_bytes=12)
    torch.cuda.synchronize()
    h = obuf.cpu().numpy()
    assert (h[:offs[2]] == 0x77).all() and (h[offs[2] + len(out):] == 0x77).all()
    return out.cpu().numpy().view(a.dtype)


@pytest.mark.parametrize("dt", [np.int32, np.uint32])
def test_tagged12_device_against_reference(cuda, dt):
    """Every device path (small-merge kernel, tile pipeline) over tile-boundary,
    empty, ragged and duplicate-heavy shapes."""
    rng = np.random.default_rng(1212 + (dt == np.uint32))
    T = T_REC12
    shapes = [(0, 0), (0, 1), (1, 0), (T - 1, 0), (0, T + 1), (T, T), (T - 1, 1), (1, T - 1),
              (2 * T + 3, 5), (5, 3 * T - 2), (3, 50000), (50000, 3), (70001, 69999),
              (1 << 20, (1 << 20) + 7), (3_000_001, 2_999_999)]
    shapes += [(int(rng.integers(0, 20000)), int(rng.integers(0, 20000))) for _ in range(6)]
    for idx, (m, n) in enumerate(shapes):
        alphabet = [0, 1, 2, 16, 1000][idx % 5]
        a = tagged(_keys(rng, dt, m, alphabet), 0)
        b = tagged(_keys(rng, dt, n, alphabet), 1)
        check_tagged(device_merge12(a, b, cuda), a, b)


def test_tagged12_any_record_offset(cuda):
    """12-byte record positions are 4-byte aligned in general: arrays at byte
    offsets 0 / 4 / 8 / 12 of an allocation, inputs and output."""
    rng = np.random.default_rng(5)
    for m, n in [(100_003, 77_777), (5000, 3), (1_000_000, 1_000_001)]:
        a = tagged(_keys(rng, np.int32, m, 40), 0)
        b = tagged(_keys(rng, np.int32, n, 40), 1)
        for offs in [(0, 0, 0), (4, 8, 12), (12, 4, 8), (8, 12, 4)]:
            check_tagged(device_merge12(a, b, cuda, offs), a, b)


def test_tagged12_host_buffers(cuda):
    """Host arrays of the reference's tagged<int32_t>: small ones staged,
    >= 2^20 records through the chunked H2D / merge / D2H pipeline."""
    rng = np.random.default_rng(12)
    for m, n, alphabet in [(1000, 999, 7), (1_500_000, 2_100_003, 1000), (3_000_001, 17, 0)]:
        a = tagged(_keys(rng, np.int32, m, alphabet), 0)
        b = tagged(_keys(rng, np.int32, n, alphabet), 1)
        out, rep = P().merge_records(a, b, workers=7)
        check_tagged(out, a, b)
        if m + n >= 1 << 20:
            assert rep.h2d_bytes == (m + n) * 12 == rep.d2h_bytes


def test_tagged12_c2_full_size(cuda):
    """C2 in the reference's tagged<int32_t> form at full size, byte for byte
    against the reference."""
    import bench
    inp = bench.make_inputs("C2", seed=5, device=cuda)
    a = tagged(inp["a"].cpu().numpy(), 0)
    b = tagged(inp["b"].cpu().numpy(), 1)
    del inp
    check_tagged(device_merge12(a, b, cuda), a, b)


# ---- the rest of the reference's generic API over records with a key-only
# less: co_rank / co_rank_counted (corank.hpp:128-147), plan
# (parallel.hpp:94-115), merge_parallel / merge_parallel_synced with
# merge_options::count_comparisons (parallel.hpp:304-336).  Only keys are
# compared, so every number equals the reference's on the records' key arrays.

def _record_cases(rng):
    for dt, size in [(np.int32, 8), (np.uint32, 8), (np.int32, 12), (np.uint32, 12),
                     (np.uint64, 16)]:
        for m, n, alphabet in [(0, 0, 3), (0, 9, 3), (7, 0, 3), (2, 2, 1), (1000, 777, 5),
                               (20_000, 30_001, 0)]:
            ka, kb = _keys(rng, dt, m, alphabet), _keys(rng, dt, n, alphabet)
            if size == 12:
                yield ka, kb, tagged(ka, 0), tagged(kb, 1)
            else:
                yield ka, kb, records(ka, 0), records(kb, 1 << 31)


def test_records_co_rank_and_plan_match_reference(cuda):
    from oracle.py import Ref
    ref = Ref()
    rng = np.random.default_rng(99)
    for ka, kb, a, b in _record_cases(rng):
        total, size, kd = len(ka) + len(kb), a.dtype.itemsize, ka.dtype
        ranks = sorted({0, total, total // 2, min(total, 1), max(total, 1) - 1,
                        *(int(x) for x in rng.integers(0, total + 1, 6))})
        ta, tb = on_device(a, cuda, 0), on_device(b, cuda, 0)
        for i in ranks:
            want, wstats = ref.co_rank(i, ka, kb, stats=True)
            st = P().CoRankStats()
            assert P().co_rank_records(i, a, b, stats=st) == want           # host arrays
            assert (st.iterations, st.comparisons) == wstats
            st = P().CoRankStats()
            assert P().co_rank_records(i, ta, tb, key_dtype=kd, record_bytes=size,
                                       stats=st) == want                     # device views
            assert (st.iterations, st.comparisons) == wstats
        with pytest.raises(IndexError, match="rank out of range"):
            P().co_rank_records(total + 1, a, b)
        # batched, on the device
        r = torch.tensor(ranks, dtype=torch.int64, device=cuda).view(torch.uint64)
        j, it, cmp = P().co_rank_batch_records(r, ta, tb, kd, size, with_stats=True)
        torch.cuda.synchronize()
        wants = [ref.co_rank(i, ka, kb, stats=True) for i in ranks]
        assert j.view(torch.int64).tolist() == [w[0][0] for w in wants]
        assert it.view(torch.int32).tolist() == [w[1][0] for w in wants]
        assert cmp.view(torch.int32).tolist() == [w[1][1] for w in wants]
        for workers in (1, 3, 16):
            got = [blk.as_tuple() for blk in P().plan_records(a, b, workers)]
            assert got == [tuple(int(x) for x in row) for row in ref.plan(ka, kb, workers)]
            assert got == [blk.as_tuple() for blk in
                           P().plan_records(ta, tb, workers, key_dtype=kd, record_bytes=size)]
    with pytest.raises(ValueError, match="worker count must be positive"):
        P().plan_records(a, b, 0)
    with pytest.raises(ValueError, match="8 or 12 bytes"):
        P().co_rank_records(0, np.zeros(32, np.uint8), np.zeros(32, np.uint8),
                            key_dtype=np.int32, record_bytes=16)


def test_records_full_report_matches_reference(cuda):
    """block sizes, co-rank iterations and count_comparisons totals of the
    record merges = the reference's merge_parallel on the key arrays, both
    modes; the merged records byte for byte (host staging, the chunked host
    pipeline and device buffers)."""
    from oracle.py import Ref
    ref = Ref()
    rng = np.random.default_rng(123)
    opts = P().MergeOptions(count_comparisons=True)
    cases = list(_record_cases(rng))
    dt = np.int32  # one case through the chunked host pipeline (>= 2^20 records)
    ka, kb = _keys(rng, dt, 1_300_000, 50), _keys(rng, dt, 900_001, 50)
    cases.append((ka, kb, tagged(ka, 0), tagged(kb, 1)))
    for ka, kb, a, b in cases:
        size, kd = a.dtype.itemsize, ka.dtype
        for workers in (1, 5, 33):
            for synced in (False, True):
                _, rrep, rbs, rits = ref.merge_parallel(ka, kb, workers, synced=synced, count=True)
                nit = workers if synced else 2 * workers
                out = np.zeros(len(a) + len(b), a.dtype)
                rep = P().merge_parallel_records(a, b, out, workers, opts=opts, synced=synced)
                if size == 12:
                    check_tagged(out, a, b)
                else:
                    check(out, a, b)
                assert rep.block_sizes == [int(x) for x in rbs[:workers]]
                assert rep.corank_iterations == [int(x) for x in rits[:nit]]
                assert rep.comparisons == int(rrep.comparisons)
                if len(a) + len(b) > 100_000:
                    continue
                ta, tb = on_device(a, cuda, 0), on_device(b, cuda, 0)
                to = torch.zeros((len(a) + len(b)) * size, dtype=torch.uint8, device=cuda)
                drep = P().merge_parallel_records(ta, tb, to, workers, key_dtype=kd,
                                                  record_bytes=size, opts=opts, synced=synced)
                assert to.cpu().numpy().tobytes() == out.tobytes()
                assert (drep.block_sizes, drep.corank_iterations, drep.comparisons) == \
                    (rep.block_sizes, rep.corank_iterations, rep.comparisons)
        assert P().merge_parallel_records(a, b, out, 2).comparisons is None
