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
