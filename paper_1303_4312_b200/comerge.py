"""Python mirror of the reference's co-rank / merge API, backed by sm_100a kernels.

Names, argument meaning and error behaviour follow the reference library
(/root/reference/proj/include/comerge/):

===========================  ==============================================
this module                  reference
===========================  ==============================================
``co_rank``                  ``comerge::co_rank``            corank.hpp:128-133
``co_rank_counted``          ``comerge::co_rank_counted``    corank.hpp:138-147
``stable_merge``             ``comerge::stable_merge``       merge.hpp:52-68
``partition_output``         ``comerge::partition_output``   parallel.hpp:60-67
``plan``                     ``comerge::plan``               parallel.hpp:94-115
``merge_parallel``           ``comerge::merge_parallel``     parallel.hpp:304-317
``merge_parallel_synced``    ``comerge::merge_parallel_synced`` :323-336
``MergeReport``              ``comerge::merge_report``       parallel.hpp:44-55
===========================  ==============================================

Exceptions: ``ValueError`` = std::invalid_argument, ``IndexError`` =
std::out_of_range, ``OverflowError`` = std::length_error (same message
substrings as the reference).  Arrays may be numpy (host) or torch CUDA
tensors (device); every merge runs on the GPU through the C ABI in
``include/comerge_cuda.h`` -- there is no CPU fallback.

Extensions beyond the reference (the B200 hot path's other shapes):
``merge_pairs`` (key + uint32 payload), ``merge_segmented`` (batched
independent pairs) and ``co_rank_batch``.
"""
from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _native as N

try:  # torch is plumbing only (device memory + streams)
    import torch
except Exception:  # pragma: no cover
    torch = None

_SUFFIX = {"int32": "i32", "uint32": "u32", "uint64": "u64"}
_KIND = {"i32": N.KEY_I32, "u32": N.KEY_U32, "u64": N.KEY_U64}


def _is_torch(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor)


def _dtype_name(x) -> str:
    if _is_torch(x):
        return str(x.dtype).replace("torch.", "")
    return np.dtype(x.dtype).name


def _suffix(x) -> str:
    name = _dtype_name(x)
    if name not in _SUFFIX:
        raise TypeError(f"comerge: unsupported key dtype {name} (int32, uint32, uint64)")
    return _SUFFIX[name]


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        if not x.is_contiguous():
            raise ValueError("comerge: arrays must be contiguous")
        return C.c_void_p(x.data_ptr()) if x.numel() else None
    if not x.flags["C_CONTIGUOUS"]:
        raise ValueError("comerge: arrays must be contiguous")
    return C.c_void_p(x.ctypes.data) if x.size else None


def _len(x) -> int:
    return int(x.numel()) if _is_torch(x) else int(x.size)


def _stream(x=None):
    if x is not None and _is_torch(x) and x.is_cuda:
        return C.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
    return None


def _on(x):
    """Run a call with x's device current (kernels launch on the current
    device; the library caches its per-device state by it)."""
    if _is_torch(x) and x.is_cuda:
        return torch.cuda.device(x.device)
    return contextlib.nullcontext()


def _empty_like_merge(a, total):
    if _is_torch(a):
        return torch.empty(total, dtype=a.dtype, device=a.device)
    return np.empty(total, dtype=a.dtype)


# ----------------------------------------------------------------- co_rank

@dataclass
class CoRankStats:
    """comerge::co_rank_stats (corank.hpp:44-47)."""
    iterations: int = 0
    comparisons: int = 0


@dataclass
class ComparisonCounter:
    """comerge::comparison_counter (corank.hpp:50-52)."""
    count: int = 0


def co_rank(target: int, a, b, stats: Optional[CoRankStats] = None):
    """Unique split (j, k), j + k = target, of the stable merge of a and b.

    Runs Algorithm 1 (corank.hpp:72-121) on the device; raises IndexError
    ("rank out of range") when target > m + n, like the reference.
    """
    suf = _suffix(a)
    if _suffix(b) != suf:
        raise TypeError("co_rank: a and b must have the same dtype")
    if target < 0:
        raise IndexError("co_rank: rank out of range (exceeds m+n)")
    j, k, it, cmp = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_uint32()
    with _on(a):
        N.check(getattr(N.lib, f"comerge_co_rank_{suf}")(
            int(target), _ptr(a), _len(a), _ptr(b), _len(b), C.byref(j), C.byref(k), C.byref(it),
            C.byref(cmp)))
    if stats is not None:
        stats.iterations, stats.comparisons = it.value, cmp.value
    return (j.value, k.value)


def co_rank_counted(target: int, a, b, counter: ComparisonCounter):
    st = CoRankStats()
    res = co_rank(target, a, b, st)
    counter.count += st.comparisons
    return res


def co_rank_batch(ranks, a, b, with_stats: bool = False):
    """Device batch of co-ranks: returns j (uint64 tensor) [, iterations, comparisons]."""
    suf = _suffix(a)
    dev = a.device
    q = int(ranks.numel())
    j = torch.empty(q, dtype=torch.uint64, device=dev)
    it = torch.empty(q, dtype=torch.uint32, device=dev) if with_stats else None
    cmp = torch.empty(q, dtype=torch.uint32, device=dev) if with_stats else None
    with _on(a):
        N.check(getattr(N.lib, f"comerge_cuda_co_rank_batch_{suf}")(
            _ptr(ranks), q, _ptr(a), _len(a), _ptr(b), _len(b), _ptr(j), _ptr(it), _ptr(cmp),
            _stream(a)))
    return (j, it, cmp) if with_stats else j


# ------------------------------------------------------------------- merges

KERNEL_PATHS = {"auto": 0, "tile": 1, "pipe": 3, "small": 4}


def set_kernel_path(path: str = "auto") -> None:
    """Select the device kernel for merges issued from this thread: "auto",
    "tile" (partition + one CTA per tile), "pipe" (persistent tile pipeline;
    the default above one wave of tiles, segmented batches included) or
    "small" (one-wave kernel, one CTA per tile; the default up to one wave)."""
    N.lib.comerge_cuda_set_path(KERNEL_PATHS[path])


def partition_output(total: int, workers: int, r: int) -> int:
    """floor(r * total / workers) without overflow (parallel.hpp:60-67)."""
    if workers < 0 or r < 0:
        raise ValueError("partition_output: worker count must be positive")
    out = C.c_uint64()
    N.check(N.lib.comerge_partition_output(total, workers, r, C.byref(out)))
    return out.value


def _check_out(who, a, b, out):
    if _len(out) != _len(a) + _len(b):
        raise ValueError(f"{who}: output length must equal |a| + |b|")


def _ws(workspace):
    if workspace is None:
        return None, 0
    return C.c_void_p(workspace.data_ptr()), int(workspace.numel() * workspace.element_size())


def workspace_bytes(m: int, n: int, dtype, has_payload: bool = False) -> int:
    """Scratch bytes a device merge of (m, n) may use (CUB-style query);
    dtype is a numpy or torch dtype of the keys."""
    name = str(dtype).replace("torch.", "") if torch is not None and isinstance(dtype, torch.dtype) \
        else np.dtype(dtype).name
    kind = _KIND[_SUFFIX[name]]
    return int(N.lib.comerge_cuda_merge_workspace_bytes(m, n, kind, int(has_payload)))


def stable_merge(a, b, out=None, workspace=None):
    """Stable two-way merge into out (merge.hpp:52-68).  Device tensors run
    asynchronously on the current stream (scratch from `workspace`, a device
    tensor of >= workspace_bytes() bytes, else from a stream-ordered pool);
    host arrays synchronously."""
    suf = _suffix(a)
    if out is None:
        out = _empty_like_merge(a, _len(a) + _len(b))
    _check_out("stable_merge", a, b, out)
    if _is_torch(a) and a.is_cuda:
        wsp, wsb = _ws(workspace)
        with _on(a):
            N.check(getattr(N.lib, f"comerge_cuda_merge_keys_{suf}")(
                _ptr(a), _len(a), _ptr(b), _len(b), _ptr(out), wsp, wsb, _stream(a)))
    else:
        rep = N.MergeReport()
        rc = getattr(N.lib, f"comerge_merge_parallel_{suf}")(
            _ptr(a), _len(a), _ptr(b), _len(b), _ptr(out), _len(out), 1, 0, C.byref(rep),
            None, None)
        if rc == N.E_INVALID:
            raise ValueError(N.last_error().replace("merge_parallel", "stable_merge"))
        N.check(rc)
    return out


@dataclass
class MergeReport:
    """comerge::merge_report (parallel.hpp:44-55) plus device-side fields."""
    m: int = 0
    n: int = 0
    workers: int = 0
    wall_ns: int = 0
    block_sizes: List[int] = field(default_factory=list)
    corank_iterations: List[int] = field(default_factory=list)
    comparisons: Optional[int] = None
    verified: Optional[bool] = None
    speedup_vs_p1: Optional[float] = None
    note: str = ""
    # B200 extras
    e2e_ns: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    tiles: int = 0


@dataclass
class MergeOptions:
    """comerge::merge_options (parallel.hpp:39-42).  `mode` is accepted for
    API compatibility; the device schedule does not depend on it.
    `count_comparisons` fills MergeReport.comparisons with the reference's
    total (co-ranks + every block's merge_into), computed exactly from the
    block windows."""
    mode: str = "threads"
    count_comparisons: bool = False


def _merge_parallel(who, a, b, out, workers, opts, synced):
    suf = _suffix(a)
    if _suffix(b) != suf or _suffix(out) != suf:
        raise TypeError(f"{who}: a, b and out must share one dtype")
    count = bool(opts is not None and opts.count_comparisons)
    if workers < 0:
        raise ValueError("merge_parallel: worker count must be positive")
    rep = N.MergeReport()
    bs = np.zeros(max(workers, 1), np.uint64)
    its = np.zeros(2 * max(workers, 1), np.uint32)
    cmp = C.c_uint64(0)
    mo = N.MergeOptions(int(synced), int(count))
    if _is_torch(out) and out.is_cuda:
        torch.cuda.current_stream(out.device).synchronize()
    with _on(out if _is_torch(out) and out.is_cuda else a):
        N.check(getattr(N.lib, f"comerge_merge_parallel_ex_{suf}")(
            _ptr(a), None, _len(a), _ptr(b), None, _len(b), _ptr(out), None, _len(out), workers,
            C.byref(mo), C.byref(rep), C.c_void_p(bs.ctypes.data), C.c_void_p(its.ctypes.data),
            C.byref(cmp)))
    return MergeReport(
        m=rep.m, n=rep.n, workers=rep.workers, wall_ns=rep.wall_ns,
        block_sizes=[int(x) for x in bs[:workers]],
        corank_iterations=[int(x) for x in its[:(workers if synced else 2 * workers)]],
        comparisons=int(cmp.value) if count else None,
        e2e_ns=rep.e2e_ns, h2d_bytes=rep.h2d_bytes, d2h_bytes=rep.d2h_bytes, tiles=rep.tiles)


def merge_parallel(a, b, out, workers: int, less=None, opts: Optional[MergeOptions] = None):
    """comerge::merge_parallel (parallel.hpp:304-317): merges a and b stably
    into out and reports per-worker block sizes and co-rank iterations for
    the reference's `workers`-way output partition.  Only the default
    ordering is supported (`less` must be None)."""
    if less is not None:
        raise TypeError("merge_parallel: only the default std::less<> ordering runs on the device")
    return _merge_parallel("merge_parallel", a, b, out, workers, opts, False)


def merge_parallel_synced(a, b, out, workers: int, less=None,
                          opts: Optional[MergeOptions] = None):
    """comerge::merge_parallel_synced (parallel.hpp:323-336)."""
    if less is not None:
        raise TypeError("merge_parallel_synced: only the default ordering runs on the device")
    return _merge_parallel("merge_parallel_synced", a, b, out, workers, opts, True)


@dataclass
class BlockAssignment:
    """comerge::block_assignment (parallel.hpp:70-84)."""
    worker: int = 0
    out_begin: int = 0
    out_end: int = 0
    a_begin: int = 0
    a_end: int = 0
    b_begin: int = 0
    b_end: int = 0

    def as_tuple(self):
        return (self.worker, self.out_begin, self.out_end, self.a_begin, self.a_end,
                self.b_begin, self.b_end)


def plan(a, b, workers: int):
    """comerge::plan (parallel.hpp:94-115): per-worker assignments from two
    independent co-ranks per block, computed in one device batch."""
    if workers <= 0:
        raise ValueError("plan: worker count must be positive")
    suf = _suffix(a)
    if _suffix(b) != suf:
        raise TypeError("plan: a and b must share one dtype")
    raw = np.zeros(7 * workers, np.uint64)
    if _is_torch(a) and a.is_cuda:
        torch.cuda.current_stream(a.device).synchronize()
    with _on(a):
        N.check(getattr(N.lib, f"comerge_plan_{suf}")(_ptr(a), _len(a), _ptr(b), _len(b), workers,
                                                       C.c_void_p(raw.ctypes.data)))
    return [BlockAssignment(*(int(x) for x in raw[7 * r:7 * r + 7])) for r in range(workers)]


def merge_pairs(a_keys, a_vals, b_keys, b_vals, out_keys=None, out_vals=None, workspace=None):
    """Key-value stable merge on the device (uint32 payload moves with its key)."""
    suf = _suffix(a_keys)
    total = _len(a_keys) + _len(b_keys)
    if out_keys is None:
        out_keys = _empty_like_merge(a_keys, total)
    if out_vals is None:
        out_vals = _empty_like_merge(a_vals, total)
    if _len(a_vals) != _len(a_keys) or _len(b_vals) != _len(b_keys):
        raise ValueError("merge_pairs: payload length must equal key length")
    _check_out("merge_pairs", a_keys, b_keys, out_keys)
    _check_out("merge_pairs", a_vals, b_vals, out_vals)
    if _is_torch(a_keys) and a_keys.is_cuda:
        wsp, wsb = _ws(workspace)
        with _on(a_keys):
            N.check(getattr(N.lib, f"comerge_cuda_merge_pairs_{suf}")(
                _ptr(a_keys), _ptr(a_vals), _len(a_keys), _ptr(b_keys), _ptr(b_vals),
                _len(b_keys), _ptr(out_keys), _ptr(out_vals), wsp, wsb, _stream(a_keys)))
    else:
        rep = N.MergeReport()
        N.check(getattr(N.lib, f"comerge_merge_parallel_pairs_{suf}")(
            _ptr(a_keys), _ptr(a_vals), _len(a_keys), _ptr(b_keys), _ptr(b_vals), _len(b_keys),
            _ptr(out_keys), _ptr(out_vals), total, 1, C.byref(rep)))
    return out_keys, out_vals


# ------------------------------------------------------------ records

_REC_SUFFIX = {"int32": "i32", "uint32": "u32", "uint64": "u64"}
_REC_SIZE = {"i32": 8, "u32": 8, "u64": 16}


def record_dtype(key_dtype, record_bytes=None):
    """numpy dtype of one key-value record (comerge_rec_* in
    include/comerge_cuda.h): the key at offset 0, a uint32 `val`, and for
    uint64 keys a uint32 `pad` (the C layout of {uint64_t key; uint32_t val;}).
    record_bytes=12 (32-bit keys): the reference's tagged<int32_t> layout
    (comerge_rec12_*: key, `origin` byte + 3 padding bytes, uint32 `index`)."""
    name = _dtype_name_of(key_dtype)
    if record_bytes == 12:
        if name not in ("int32", "uint32"):
            raise TypeError("records: 12-byte records have 32-bit keys")
        return np.dtype({"names": ["key", "origin", "index"],
                         "formats": [np.dtype(name), np.uint8, np.uint32],
                         "offsets": [0, 4, 8], "itemsize": 12})
    if name == "uint64":
        return np.dtype({"names": ["key", "val", "pad"], "formats": [np.uint64, np.uint32, np.uint32],
                         "offsets": [0, 8, 12], "itemsize": 16})
    if name not in ("int32", "uint32"):
        raise TypeError(f"records: unsupported key dtype {name} (int32, uint32, uint64)")
    return np.dtype([("key", np.dtype(name)), ("val", np.uint32)])


def _dtype_name_of(dtype):
    if torch is not None and isinstance(dtype, torch.dtype):
        return str(dtype).replace("torch.", "")
    return np.dtype(dtype).name


def _rec_count(x, size):
    nbytes = int(x.numel() * x.element_size()) if _is_torch(x) else int(x.nbytes)
    if nbytes % size:
        raise ValueError(f"records: buffer of {nbytes} bytes is not a whole number of "
                         f"{size}-byte records")
    return nbytes // size


def records_workspace_bytes(m: int, n: int, key_dtype, record_bytes=None) -> int:
    suf = _REC_SUFFIX[_dtype_name_of(key_dtype)]
    if record_bytes == 12:
        return int(N.lib.comerge_cuda_records12_workspace_bytes(m, n))
    return int(N.lib.comerge_cuda_records_workspace_bytes(m, n, _KIND[suf]))


def _rec_abi(suf, size):
    """(device, host) entry-point names of suf's records of `size` bytes."""
    if size == 12:
        if suf == "u64":
            raise TypeError("records: 12-byte records have 32-bit keys")
        return f"comerge_cuda_merge_records12_{suf}", f"comerge_merge_parallel_records12_{suf}"
    if size != _REC_SIZE[suf]:
        raise TypeError(f"records: {suf} keys take {_REC_SIZE[suf]}-byte (or 12-byte) records")
    return f"comerge_cuda_merge_records_{suf}", f"comerge_merge_parallel_records_{suf}"


def merge_records(a, b, out=None, key_dtype=None, workers: int = 1, workspace=None,
                  record_bytes=None):
    """Stable merge of key-value records by key alone -- the reference's own
    key-value call shape: merge_parallel<T>(a, b, out, workers, key_less) over
    {key, val} structs (tagged<K> / tagged_key_less, oracle.hpp:22-37;
    parallel.hpp:304-317).  Ties keep A first, then input order; every record
    is copied whole (payload and padding bytes).

    Host: numpy structured arrays of record_dtype(key[, 12]) (synchronous;
    returns (out, MergeReport)).  Device: CUDA tensors of any dtype holding
    whole records (e.g. int64 of shape (n, 2) for uint64-key records),
    `key_dtype` given, `record_bytes` 12 for the tagged<int32_t> layout
    (asynchronous on the current stream; returns out)."""
    if _is_torch(a) and a.is_cuda:
        if key_dtype is None:
            raise TypeError("merge_records: key_dtype is required for device tensors")
        suf = _REC_SUFFIX[_dtype_name_of(key_dtype)]
        size = record_bytes or _REC_SIZE[suf]
        dev_fn, _ = _rec_abi(suf, size)
        m, n = _rec_count(a, size), _rec_count(b, size)
        if out is None:
            out = torch.empty((m + n) * size // a.element_size(), dtype=a.dtype, device=a.device)
        if _rec_count(out, size) != m + n:
            raise ValueError("merge_records: output length must equal |a| + |b|")
        wsp, wsb = _ws(workspace)
        with _on(a):
            N.check(getattr(N.lib, dev_fn)(_ptr(a), m, _ptr(b), n, _ptr(out), wsp, wsb,
                                           _stream(a)))
        return out
    kd = a.dtype["key"] if a.dtype.names else key_dtype
    suf = _REC_SUFFIX[_dtype_name_of(kd)]
    size = record_bytes or a.dtype.itemsize
    _, host_fn = _rec_abi(suf, size)
    if a.dtype.itemsize != size or b.dtype != a.dtype:
        raise TypeError(f"merge_records: a and b must be {size}-byte records of one dtype")
    m, n = len(a), len(b)
    if out is None:
        out = np.empty(m + n, dtype=a.dtype)
    if workers <= 0:
        raise ValueError("merge_parallel: worker count must be positive")
    rep = N.MergeReport()
    bs = np.zeros(workers, np.uint64)
    its = np.zeros(2 * workers, np.uint32)
    N.check(getattr(N.lib, host_fn)(
        _ptr(a), m, _ptr(b), n, _ptr(out), len(out), workers, 0, C.byref(rep),
        C.c_void_p(bs.ctypes.data), C.c_void_p(its.ctypes.data)))
    return out, MergeReport(m=rep.m, n=rep.n, workers=rep.workers, wall_ns=rep.wall_ns,
                            block_sizes=[int(x) for x in bs], corank_iterations=[int(x) for x in its],
                            e2e_ns=rep.e2e_ns, h2d_bytes=rep.h2d_bytes, d2h_bytes=rep.d2h_bytes,
                            tiles=rep.tiles)


def _rec_info(x, key_dtype, record_bytes):
    """(suffix, record size, record count) of a record array: a numpy
    structured array of record_dtype(), or any buffer of whole records with
    `key_dtype` (and `record_bytes` when not the default size) given."""
    if not _is_torch(x) and x.dtype.names:
        kd, size = x.dtype["key"], record_bytes or x.dtype.itemsize
        if x.dtype.itemsize != size:
            raise TypeError(f"records: the array holds {x.dtype.itemsize}-byte records, not {size}")
    else:
        if key_dtype is None:
            raise TypeError("records: key_dtype is required for unstructured buffers")
        kd = key_dtype
        size = record_bytes or _REC_SIZE[_REC_SUFFIX[_dtype_name_of(kd)]]
    return _REC_SUFFIX[_dtype_name_of(kd)], size, _rec_count(x, size)


def co_rank_records(target: int, a, b, key_dtype=None, record_bytes=None,
                    stats: Optional[CoRankStats] = None):
    """comerge::co_rank over records with a key-only less (corank.hpp:128-133
    instantiated as in corank_test.cpp:205-214): the split, iterations and
    comparisons of the records' key arrays.  Host or device buffers."""
    suf, size, m = _rec_info(a, key_dtype, record_bytes)
    n = _rec_info(b, key_dtype, record_bytes)[2]
    if target < 0:
        raise IndexError("co_rank: rank out of range (exceeds m+n)")
    j, k, it, cmp = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_uint32()
    with _on(a):
        N.check(getattr(N.lib, f"comerge_co_rank_records_{suf}")(
            int(target), _ptr(a), m, _ptr(b), n, size, C.byref(j), C.byref(k), C.byref(it),
            C.byref(cmp)))
    if stats is not None:
        stats.iterations, stats.comparisons = it.value, cmp.value
    return (j.value, k.value)


def co_rank_batch_records(ranks, a, b, key_dtype, record_bytes=None, with_stats: bool = False):
    """Device batch of co-ranks over record arrays (see co_rank_batch)."""
    suf, size, m = _rec_info(a, key_dtype, record_bytes)
    n = _rec_info(b, key_dtype, record_bytes)[2]
    q = int(ranks.numel())
    j = torch.empty(q, dtype=torch.uint64, device=a.device)
    it = torch.empty(q, dtype=torch.uint32, device=a.device) if with_stats else None
    cmp = torch.empty(q, dtype=torch.uint32, device=a.device) if with_stats else None
    with _on(a):
        N.check(getattr(N.lib, f"comerge_cuda_co_rank_batch_records_{suf}")(
            _ptr(ranks), q, _ptr(a), m, _ptr(b), n, size, _ptr(j), _ptr(it), _ptr(cmp),
            _stream(a)))
    return (j, it, cmp) if with_stats else j


def plan_records(a, b, workers: int, key_dtype=None, record_bytes=None):
    """comerge::plan over records with a key-only less (parallel.hpp:94-115)."""
    if workers <= 0:
        raise ValueError("plan: worker count must be positive")
    suf, size, m = _rec_info(a, key_dtype, record_bytes)
    n = _rec_info(b, key_dtype, record_bytes)[2]
    raw = np.zeros(7 * workers, np.uint64)
    if _is_torch(a) and a.is_cuda:
        torch.cuda.current_stream(a.device).synchronize()
    with _on(a):
        N.check(getattr(N.lib, f"comerge_plan_records_{suf}")(
            _ptr(a), m, _ptr(b), n, size, workers, C.c_void_p(raw.ctypes.data)))
    return [BlockAssignment(*(int(x) for x in raw[7 * r:7 * r + 7])) for r in range(workers)]


def merge_parallel_records(a, b, out, workers: int, key_dtype=None, record_bytes=None,
                           opts: Optional[MergeOptions] = None, synced: bool = False):
    """comerge::merge_parallel / merge_parallel_synced over records with a
    key-only less and the full report (merge_options::count_comparisons
    included; parallel.hpp:304-336).  Synchronous; host or device buffers."""
    suf, size, m = _rec_info(a, key_dtype, record_bytes)
    n = _rec_info(b, key_dtype, record_bytes)[2]
    out_len = _rec_info(out, key_dtype, record_bytes)[2]
    if workers < 0:
        raise ValueError("merge_parallel: worker count must be positive")
    count = bool(opts is not None and opts.count_comparisons)
    rep = N.MergeReport()
    bs = np.zeros(max(workers, 1), np.uint64)
    its = np.zeros(2 * max(workers, 1), np.uint32)
    cmp = C.c_uint64(0)
    mo = N.MergeOptions(int(synced), int(count))
    if _is_torch(out) and out.is_cuda:
        torch.cuda.current_stream(out.device).synchronize()
    with _on(out if _is_torch(out) and out.is_cuda else a):
        N.check(getattr(N.lib, f"comerge_merge_parallel_records_ex_{suf}")(
            _ptr(a), m, _ptr(b), n, _ptr(out), out_len, size, workers, C.byref(mo), C.byref(rep),
            C.c_void_p(bs.ctypes.data), C.c_void_p(its.ctypes.data), C.byref(cmp)))
    return MergeReport(
        m=rep.m, n=rep.n, workers=rep.workers, wall_ns=rep.wall_ns,
        block_sizes=[int(x) for x in bs[:workers]],
        corank_iterations=[int(x) for x in its[:(workers if synced else 2 * workers)]],
        comparisons=int(cmp.value) if count else None,
        e2e_ns=rep.e2e_ns, h2d_bytes=rep.h2d_bytes, d2h_bytes=rep.d2h_bytes, tiles=rep.tiles)


def merge_segmented(a, a_off, b, b_off, out=None, workspace=None, report=False):
    """Merge every pair s (a[a_off[s]:a_off[s+1]], b[b_off[s]:b_off[s+1]]) into
    out[a_off[s]+b_off[s]:...]: device tensors in one asynchronous launch;
    host (numpy) arrays synchronously through a chunked H2D / merge / D2H
    pipeline (comerge_merge_segmented_host_*; `report=True` also returns the
    MergeReport).  The reference has no batched call: its equivalent is a
    loop of comerge::stable_merge over the pairs (merge.hpp:52-68)."""
    suf = _suffix(a)
    if suf == "u64":
        raise TypeError("merge_segmented: int32 / uint32 keys")
    nseg = int(_len(a_off)) - 1
    if out is None:
        out = _empty_like_merge(a, _len(a) + _len(b))
    _check_out("merge_segmented", a, b, out)
    if not (_is_torch(a) and a.is_cuda):
        rep = N.MergeReport()
        with _on(out):
            N.check(getattr(N.lib, f"comerge_merge_segmented_host_{suf}")(
                _ptr(a), _ptr(a_off), _len(a), _ptr(b), _ptr(b_off), _len(b), max(nseg, 0),
                _ptr(out), _len(out), C.byref(rep)))
        if report:
            return out, MergeReport(m=rep.m, n=rep.n, workers=rep.workers, wall_ns=rep.wall_ns,
                                    e2e_ns=rep.e2e_ns, h2d_bytes=rep.h2d_bytes,
                                    d2h_bytes=rep.d2h_bytes, tiles=rep.tiles)
        return out
    wsp, wsb = _ws(workspace)
    with _on(a):
        N.check(getattr(N.lib, f"comerge_cuda_merge_segmented_{suf}")(
            _ptr(a), _ptr(a_off), _len(a), _ptr(b), _ptr(b_off), _len(b), max(nseg, 0),
            _ptr(out), wsp, wsb, _stream(a)))
    return out


def sort_workspace_bytes(n, dtype):
    """Workspace for sort() of n keys of `dtype` (CUB-style query)."""
    name = str(dtype).replace("torch.", "") if torch is not None and isinstance(dtype, torch.dtype) \
        else np.dtype(dtype).name
    return int(N.lib.comerge_cuda_sort_workspace_bytes(int(n), _KIND[_SUFFIX[name]]))


def sort(keys, out=None, workspace=None):
    """Stable merge sort of a device tensor of int32 / uint32 / uint64 keys
    (block-sorted runs, then merge passes of the pipeline).
    ``out`` may be ``keys`` itself (in place)."""
    if not (_is_torch(keys) and keys.is_cuda):
        raise TypeError("sort: keys must be a CUDA tensor (there is no host path)")
    suf = _suffix(keys)
    if out is None:
        out = _empty_like_merge(keys, _len(keys))
    if _len(out) != _len(keys):
        raise ValueError("sort: output length must equal the input length")
    wsp, wsb = _ws(workspace)
    with _on(keys):
        N.check(getattr(N.lib, f"comerge_cuda_sort_keys_{suf}")(
            _ptr(keys), _len(keys), _ptr(out), wsp, wsb, _stream(keys)))
    return out


def sort_pairs(keys, vals, out_keys=None, out_vals=None, workspace=None):
    """Stable key-value merge sort of device tensors (uint32 payloads move
    with their keys; equal keys keep their input order)."""
    if not (_is_torch(keys) and keys.is_cuda):
        raise TypeError("sort_pairs: keys must be a CUDA tensor (there is no host path)")
    suf = _suffix(keys)
    if _len(vals) != _len(keys):
        raise ValueError("sort_pairs: payload length must equal key length")
    if out_keys is None:
        out_keys = _empty_like_merge(keys, _len(keys))
    if out_vals is None:
        out_vals = _empty_like_merge(vals, _len(vals))
    if _len(out_keys) != _len(keys) or _len(out_vals) != _len(keys):
        raise ValueError("sort_pairs: output length must equal the input length")
    if workspace is None:
        wsp, wsb = None, 0
    else:
        wsp, wsb = _ws(workspace)
    with _on(keys):
        N.check(getattr(N.lib, f"comerge_cuda_sort_pairs_{suf}")(
            _ptr(keys), _ptr(vals), _len(keys), _ptr(out_keys), _ptr(out_vals), wsp, wsb,
            _stream(keys)))
    return out_keys, out_vals


def sort_pairs_workspace_bytes(n, dtype):
    name = str(dtype).replace("torch.", "") if torch is not None and isinstance(dtype, torch.dtype) \
        else np.dtype(dtype).name
    return int(N.lib.comerge_cuda_sort_pairs_workspace_bytes(int(n), _KIND[_SUFFIX[name]]))


def merge_pieces(a_pieces, b_pieces, out_begin: int, out_end: int, out=None, workspace=None,
                 a_val_pieces=None, b_val_pieces=None, out_vals=None):
    """Output ranks [out_begin, out_end) of stable_merge(cat(a_pieces),
    cat(b_pieces)) in one device launch, without concatenating: the pieces may
    live on other GPUs (peer tensors opened over CUDA IPC / NVLink).  Every
    piece but the last must hold a multiple of 16 bytes (and, with uint32
    payload pieces cut like their keys, a multiple of 4 elements); all 16-byte
    aligned.  Returns out (keys) or (out, out_vals)."""
    if not a_pieces or not b_pieces or len(a_pieces) > 8 or len(b_pieces) > 8:
        raise ValueError("merge_pieces: 1 to 8 pieces per input")
    pairs = a_val_pieces is not None or b_val_pieces is not None
    if pairs and (a_val_pieces is None or b_val_pieces is None or
                  len(a_val_pieces) != len(a_pieces) or len(b_val_pieces) != len(b_pieces)):
        raise ValueError("merge_pieces: one payload piece per key piece")
    suf = _suffix(a_pieces[0])
    for t in list(a_pieces) + list(b_pieces):
        if not (_is_torch(t) and t.is_cuda) or _suffix(t) != suf:
            raise TypeError("merge_pieces: pieces must be CUDA tensors of one key dtype")
    dev_ = torch.cuda.current_device()
    if out is None:
        out = torch.empty(out_end - out_begin, dtype=a_pieces[0].dtype, device=dev_)
    if _len(out) != out_end - out_begin:
        raise ValueError("merge_pieces: output length must equal out_end - out_begin")

    def ptrs(ts):
        return (C.c_void_p * len(ts))(*[t.data_ptr() if t.numel() else 0 for t in ts])

    al = (C.c_uint64 * len(a_pieces))(*[t.numel() for t in a_pieces])
    bl = (C.c_uint64 * len(b_pieces))(*[t.numel() for t in b_pieces])
    wsp, wsb = _ws(workspace)
    if not pairs:
        with _on(out):
            N.check(getattr(N.lib, f"comerge_cuda_merge_keys_pieces_{suf}")(
                ptrs(a_pieces), al, len(a_pieces), ptrs(b_pieces), bl, len(b_pieces), out_begin,
                out_end, _ptr(out), wsp, wsb, _stream(out)))
        return out
    for v, k in zip(list(a_val_pieces) + list(b_val_pieces), list(a_pieces) + list(b_pieces)):
        if _len(v) != _len(k):
            raise ValueError("merge_pieces: payload length must equal key length")
    if out_vals is None:
        out_vals = torch.empty(out_end - out_begin, dtype=torch.uint32, device=dev_)
    with _on(out):
        N.check(getattr(N.lib, f"comerge_cuda_merge_pairs_pieces_{suf}")(
            ptrs(a_pieces), ptrs(a_val_pieces), al, len(a_pieces), ptrs(b_pieces),
            ptrs(b_val_pieces), bl, len(b_pieces), out_begin, out_end, _ptr(out), _ptr(out_vals),
            wsp, wsb, _stream(out)))
    return out, out_vals
