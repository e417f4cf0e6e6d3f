"""ctypes wrappers over the two CPU oracles (TEST INFRASTRUCTURE ONLY).

``Port``  wraps oracle/liboracle.so (C restatement, comerge_oracle.c).
``Ref``   wraps oracle/_ref/libcomerge_ref.so (the reference itself).

Arrays are numpy; key kinds follow the dtype: int32 -> 0, uint32 -> 1,
uint64 -> 2.  Errors map to the reference's exception types the same way the
product's Python mirror does (invalid_argument -> ValueError, out_of_range ->
IndexError, length_error -> OverflowError).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcomerge_ref.so")

KIND = {np.dtype(np.int32): 0, np.dtype(np.uint32): 1, np.dtype(np.uint64): 2}
DTYPE = {0: np.int32, 1: np.uint32, 2: np.uint64}

_p = C.c_void_p
_u64 = C.c_uint64
_u32p = C.POINTER(C.c_uint32)


def kind_of(arr) -> int:
    return KIND[np.dtype(arr.dtype)]


def ptr(arr):
    return None if arr is None else arr.ctypes.data_as(_p)


def _raise(code: int, msg: str):
    if code == 0:
        return
    if code == 1:
        raise ValueError(msg)
    if code == 2:
        raise IndexError(msg)
    if code == 3:
        raise OverflowError(msg)
    raise RuntimeError(msg)


class Port:
    """The C restatement (oracle/comerge_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        lib = C.CDLL(path)
        lib.oracle_co_rank.argtypes = [C.c_int, _u64, _p, _u64, _p, _u64, C.POINTER(_u64),
                                       C.POINTER(_u64), _u32p, _u32p]
        lib.oracle_partition_output.argtypes = [_u64, _u64, _u64, C.POINTER(_u64)]
        lib.oracle_merge_into.argtypes = [C.c_int, _p, _p, _u64, _p, _p, _u64, _p, _p]
        lib.oracle_merge_into.restype = None
        lib.oracle_merge_parallel.argtypes = [C.c_int, _p, _p, _u64, _p, _p, _u64, _p, _p, _u64,
                                              C.c_int, _p, _p]
        lib.oracle_merge_segmented.argtypes = [C.c_int, _p, _p, _p, _p, _u64, _p, C.c_int]
        lib.oracle_merge_sort.argtypes = [C.c_int, _p, _u64, _p]
        lib.oracle_merge_sort_pairs.argtypes = [C.c_int, _p, _p, _u64, _p, _p]
        lib.oracle_merge_report.argtypes = [C.c_int, _p, _u64, _p, _u64, _u64, C.c_int, _p, _p,
                                            C.POINTER(_u64)]
        lib.oracle_generate_sorted.argtypes = [C.c_int, _u64, _u64, _u64, _u64, _p]
        lib.oracle_generate_sorted.restype = None
        lib.oracle_generate_raw.argtypes = [_u64, _u64, _u64, _u64, _p]
        lib.oracle_generate_raw.restype = None
        lib.oracle_multiset_checksum.argtypes = [C.c_int, _p, _u64]
        lib.oracle_multiset_checksum.restype = _u64
        lib.oracle_mix64.argtypes = [_u64]
        lib.oracle_mix64.restype = _u64
        self.lib = lib

    def co_rank(self, target, a, b, stats=False):
        j, k, it, cmp = _u64(), _u64(), C.c_uint32(), C.c_uint32()
        rc = self.lib.oracle_co_rank(kind_of(a), target, ptr(a), len(a), ptr(b), len(b),
                                     C.byref(j), C.byref(k), C.byref(it), C.byref(cmp))
        _raise(rc, "co_rank: rank out of range (exceeds m+n)" if rc == 2 else "co_rank failed")
        if stats:
            return (j.value, k.value), (it.value, cmp.value)
        return (j.value, k.value)

    def partition_output(self, total, workers, r):
        out = _u64()
        rc = self.lib.oracle_partition_output(total, workers, r, C.byref(out))
        _raise(rc, "partition_output: worker count must be positive" if workers == 0
               else "partition_output: worker id out of range")
        return out.value

    def merge(self, a, b, av=None, bv=None):
        out = np.empty(len(a) + len(b), dtype=a.dtype)
        outv = None if av is None else np.empty(len(a) + len(b), dtype=np.uint32)
        self.lib.oracle_merge_into(kind_of(a), ptr(a), ptr(av), len(a), ptr(b), ptr(bv), len(b),
                                   ptr(out), ptr(outv))
        return out if av is None else (out, outv)

    def merge_parallel(self, a, b, workers, av=None, bv=None, threads=1):
        out = np.empty(len(a) + len(b), dtype=a.dtype)
        outv = None if av is None else np.empty(len(a) + len(b), dtype=np.uint32)
        bs = np.zeros(max(workers, 1), dtype=np.uint64)
        its = np.zeros(2 * max(workers, 1), dtype=np.uint32)
        rc = self.lib.oracle_merge_parallel(kind_of(a), ptr(a), ptr(av), len(a), ptr(b), ptr(bv),
                                            len(b), ptr(out), ptr(outv), workers, threads,
                                            ptr(bs), ptr(its))
        _raise(rc, "merge_parallel: worker count must be positive")
        return out, outv, bs, its

    def merge_segmented(self, a, a_off, b, b_off, threads=1):
        nseg = len(a_off) - 1
        out = np.empty(len(a) + len(b), dtype=a.dtype)
        rc = self.lib.oracle_merge_segmented(kind_of(a), ptr(a), ptr(a_off), ptr(b), ptr(b_off),
                                             nseg, ptr(out), threads)
        _raise(rc, "merge_segmented: offsets must be nondecreasing")
        return out

    def merge_report(self, a, b, workers, synced=False):
        """(block_sizes, corank_iterations, comparisons) of merge_parallel."""
        bs = np.zeros(max(workers, 1), dtype=np.uint64)
        its = np.zeros((1 if synced else 2) * max(workers, 1), dtype=np.uint32)
        cmp = _u64(0)
        rc = self.lib.oracle_merge_report(kind_of(a), ptr(a), len(a), ptr(b), len(b), workers,
                                          int(synced), ptr(bs), ptr(its), C.byref(cmp))
        _raise(rc, "merge_parallel: worker count must be positive")
        return bs, its, int(cmp.value)

    def merge_sort(self, keys):
        keys = np.ascontiguousarray(keys)
        out = np.empty_like(keys)
        rc = self.lib.oracle_merge_sort(kind_of(keys), ptr(keys), len(keys), ptr(out))
        if rc:
            raise MemoryError("oracle_merge_sort: allocation failed")
        return out

    def merge_sort_pairs(self, keys, vals):
        keys = np.ascontiguousarray(keys)
        vals = np.ascontiguousarray(vals, dtype=np.uint32)
        ok, ov = np.empty_like(keys), np.empty_like(vals)
        rc = self.lib.oracle_merge_sort_pairs(kind_of(keys), ptr(keys), ptr(vals), len(keys),
                                              ptr(ok), ptr(ov))
        if rc:
            raise MemoryError("oracle_merge_sort_pairs: allocation failed")
        return ok, ov

    def generate_sorted(self, dtype, seed, lane, length, width):
        out = np.empty(length, dtype=dtype)
        self.lib.oracle_generate_sorted(KIND[np.dtype(dtype)], seed, lane, length, width, ptr(out))
        return out

    def generate_raw(self, seed, lane, length, width):
        out = np.empty(length, dtype=np.uint64)
        self.lib.oracle_generate_raw(seed, lane, length, width, ptr(out))
        return out

    def checksum(self, keys):
        return int(self.lib.oracle_multiset_checksum(kind_of(keys), ptr(keys), len(keys)))


class RefReport(C.Structure):
    _fields_ = [("m", C.c_uint64), ("n", C.c_uint64), ("workers", C.c_uint64),
                ("wall_ns", C.c_uint64), ("comparisons", C.c_uint64),
                ("has_comparisons", C.c_int32), ("pad", C.c_int32)]


def tagged_dtype(kind: int):
    """numpy mirror of the reference's comerge::tagged<K> (oracle.hpp:22-27):
    key, origin byte (+ padding), uint32 index."""
    ks = 8 if DTYPE[kind] == np.uint64 else 4
    return np.dtype({"names": ["key", "origin", "index"],
                     "formats": [DTYPE[kind], np.uint8, np.uint32],
                     "offsets": [0, ks, ks + 4], "itemsize": ks + 8})


def kv_dtype(kind: int):
    """numpy mirror of ref_shim.cpp's kv_i32 / kv_u32 / kv_u64 structs."""
    return np.dtype([("key", DTYPE[kind]), ("val", np.uint32)], align=True)


class Ref:
    """The unmodified reference library (oracle/_ref/libcomerge_ref.so)."""

    def __init__(self, path: str = REF_SO):
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_hardware_concurrency.restype = C.c_uint
        lib.ref_report_size.restype = C.c_size_t
        lib.ref_kv_size.argtypes = [C.c_int]
        lib.ref_kv_size.restype = C.c_size_t
        lib.ref_co_rank.argtypes = [C.c_int, _u64, _p, C.c_size_t, _p, C.c_size_t,
                                    C.POINTER(_u64), C.POINTER(_u64), _u32p, _u32p]
        lib.ref_partition_output.argtypes = [C.c_size_t, C.c_size_t, C.c_size_t, C.POINTER(_u64)]
        lib.ref_stable_merge.argtypes = [C.c_int, _p, C.c_size_t, _p, C.c_size_t, _p, C.c_size_t]
        lib.ref_merge_parallel.argtypes = [C.c_int, _p, C.c_size_t, _p, C.c_size_t, _p,
                                           C.c_size_t, C.c_size_t, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(RefReport), _p, _p]
        lib.ref_merge_parallel_kv.argtypes = [C.c_int, _p, C.c_size_t, _p, C.c_size_t, _p,
                                              C.c_size_t, C.c_size_t, C.c_int, C.c_int,
                                              C.POINTER(RefReport), _p, _p]
        lib.ref_plan.argtypes = [C.c_int, _p, C.c_size_t, _p, C.c_size_t, C.c_size_t, _p]
        lib.ref_tagged_size.argtypes = [C.c_int]
        lib.ref_tagged_size.restype = C.c_size_t
        lib.ref_merge_parallel_tagged.argtypes = [C.c_int, _p, C.c_size_t, _p, C.c_size_t, _p,
                                                  C.c_size_t, C.c_size_t, C.c_int,
                                                  C.POINTER(RefReport)]
        lib.ref_merge_segmented.argtypes = [C.c_int, _p, _p, _p, _p, C.c_size_t, _p, C.c_int,
                                            C.POINTER(_u64)]
        lib.ref_oracle_merge_tagged.argtypes = [_p, C.c_size_t, _p, C.c_size_t, _p, _p, _p]
        lib.ref_generate.argtypes = [C.c_int, _u64, _u64, C.c_size_t, C.c_size_t, _p, _p]
        lib.ref_multiset_checksum.argtypes = [_p, C.c_size_t]
        lib.ref_multiset_checksum.restype = _u64
        assert lib.ref_report_size() == C.sizeof(RefReport)
        for k in (0, 1, 2):
            assert lib.ref_kv_size(k) == kv_dtype(k).itemsize
            assert lib.ref_tagged_size(k) == tagged_dtype(k).itemsize
        self.lib = lib

    def _check(self, rc):
        if rc:
            _raise(rc, self.lib.ref_last_error().decode())

    def hardware_concurrency(self) -> int:
        return int(self.lib.ref_hardware_concurrency())

    def co_rank(self, target, a, b, stats=False):
        j, k, it, cmp = _u64(), _u64(), C.c_uint32(), C.c_uint32()
        self._check(self.lib.ref_co_rank(kind_of(a), target, ptr(a), len(a), ptr(b), len(b),
                                         C.byref(j), C.byref(k), C.byref(it), C.byref(cmp)))
        if stats:
            return (j.value, k.value), (it.value, cmp.value)
        return (j.value, k.value)

    def partition_output(self, total, workers, r):
        out = _u64()
        self._check(self.lib.ref_partition_output(total, workers, r, C.byref(out)))
        return out.value

    def stable_merge(self, a, b, out_len=None):
        out = np.empty(len(a) + len(b) if out_len is None else out_len, dtype=a.dtype)
        self._check(self.lib.ref_stable_merge(kind_of(a), ptr(a), len(a), ptr(b), len(b),
                                              ptr(out), len(out)))
        return out

    def merge_parallel(self, a, b, workers, simulated=False, synced=False, count=False,
                       out=None):
        if out is None:
            out = np.empty(len(a) + len(b), dtype=a.dtype)
        rep = RefReport()
        bs = np.zeros(max(workers, 1), dtype=np.uint64)
        its = np.zeros(2 * max(workers, 1), dtype=np.uint32)
        self._check(self.lib.ref_merge_parallel(kind_of(a), ptr(a), len(a), ptr(b), len(b),
                                                ptr(out), len(out), workers, int(simulated),
                                                int(synced), int(count), C.byref(rep), ptr(bs),
                                                ptr(its)))
        return out, rep, bs, its

    def merge_parallel_tagged(self, a, b, workers, synced=False, out=None):
        """comerge::merge_parallel over the reference's tagged<K> with
        tagged_key_less; a / b: numpy arrays of tagged_dtype(kind)."""
        kind = KIND[np.dtype(a.dtype["key"])]
        if out is None:
            out = np.empty(len(a) + len(b), dtype=a.dtype)
        rep = RefReport()
        self._check(self.lib.ref_merge_parallel_tagged(kind, ptr(a), len(a), ptr(b), len(b),
                                                       ptr(out), len(out), workers, int(synced),
                                                       C.byref(rep)))
        return out, rep

    def merge_parallel_kv(self, a_aos, b_aos, workers, simulated=False, synced=False,
                          out=None):
        """a_aos / b_aos: numpy arrays of kv_dtype(kind)."""
        kind = KIND[np.dtype(a_aos.dtype["key"])]
        if out is None:
            out = np.empty(len(a_aos) + len(b_aos), dtype=a_aos.dtype)
        rep = RefReport()
        self._check(self.lib.ref_merge_parallel_kv(kind, ptr(a_aos), len(a_aos), ptr(b_aos),
                                                   len(b_aos), ptr(out), len(out), workers,
                                                   int(simulated), int(synced), C.byref(rep),
                                                   None, None))
        return out, rep

    def plan(self, a, b, workers):
        blocks = np.zeros((max(workers, 1), 7), dtype=np.uint64)
        self._check(self.lib.ref_plan(kind_of(a), ptr(a), len(a), ptr(b), len(b), workers,
                                      ptr(blocks)))
        return blocks

    def merge_segmented(self, a, a_off, b, b_off, threads=1, out=None):
        if out is None:
            out = np.empty(len(a) + len(b), dtype=a.dtype)
        wall = _u64()
        self._check(self.lib.ref_merge_segmented(kind_of(a), ptr(a), ptr(a_off), ptr(b),
                                                 ptr(b_off), len(a_off) - 1, ptr(out), threads,
                                                 C.byref(wall)))
        return out, wall.value

    def oracle_merge_tagged(self, a, b):
        n = len(a) + len(b)
        keys = np.empty(n, np.uint64)
        origin = np.empty(n, np.uint8)
        index = np.empty(n, np.uint32)
        self._check(self.lib.ref_oracle_merge_tagged(ptr(a), len(a), ptr(b), len(b), ptr(keys),
                                                     ptr(origin), ptr(index)))
        return keys, origin, index

    def generate(self, dist, seed, param, m, n):
        a = np.empty(m, np.uint64)
        b = np.empty(n, np.uint64)
        self._check(self.lib.ref_generate(dist, seed, param, m, n, ptr(a), ptr(b)))
        return a, b

    def checksum(self, keys):
        return int(self.lib.ref_multiset_checksum(ptr(keys), len(keys)))


def to_aos(keys, vals):
    kind = KIND[np.dtype(keys.dtype)]
    out = np.empty(len(keys), dtype=kv_dtype(kind))
    out["key"] = keys
    out["val"] = vals
    return out


def available_ref() -> bool:
    return os.path.exists(REF_SO)
