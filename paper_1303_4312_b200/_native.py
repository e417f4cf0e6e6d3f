"""ctypes binding of libcomerge_cuda.so (the C ABI in include/comerge_cuda.h).

The product has no CPU fallback: if the in-tree shared object is missing or
fails to load, importing this module raises.  Build it with `make` (or
`__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.environ.get("COMERGE_LIB_PATH") or os.path.join(PKG_DIR, "lib", "libcomerge_cuda.so")
# test / bench infrastructure (seeded generators, checkers): a separate library
TESTKIT_PATH = os.path.join(PKG_DIR, "lib", "libcomerge_cuda_testkit.so")
HEADERS = [os.path.join(REPO_DIR, "include", "comerge_cuda.h")]
TESTKIT_HEADERS = [os.path.join(REPO_DIR, "include", "comerge_cuda_testkit.h")]

OK, E_INVALID, E_RANGE, E_LENGTH, E_CUDA = 0, 1, 2, 3, 4
KEY_I32, KEY_U32, KEY_U64 = 0, 1, 2

_p = C.c_void_p
_sz = C.c_size_t
_u64 = C.c_uint64
_i = C.c_int


class MergeReport(C.Structure):
    """struct comerge_merge_report (include/comerge_cuda.h)."""
    _fields_ = [("m", _u64), ("n", _u64), ("workers", _u64), ("wall_ns", _u64),
                ("e2e_ns", _u64), ("h2d_bytes", _u64), ("d2h_bytes", _u64), ("tiles", _u64)]


class MergeOptions(C.Structure):
    """comerge_merge_options (include/comerge_cuda.h)."""
    _fields_ = [("synced", C.c_int), ("count_comparisons", C.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libcomerge_cuda.so not built at {LIB_PATH}; run `make` in {REPO_DIR} "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    lib.comerge_cuda_last_error.restype = C.c_char_p
    lib.comerge_cuda_abi_version.restype = _i
    lib.comerge_cuda_merge_workspace_bytes.argtypes = [_sz, _sz, _i, _i]
    lib.comerge_cuda_merge_workspace_bytes.restype = _sz
    lib.comerge_cuda_segmented_workspace_bytes.argtypes = [_sz, _sz, _i]
    lib.comerge_cuda_segmented_workspace_bytes.restype = _sz
    for suf in ("i32", "u32", "u64"):
        getattr(lib, f"comerge_cuda_merge_keys_{suf}").argtypes = [_p, _sz, _p, _sz, _p, _p, _sz, _p]
        getattr(lib, f"comerge_cuda_merge_pairs_{suf}").argtypes = [
            _p, _p, _sz, _p, _p, _sz, _p, _p, _p, _sz, _p]
        getattr(lib, f"comerge_cuda_co_rank_batch_{suf}").argtypes = [
            _p, _sz, _p, _sz, _p, _sz, _p, _p, _p, _p]
        getattr(lib, f"comerge_merge_parallel_{suf}").argtypes = [
            _p, _sz, _p, _sz, _p, _sz, _sz, _i, C.POINTER(MergeReport), _p, _p]
        getattr(lib, f"comerge_merge_parallel_ex_{suf}").argtypes = [
            _p, _p, _sz, _p, _p, _sz, _p, _p, _sz, _sz, C.POINTER(MergeOptions),
            C.POINTER(MergeReport), _p, _p, C.POINTER(_u64)]
        getattr(lib, f"comerge_merge_parallel_pairs_{suf}").argtypes = [
            _p, _p, _sz, _p, _p, _sz, _p, _p, _sz, _sz, C.POINTER(MergeReport)]
        getattr(lib, f"comerge_plan_{suf}").argtypes = [_p, _sz, _p, _sz, _sz, _p]
        getattr(lib, f"comerge_cuda_merge_keys_pieces_{suf}").argtypes = [
            _p, _p, _i, _p, _p, _i, _u64, _u64, _p, _p, _sz, _p]
        getattr(lib, f"comerge_cuda_merge_pairs_pieces_{suf}").argtypes = [
            _p, _p, _p, _i, _p, _p, _p, _i, _u64, _u64, _p, _p, _p, _sz, _p]
        getattr(lib, f"comerge_co_rank_{suf}").argtypes = [
            _u64, _p, _sz, _p, _sz, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(C.c_uint32),
            C.POINTER(C.c_uint32)]
    lib.comerge_cuda_records_workspace_bytes.argtypes = [_sz, _sz, _i]
    lib.comerge_cuda_records_workspace_bytes.restype = _sz
    for suf in ("i32", "u32", "u64"):
        getattr(lib, f"comerge_cuda_merge_records_{suf}").argtypes = [_p, _sz, _p, _sz, _p, _p,
                                                                      _sz, _p]
        getattr(lib, f"comerge_merge_parallel_records_{suf}").argtypes = [
            _p, _sz, _p, _sz, _p, _sz, _sz, _i, C.POINTER(MergeReport), _p, _p]
        # records by run-time size: co_rank / plan / batched co-rank / full report
        getattr(lib, f"comerge_co_rank_records_{suf}").argtypes = [
            _u64, _p, _sz, _p, _sz, _sz, C.POINTER(_u64), C.POINTER(_u64),
            C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        getattr(lib, f"comerge_plan_records_{suf}").argtypes = [_p, _sz, _p, _sz, _sz, _sz, _p]
        getattr(lib, f"comerge_cuda_co_rank_batch_records_{suf}").argtypes = [
            _p, _sz, _p, _sz, _p, _sz, _sz, _p, _p, _p, _p]
        getattr(lib, f"comerge_merge_parallel_records_ex_{suf}").argtypes = [
            _p, _sz, _p, _sz, _p, _sz, _sz, _sz, C.POINTER(MergeOptions),
            C.POINTER(MergeReport), _p, _p, C.POINTER(_u64)]
    lib.comerge_cuda_records12_workspace_bytes.argtypes = [_sz, _sz]
    lib.comerge_cuda_records12_workspace_bytes.restype = _sz
    for suf in ("i32", "u32"):
        getattr(lib, f"comerge_cuda_merge_records12_{suf}").argtypes = [_p, _sz, _p, _sz, _p, _p,
                                                                        _sz, _p]
        getattr(lib, f"comerge_merge_parallel_records12_{suf}").argtypes = [
            _p, _sz, _p, _sz, _p, _sz, _sz, _i, C.POINTER(MergeReport), _p, _p]
    lib.comerge_cuda_sort_workspace_bytes.argtypes = [_sz, _i]
    lib.comerge_cuda_sort_workspace_bytes.restype = _sz
    lib.comerge_cuda_sort_pairs_workspace_bytes.argtypes = [_sz, _i]
    lib.comerge_cuda_sort_pairs_workspace_bytes.restype = _sz
    for suf in ("i32", "u32", "u64"):
        getattr(lib, f"comerge_cuda_sort_keys_{suf}").argtypes = [_p, _sz, _p, _p, _sz, _p]
        getattr(lib, f"comerge_cuda_sort_pairs_{suf}").argtypes = [_p, _p, _sz, _p, _p, _p, _sz,
                                                                   _p]
    for suf in ("i32", "u32"):
        getattr(lib, f"comerge_merge_segmented_host_{suf}").argtypes = [
            _p, _p, _sz, _p, _p, _sz, _sz, _p, _sz, C.POINTER(MergeReport)]
        getattr(lib, f"comerge_cuda_merge_segmented_{suf}").argtypes = [
            _p, _p, _sz, _p, _p, _sz, _sz, _p, _p, _sz, _p]
    lib.comerge_cuda_set_kernel_events.argtypes = [_p, _p]
    lib.comerge_cuda_set_kernel_events.restype = None
    lib.comerge_cuda_set_path.argtypes = [_i]
    lib.comerge_cuda_set_path.restype = None
    lib.comerge_cuda_last_path.restype = _i
    lib.comerge_cuda_set_host_mode.argtypes = [_i]
    lib.comerge_cuda_set_host_mode.restype = None
    lib.comerge_cuda_set_trace.argtypes = [_p]
    lib.comerge_cuda_set_trace.restype = None
    lib.comerge_cuda_set_tuning.argtypes = [_i, _i, _i]
    lib.comerge_cuda_set_tuning.restype = None
    lib.comerge_partition_output.argtypes = [_u64, _u64, _u64, C.POINTER(_u64)]
    return lib


lib = _load()
_tk = None


def tk():
    """The testkit library (libcomerge_cuda_testkit.so: seeded device
    generators and full-size checkers for tests and the bench), loaded on first
    use.  Not part of the merge path."""
    global _tk
    if _tk is None:
        if not os.path.exists(TESTKIT_PATH):
            raise ImportError(f"libcomerge_cuda_testkit.so not built at {TESTKIT_PATH}; run `make`")
        t = C.CDLL(TESTKIT_PATH)
        t.comerge_testkit_last_error.restype = C.c_char_p
        t.comerge_testkit_generate_raw.argtypes = [_u64, _u64, _sz, _u64, _p, _p]
        t.comerge_testkit_generate_runs.argtypes = [_i, _u64, _u64, _p, _sz, _sz, _u64, _p, _p]
        t.comerge_testkit_generate_sorted.argtypes = [_i, _u64, _u64, _sz, _u64, _p, _p]
        t.comerge_testkit_iota.argtypes = [_p, _sz, C.c_uint32, _p]
        t.comerge_testkit_fill_runs.argtypes = [_i, _sz, _u64, _u64, _p, _p]
        t.comerge_testkit_verify_pairs.argtypes = [_i, _p, _sz, _p, _sz, _p, _p, _p, _p]
        t.comerge_testkit_checksum.argtypes = [_i, _p, _sz, _p, _p]
        t.comerge_testkit_count_unsorted.argtypes = [_i, _p, _sz, _p, _p]
        t.comerge_testkit_cub_sort_bytes.argtypes = [_sz]
        t.comerge_testkit_cub_sort_bytes.restype = _sz
        t.comerge_testkit_cub_sort.argtypes = [_i, _p, _p, _p, _p, _sz, _p, _sz, _p]
        _tk = t
    return _tk


def declared_symbols(headers=None):
    """Every function name declared in the product header (or `headers`)."""
    names = []
    for h in headers or HEADERS:
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        names += re.findall(r"\b(comerge_\w+)\s*\(", text)
    return sorted(set(names))


def last_error() -> str:
    return lib.comerge_cuda_last_error().decode()


def check(rc: int, testkit: bool = False):
    """Map a status code onto the reference's exception types."""
    if rc == OK:
        return
    msg = (tk().comerge_testkit_last_error() if testkit else lib.comerge_cuda_last_error()).decode()
    if rc == E_INVALID:
        raise ValueError(msg)        # std::invalid_argument
    if rc == E_RANGE:
        raise IndexError(msg)        # std::out_of_range
    if rc == E_LENGTH:
        raise OverflowError(msg)     # std::length_error
    raise RuntimeError(msg)          # CUDA failure
