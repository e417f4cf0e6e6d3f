"""Device-side seeded inputs and full-size verification (include/comerge_cuda_testkit.h).

Test / bench infrastructure: not on the merge path.  The generator reproduces
the reference's splitmix64 recipe (generate.cpp:17-29) on the GPU.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _native as N

_KIND = {torch.int32: N.KEY_I32, torch.uint32: N.KEY_U32, torch.uint64: N.KEY_U64}


def _stream(dev):
    return C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def generate_sorted(dtype, seed: int, lane: int, length: int, width: int, device="cuda"):
    """sorted(below(width) draws of stream(seed, lane)) as `dtype` (width 0: next())."""
    out = torch.empty(length, dtype=dtype, device=device)
    if length:
        N.check(N.tk().comerge_testkit_generate_sorted(_KIND[dtype], seed, lane, length, width,
                                                       C.c_void_p(out.data_ptr()),
                                                       _stream(out.device)), testkit=True)
    return out


def generate_raw(seed: int, lane: int, length: int, width: int, device="cuda"):
    """Unsorted accepted draws (uint64) of stream(seed, lane)."""
    out = torch.empty(length, dtype=torch.uint64, device=device)
    if length:
        N.check(N.tk().comerge_testkit_generate_raw(seed, lane, length, width,
                                                    C.c_void_p(out.data_ptr()),
                                                    _stream(out.device)), testkit=True)
    return out


def generate_runs(dtype, seed: int, lane: int, offsets, width: int):
    """Keys of stream(seed, lane), each run [offsets[s], offsets[s+1]) sorted."""
    total = int(offsets[-1].item())
    out = torch.empty(total, dtype=dtype, device=offsets.device)
    if total:
        N.check(N.tk().comerge_testkit_generate_runs(
            _KIND[dtype], seed, lane, C.c_void_p(offsets.data_ptr()), offsets.numel() - 1, total,
            width, C.c_void_p(out.data_ptr()), _stream(out.device)), testkit=True)
    return out


def fill_runs(length: int, run_len: int, dtype, offset: int = 0, device="cuda"):
    """Sorted keys (i + offset) // run_len of `dtype` on the device."""
    out = torch.empty(length, dtype=dtype, device=device)
    if length:
        N.check(N.tk().comerge_testkit_fill_runs(_KIND[dtype], length, run_len, offset,
                                                 C.c_void_p(out.data_ptr()),
                                                 _stream(out.device)), testkit=True)
    return out


def iota(length: int, tag: int, device="cuda"):
    """uint32 payloads i | tag (A: tag 0, B: tag 1<<31)."""
    out = torch.empty(length, dtype=torch.uint32, device=device)
    if length:
        N.check(N.tk().comerge_testkit_iota(C.c_void_p(out.data_ptr()), length, tag,
                                            _stream(out.device)), testkit=True)
    return out


def verify_pairs(a, b, out_keys, out_vals):
    """[unsorted, unstable, key mismatch, bad tag] counts; all 0 <=> exact stable merge."""
    counts = torch.zeros(4, dtype=torch.uint64, device=a.device)
    N.check(N.tk().comerge_testkit_verify_pairs(
        _KIND[a.dtype], C.c_void_p(a.data_ptr()), a.numel(), C.c_void_p(b.data_ptr()),
        b.numel(), C.c_void_p(out_keys.data_ptr()), C.c_void_p(out_vals.data_ptr()),
        C.c_void_p(counts.data_ptr()), _stream(a.device)), testkit=True)
    return [int(x) for x in counts.cpu().tolist()]


def checksum(keys):
    acc = torch.zeros(1, dtype=torch.uint64, device=keys.device)
    if keys.numel():
        N.check(N.tk().comerge_testkit_checksum(_KIND[keys.dtype], C.c_void_p(keys.data_ptr()),
                                                keys.numel(), C.c_void_p(acc.data_ptr()),
                                                _stream(keys.device)), testkit=True)
    return int(acc.cpu().view(torch.int64).item()) & (2**64 - 1)


def count_unsorted(keys):
    acc = torch.zeros(1, dtype=torch.uint64, device=keys.device)
    if keys.numel() > 1:
        N.check(N.tk().comerge_testkit_count_unsorted(_KIND[keys.dtype],
                                                      C.c_void_p(keys.data_ptr()), keys.numel(),
                                                      C.c_void_p(acc.data_ptr()),
                                                      _stream(keys.device)), testkit=True)
    return int(acc.cpu().view(torch.int64).item())
