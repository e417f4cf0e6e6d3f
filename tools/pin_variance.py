"""Is the host-buffer (e2e) time a property of the pinned allocation?  C2's
shape through comerge_merge_parallel_pairs_i32, host buffers re-allocated
several times, each allocation timed over a few calls:
  torch  -- torch's pinned allocator (cudaHostAlloc)
  thp    -- 2 MB-aligned anonymous memory, madvise(MADV_HUGEPAGE), touched,
            then cudaHostRegister'ed
    python tools/pin_variance.py [C2|C4] [allocs] [calls]"""
import ctypes as C
import mmap
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1303_4312_b200._native as N  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
allocs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rt = C.CDLL("libcudart.so.12")
print("THP:", open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(),
      "defrag:", open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
dev = torch.device("cuda:0")
inp = bench.make_inputs(cfg, device=dev)
suf = {"int32": "i32", "uint64": "u64"}[bench.CONFIGS[cfg]["dtype"]]
fn = getattr(N.lib, f"comerge_merge_parallel_pairs_{suf}")
keep = []


def thp_empty(nbytes, dtype):
    H = 2 << 20
    size = (nbytes + H - 1) // H * H
    mm = mmap.mmap(-1, size + H, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = C.addressof(C.c_char.from_buffer(mm))
    off = (-base) % H
    mv = memoryview(mm)[off: off + size]
    mm.madvise(mmap.MADV_HUGEPAGE, off, size)
    arr = np.frombuffer(mv, dtype=np.uint8)
    arr[::4096] = 0  # touch
    assert rt.cudaHostRegister(C.c_void_p(base + off), C.c_size_t(size), 0) == 0
    keep.append((mm, mv, base + off))
    return torch.from_numpy(arr[:nbytes]).view(dtype)


def host_like(t, kind):
    if kind == "torch":
        return t.cpu().pin_memory()
    h = thp_empty(t.numel() * t.element_size(), t.dtype)
    h.copy_(t.cpu())
    return h


def alloc(kind):
    pin = {k: host_like(v, kind) for k, v in inp.items() if hasattr(v, "cpu")}
    total = inp["a"].numel() + inp["b"].numel()
    if kind == "torch":
        ok = torch.empty(total, dtype=inp["a"].dtype).pin_memory()
        ov = torch.empty(total, dtype=torch.uint32).pin_memory()
    else:
        ok = thp_empty(total * inp["a"].element_size(), inp["a"].dtype)
        ov = thp_empty(total * 4, torch.uint32)
    return pin, ok, ov, total


p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
rep = N.MergeReport()
for kind in ("torch", "thp", "torch", "thp"):
    for r in range(allocs):
        pin, ok, ov, total = alloc(kind)
        ts = []
        for _ in range(calls + 1):
            t0 = time.perf_counter()
            N.check(fn(p(pin["a"]), p(pin["av"]), pin["a"].numel(), p(pin["b"]), p(pin["bv"]),
                       pin["b"].numel(), p(ok), p(ov), total, 1, C.byref(rep)))
            ts.append(time.perf_counter() - t0)
        ts = ts[1:]
        print(f"{cfg} {kind:5s} alloc {r}: e2e ms median {1e3 * statistics.median(ts):7.2f} "
              f"min {1e3 * min(ts):7.2f} max {1e3 * max(ts):7.2f}", flush=True)
        del pin, ok, ov
    while keep:
        mm, mv, addr = keep.pop()
        rt.cudaHostUnregister(C.c_void_p(addr))
        mv.release()
        mm.close()
