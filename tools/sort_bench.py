"""Time the GPU merge sort (comerge_cuda_sort_keys_*) against torch.sort
(stable=True; CUB radix) on the same device keys.  L2 flushed between reps."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1303_4312_b200 as P  # noqa: E402
import paper_1303_4312_b200._native as N  # noqa: E402


def keys(n, dt, width):
    raw = torch.empty(n, dtype=torch.int64, device="cuda")
    N.check(N.tk().comerge_testkit_generate_raw(3, 0, n, width, raw.data_ptr(), None), True)
    return raw.to(dt)


def timeit(fn, reps=10):
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device="cuda")
    ts = []
    for r in range(reps + 2):
        flush.fill_(r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for n, dt, width in ((1 << 20, torch.int32, 1 << 31), (1 << 24, torch.int32, 1 << 31),
                     (1 << 26, torch.int32, 1 << 31), (1 << 26, torch.int32, 16),
                     (1 << 26, torch.int64, 1 << 62)):
    k = keys(n, dt, width)
    if dt == torch.int64:
        k = k.view(torch.uint64)
    out = torch.empty_like(k)
    ws = torch.empty(P.sort_workspace_bytes(n, k.dtype), dtype=torch.uint8, device="cuda")
    t_ours = timeit(lambda: P.sort(k, out=out, workspace=ws))
    kk = k.view(torch.int64) if k.dtype == torch.uint64 else k
    t_torch = timeit(lambda: torch.sort(kk, stable=True))
    ref = torch.sort(kk, stable=True).values
    ok = torch.equal(out.view(kk.dtype), ref) if k.dtype != torch.uint64 else None
    print(f"n=2^{n.bit_length() - 1} {str(k.dtype):13s} width {width:>20d}: merge sort {t_ours:7.3f} ms "
          f"({n / t_ours / 1e6:6.2f} G keys/s)  torch.sort(stable) {t_torch:7.3f} ms  equal={ok}")

# key-value (uint32 payload) sorts
for n, dt, width in ((1 << 24, torch.int32, 1 << 31), (1 << 26, torch.int32, 1 << 31),
                     (1 << 26, torch.int32, 16), (1 << 26, torch.int64, 1 << 62)):
    k = keys(n, dt, width)
    v = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    ok, ov = torch.empty_like(k), torch.empty_like(v)
    ku = k.view(torch.uint64) if dt == torch.int64 else k  # uint64 keys (values < 2^63)
    oku = ok.view(torch.uint64) if dt == torch.int64 else ok
    ws = torch.empty(P.sort_pairs_workspace_bytes(n, ku.dtype), dtype=torch.uint8, device="cuda")
    t_ours = timeit(lambda: P.sort_pairs(ku, v, out_keys=oku, out_vals=ov, workspace=ws))
    t_torch = timeit(lambda: torch.sort(k, stable=True))  # values + int64 indices
    ref = torch.sort(k, stable=True)
    equal = torch.equal(ok, ref.values) and torch.equal(ov.view(torch.int32).long(), ref.indices)
    print(f"pairs n=2^{n.bit_length() - 1} {str(ku.dtype)[6:]} width {width:>11d}: merge sort {t_ours:7.3f} ms "
          f"({n / t_ours / 1e6:6.2f} G pairs/s)  torch.sort(stable, indices) {t_torch:7.3f} ms  "
          f"equal={equal}")
