"""e2e of C2 with the host arrays as separate pinned tensors vs one pinned slab
(keys and payloads of a side adjacent: the library's two-row copy path)."""
import ctypes as C, os, sys, time, statistics
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_1303_4312_b200._native as N
inp = bench.make_inputs("C2", device=torch.device("cuda:0"))
m, n = inp["a"].numel(), inp["b"].numel()
tot = m + n
p = lambda t: C.c_void_p(t.data_ptr())
def run(a, av, b, bv, ok, ov, reps=6):
    rep = N.MergeReport()
    ts = []
    for r in range(reps):
        t0 = time.perf_counter()
        N.check(N.lib.comerge_merge_parallel_pairs_i32(p(a), p(av), m, p(b), p(bv), n, p(ok), p(ov), tot, 1, C.byref(rep)))
        if r: ts.append(time.perf_counter() - t0)
    return statistics.mean(ts) * 1e3
sep = {k: v.cpu().pin_memory() for k, v in inp.items()}
ok = torch.empty(tot, dtype=torch.int32).pin_memory(); ov = torch.empty(tot, dtype=torch.uint32).pin_memory()
print("separate pinned tensors: %.2f ms" % run(sep["a"], sep["av"], sep["b"], sep["bv"], ok, ov))
slab = torch.empty(2 * m + 2 * n, dtype=torch.int32).pin_memory()
a, av = slab[:m], slab[m:2 * m].view(torch.uint32)
b, bv = slab[2 * m:2 * m + n], slab[2 * m + n:].view(torch.uint32)
a.copy_(sep["a"]); av.copy_(sep["av"]); b.copy_(sep["b"]); bv.copy_(sep["bv"])
oslab = torch.empty(2 * tot, dtype=torch.int32).pin_memory()
ok2, ov2 = oslab[:tot], oslab[tot:].view(torch.uint32)
print("one pinned slab (2-row copies): %.2f ms" % run(a, av, b, bv, ok2, ov2))
assert torch.equal(ok2, ok) and torch.equal(ov2, ov)
for ch in (4, 6, 12):
    pass
