"""Small merges through every device path, for compute-sanitizer runs
(memcheck / racecheck / synccheck): key and key-value pipeline merges, a
segmented batch, sorts, a pieced range merge and the host-buffer pipeline."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_1303_4312_b200 as P
from oracle.py import Port
port = Port()
dev = torch.device("cuda:0")
rng = np.random.default_rng(5)
m, n = 150_001, 120_007
a = np.sort(rng.integers(0, 40, m)).astype(np.int32)
b = np.sort(rng.integers(0, 40, n)).astype(np.int32)
av, bv = np.arange(m, dtype=np.uint32), np.arange(n, dtype=np.uint32) | np.uint32(1 << 31)
ta, tb = torch.from_numpy(a).to(dev), torch.from_numpy(b).to(dev)
ok, ov = P.merge_pairs(ta, torch.from_numpy(av).to(dev), tb, torch.from_numpy(bv).to(dev))
ks = P.stable_merge(ta, tb)
torch.cuda.synchronize()
ek, ev = port.merge(a, b, av, bv)
assert np.array_equal(ok.cpu().numpy(), ek) and np.array_equal(ov.cpu().numpy(), ev)
assert np.array_equal(ks.cpu().numpy(), ek)
la, lb = rng.integers(0, 900, 150), rng.integers(0, 900, 150)
sa = np.concatenate([np.sort(rng.integers(0, 1 << 20, x)) for x in la]).astype(np.int32)
sb = np.concatenate([np.sort(rng.integers(0, 1 << 20, x)) for x in lb]).astype(np.int32)
ao = np.concatenate([[0], np.cumsum(la)]).astype(np.uint64)
bo = np.concatenate([[0], np.cumsum(lb)]).astype(np.uint64)
so = P.merge_segmented(*(torch.from_numpy(x).to(dev) for x in (sa, ao, sb, bo)))
assert np.array_equal(so.cpu().numpy(), port.merge_segmented(sa, ao, sb, bo))
k = rng.integers(-500, 500, 70_001).astype(np.int32)
assert np.array_equal(P.sort(torch.from_numpy(k).to(dev)).cpu().numpy(), port.merge_sort(k))
v = np.arange(len(k), dtype=np.uint32)
sk, sv = P.sort_pairs(torch.from_numpy(k).to(dev), torch.from_numpy(v).to(dev))
ek2, ev2 = port.merge_sort_pairs(k, v)
assert np.array_equal(sk.cpu().numpy(), ek2) and np.array_equal(sv.cpu().numpy(), ev2)
out = np.empty(2_000_000, np.int32)
a2 = np.sort(rng.integers(0, 1 << 30, 1_000_000)).astype(np.int32)
b2 = np.sort(rng.integers(0, 1 << 30, 1_000_000)).astype(np.int32)
P.merge_parallel(a2, b2, out, 4)  # host buffers: the chunked pipeline
assert np.array_equal(out, port.merge(a2, b2))
print("sanitize_small: OK")
