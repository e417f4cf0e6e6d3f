"""Three stable pair sorts of 2^26 int32 keys + uint32 payloads (for ncu)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1303_4312_b200 as P
import paper_1303_4312_b200._native as N
n = 1 << 26
raw = torch.empty(n, dtype=torch.int64, device="cuda")
N.check(N.tk().comerge_testkit_generate_raw(3, 0, n, 1 << 31, raw.data_ptr(), None), True)
k = raw.to(torch.int32)
v = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
ok, ov = torch.empty_like(k), torch.empty_like(v)
for _ in range(3):
    P.sort_pairs(k, v, ok, ov)
torch.cuda.synchronize()
