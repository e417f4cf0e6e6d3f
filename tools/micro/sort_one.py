import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1303_4312_b200 as P
import paper_1303_4312_b200._native as N
n = 1 << 26
raw = torch.empty(n, dtype=torch.int64, device="cuda")
N.check(N.tk().comerge_testkit_generate_raw(3, 0, n, 1 << 31, raw.data_ptr(), None), True)
k = raw.to(torch.int32)
out = torch.empty_like(k)
for _ in range(3):
    P.sort(k, out=out)
torch.cuda.synchronize()
