"""Run the merge sort a few times on seeded keys (for ncu):
    python tools/run_sort.py [lg=26] [int32|uint64] [pairs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1303_4312_b200 as P  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
dt = sys.argv[2] if len(sys.argv) > 2 else "int32"
pairs = len(sys.argv) > 3 and sys.argv[3] == "pairs"
g = torch.Generator(device="cuda")
g.manual_seed(3)
k = torch.randint(0, 2**31 - 1, (1 << lg,), dtype=torch.int64, device="cuda", generator=g)
k = k.to(torch.int32) if dt == "int32" else (k * 2**31 + k).view(torch.uint64)
v = torch.arange(1 << lg, dtype=torch.int32, device="cuda").view(torch.uint32)
for _ in range(3):
    out = P.sort_pairs(k, v) if pairs else P.sort(k)
torch.cuda.synchronize()
print("sorted", 1 << lg, dt, "pairs" if pairs else "keys")
