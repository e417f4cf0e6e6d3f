import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1303_4312_b200 as P
from oracle.py import Port
port = Port()
rng = np.random.default_rng(12)
def draw(n): return np.sort(rng.integers(0, 60, n)).astype(np.int32)
case = sys.argv[1]
if case == "small":
    a, b = draw(1000), draw(996)
else:
    a, b = draw(400_004), draw(333_332)
exp = port.merge(a, b)
pa, pb = [torch.from_numpy(a).cuda()], [torch.from_numpy(b).cuda()]
total = len(a) + len(b)
for lo, hi in ((0, total), (5, total - 3)):
    out = P.merge_pieces(pa, pb, lo, hi)
    torch.cuda.synchronize()
    print(case, lo, hi, np.array_equal(out.cpu().numpy(), exp[lo:hi]), flush=True)
