import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1303_4312_b200 as P
from oracle.py import Port
port = Port()
P.set_kernel_path("pipe")
g = dict(np.load('tests/golden/ref_vectors.npz'))
for name in sorted({k.rsplit("__",1)[0] for k in g if k.startswith("merge__")}):
    a, b, o = g[name+"__a"], g[name+"__b"], g[name+"__out"]
    print(name, len(a), len(b), flush=True)
    out = P.stable_merge(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), o), name
print("ok")
