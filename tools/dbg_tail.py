import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1303_4312_b200 as P
from oracle.py import Port
port = Port()
P.set_kernel_path("pipe")
rng = np.random.default_rng(1)
for (m, n) in [(3, 50000), (50000, 3), (20000, 30003), (3, 50000)]:
    for kv in (False, True, False, True):
        a = np.sort(rng.integers(-2**30, 2**30, m)).astype(np.int32)
        b = np.sort(rng.integers(-2**30, 2**30, n)).astype(np.int32)
        av = np.arange(m, dtype=np.uint32); bv = np.arange(n, dtype=np.uint32) | np.uint32(1 << 31)
        if kv:
            ok, ov = P.merge_pairs(torch.from_numpy(a).cuda(), torch.from_numpy(av).cuda(), torch.from_numpy(b).cuda(), torch.from_numpy(bv).cuda())
        else:
            ok = P.stable_merge(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
        torch.cuda.synchronize()
        ek = port.merge(a, b)
        got = ok.cpu().numpy()
        bad = np.nonzero(got != ek)[0]
        print(m, n, "kv" if kv else "keys", "bad", len(bad), (bad.min(), bad.max()) if len(bad) else "", "tiles@3840:", sorted(set((bad // 3840).tolist())))
