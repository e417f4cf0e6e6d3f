"""Sort timings (2^26 int32 keys) per static share of the merge passes' tiles:
python tools/micro/sort_static.py 60,70,80,90 [flags]"""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_1303_4312_b200 as P
import paper_1303_4312_b200._native as N
n = 1 << 26
raw = torch.empty(n, dtype=torch.int64, device="cuda")
N.check(N.tk().comerge_testkit_generate_raw(3, 0, n, 1 << 31, raw.data_ptr(), None), True)
k = raw.to(torch.int32); del raw
ok = torch.empty_like(k)
ws = torch.empty(P.sort_workspace_bytes(n, torch.int32), dtype=torch.uint8, device="cuda")
flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device="cuda")
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for rnd in range(2):
    for pct in [int(x) for x in sys.argv[1].split(",")]:
        N.lib.comerge_cuda_set_tuning(pct, flags, 0)
        tk = []
        for r in range(10):
            flush.fill_(r)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); P.sort(k, out=ok, workspace=ws); b.record(); torch.cuda.synchronize()
            if r >= 2: tk.append(a.elapsed_time(b))
        print("static", pct, "sort keys ms", round(statistics.median(tk), 4), flush=True)
N.lib.comerge_cuda_set_tuning(0, 0, 0)
