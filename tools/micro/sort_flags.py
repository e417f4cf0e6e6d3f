"""Sort timings (2^26 int32 keys / pairs) per tuning-flags value: python tools/micro/sort_flags.py 0,262144"""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_1303_4312_b200 as P
import paper_1303_4312_b200._native as N
n = 1 << 26
raw = torch.empty(n, dtype=torch.int64, device="cuda")
N.check(N.tk().comerge_testkit_generate_raw(3, 0, n, 1 << 31, raw.data_ptr(), None), True)
k = raw.to(torch.int32); del raw
v = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
ok, ov = torch.empty_like(k), torch.empty_like(v)
ws = torch.empty(P.sort_pairs_workspace_bytes(n, torch.int32), dtype=torch.uint8, device="cuda")
flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device="cuda")
for f in [int(x) for x in sys.argv[1].split(",")]:
    N.lib.comerge_cuda_set_tuning(0, f, 0)
    ts = []
    for r in range(8):
        flush.fill_(r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); P.sort_pairs(k, v, ok, ov, workspace=ws); b.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(a.elapsed_time(b))
    tk = []
    for r in range(8):
        flush.fill_(r)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); P.sort(k, out=ok, workspace=ws); b.record(); torch.cuda.synchronize()
        if r >= 2: tk.append(a.elapsed_time(b))
    print("flags", f, "sort_pairs ms", round(statistics.median(ts), 3), "sort keys ms",
          round(statistics.median(tk), 3), flush=True)
N.lib.comerge_cuda_set_tuning(0, 0, 0)
