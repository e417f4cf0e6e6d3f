"""Per-CTA trace of the LAST merge pass of a 2^26 int32 merge sort (the
trace buffer keeps the last pipeline launch), plus the sort's time.
    python tools/trace_sort.py [log2 n]"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_1303_4312_b200 as P  # noqa: E402
import paper_1303_4312_b200._native as N  # noqa: E402
import run_config  # noqa: E402

n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 26)
raw = torch.empty(n, dtype=torch.int64, device="cuda")
N.check(N.tk().comerge_testkit_generate_raw(3, 0, n, 1 << 31, raw.data_ptr(), None), True)
k = raw.to(torch.int32)
out = torch.empty_like(k)
ws = torch.empty(P.sort_workspace_bytes(n, k.dtype), dtype=torch.uint8, device="cuda")
for _ in range(3):
    P.sort(k, out=out, workspace=ws)
trace = torch.zeros(20 * 4096, dtype=torch.int64, device="cuda")
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N.lib.comerge_cuda_set_trace(C.c_void_p(trace.data_ptr()))
s.record()
P.sort(k, out=out, workspace=ws)
e.record()
torch.cuda.synchronize()
N.lib.comerge_cuda_set_trace(None)
print(f"sort 2^{n.bit_length() - 1} int32: {s.elapsed_time(e):.3f} ms (traced)")
run_config.report(trace)
