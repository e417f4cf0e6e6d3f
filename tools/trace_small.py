"""Per-CTA phase timeline of the one-wave small-merge kernel:
python tools/trace_small.py C1 [flags]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1303_4312_b200 as P  # noqa: E402
from paper_1303_4312_b200 import _native as N  # noqa: E402

cfg = sys.argv[1]
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 0
dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
inp = bench.make_inputs(cfg, device=dev)
out = bench.alloc_outputs(cfg, inp)
P.set_kernel_path("small")
N.lib.comerge_cuda_set_tuning(0, flags, 0)
trace = torch.zeros(8 * 4096, dtype=torch.int64, device=dev)
for r in range(5):
    flush()
    torch.cuda.synchronize()
    if r == 4:
        N.lib.comerge_cuda_set_trace(C.c_void_p(trace.data_ptr()))
    bench.run_config(cfg, inp, out)
    torch.cuda.synchronize()
    N.lib.comerge_cuda_set_trace(None)
rows = trace.view(-1, 8).cpu()
rows = rows[rows[:, 0] > 0]
t0 = rows[:, 0].min()
rel = (rows[:, :5] - t0).double() / 1e3
q = lambda x: [round(float(x.quantile(p)), 2) for p in (0.0, 0.5, 0.9, 1.0)]  # noqa: E731
print(f"{cfg} flags {flags}: CTAs {rows.shape[0]}; us from first CTA start [min, p50, p90, max]")
for k, name in enumerate(["start", "co-ranked", "windows in", "merged", "stored"]):
    print(f"  {name:11s}", q(rel[:, k]))
