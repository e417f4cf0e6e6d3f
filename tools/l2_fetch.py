"""Effect of cudaLimitMaxL2FetchGranularity on the merge kernels: kernel time
(bench timing) and, with --ncu, nothing else (run under ncu for DRAM bytes).
    python tools/l2_fetch.py C4 [granularity ...]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402

cfg = sys.argv[1]
grans = [int(x) for x in sys.argv[2:]] or [128, 32]
rt = C.CDLL("libcudart.so.12")
dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
inp = bench.make_inputs(cfg, device=dev)
out = bench.alloc_outputs(cfg, inp)
cudaLimitMaxL2FetchGranularity = 0x05
for r in range(2):
    for g in grans:
        assert rt.cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, C.c_size_t(g)) == 0
        v = C.c_size_t(0)
        rt.cudaDeviceGetLimit(C.byref(v), cudaLimitMaxL2FetchGranularity)
        t = bench.time_steps(lambda: bench.run_config(cfg, inp, out), 10, 3, dev, flush)
        print(f"{cfg} L2 fetch granularity {g} (now {v.value}): kernel us "
              f"{statistics.mean(t['kern_ms']) * 1e3:.1f}", flush=True)
