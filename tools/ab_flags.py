"""A/B of the runtime tuning flags on one config, bench timing (median kernel
and step times over interleaved reps): python tools/ab_flags.py C1 0,4096"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1303_4312_b200 as P  # noqa: E402
from paper_1303_4312_b200 import _native as N  # noqa: E402

cfg = sys.argv[1]
variants = [int(x) for x in sys.argv[2].split(",")]
path = sys.argv[3] if len(sys.argv) > 3 else "auto"
bench.CONFIGS.update(bench.EXTRA)
dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
inp = bench.make_inputs(cfg, device=dev)
out = bench.alloc_outputs(cfg, inp)
P.set_kernel_path(path)
res = {v: ([], []) for v in variants}
for rnd in range(6):
    for v in variants:
        N.lib.comerge_cuda_set_tuning(0, v, 0)
        r = bench.time_steps(lambda: bench.run_config(cfg, inp, out), 10, 3, dev, flush)
        res[v][0].extend(r["step_ms"])
        res[v][1].extend(r["kern_ms"])
for v in variants:
    print(f"{cfg} flags {v}: step {1e3 * statistics.median(res[v][0]):.1f} us, kernel "
          f"{1e3 * statistics.median(res[v][1]):.1f} us (path {N.lib.comerge_cuda_last_path()})")
