"""e2e of one config under several tuning-flag values (same process):
    python tools/e2e_flags.py C1 0,8388608"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1303_4312_b200._native as N  # noqa: E402

cfg = sys.argv[1]
flags = [int(x) for x in sys.argv[2].split(",")]
inp = bench.make_inputs(cfg, device=torch.device("cuda:0"))
for r in range(2):
    for f in flags:
        N.lib.comerge_cuda_set_tuning(0, f, 0)
        res = bench.e2e_measure(cfg, inp, 7, 2)
        print(f"{cfg} flags={f}: e2e {res['ms_per_step']:.3f} ms  calls {res['calls_ms']}", flush=True)
N.lib.comerge_cuda_set_tuning(0, 0, 0)
