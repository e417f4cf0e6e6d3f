"""Per-chunk timeline of the host-buffer pipeline for one config
(COMERGE_HOST_TRACE=1): python tools/e2e_trace.py C4r"""
import os
import sys
import time

os.environ["COMERGE_HOST_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import torch  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4r"
inp = bench.make_inputs(cfg, device=torch.device("cuda", 0))
r = bench.e2e_measure(cfg, inp, 3, 1)
print(cfg, r, flush=True)
