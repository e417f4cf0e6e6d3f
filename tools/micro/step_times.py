"""Per-step device times of the bench's headline measurement (first call in a
fresh process, as bench.py does), to see outliers."""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch, bench
dev = torch.device("cuda:0")
for r in range(3):
    t = bench.time_config("C2", 20, 5, dev, clocks=(r == 0))
    print("call", r, "steps us", [round(x * 1e3, 1) for x in t["step_ms"]], flush=True)
    print("        kern us", [round(x * 1e3, 1) for x in t["kern_ms"]], flush=True)
