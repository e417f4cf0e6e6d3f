import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch, bench
dev = torch.device("cuda:0")
for r in range(3):
    for clk in (False, True):
        t = bench.time_config("C2", 20, 5, dev, clocks=clk)
        print("clocks", clk, "step us", round(statistics.mean(t["step_ms"]) * 1e3, 1),
              "kernel us", round(statistics.mean(t["kern_ms"]) * 1e3, 1),
              "max step", round(max(t["step_ms"]) * 1e3, 1), flush=True)
