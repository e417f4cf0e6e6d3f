import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch, bench
dev = torch.device("cuda:0")
flush = bench.L2Flush(dev)
for r in range(6):
    t = bench.time_config("C4", 20, 5, dev, flush, clocks=(r % 2 == 0))
    s = t["step_ms"]
    print("call", r, "clocks", r % 2 == 0, "mean", round(statistics.mean(s) * 1e3, 1), "median", round(statistics.median(s) * 1e3, 1),
          "max", round(max(s) * 1e3, 1), "steps > 1.05ms:", [round(x * 1e3) for x in s if x > 1.05], flush=True)
