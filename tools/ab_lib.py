"""Kernel time per config for the library at COMERGE_LIB_PATH (A/B of build
variants: run once per variant).   python tools/ab_lib.py NAME C1,C2,... [--steps 20]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("name")
    ap.add_argument("configs")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=2)
    args = ap.parse_args()
    import torch
    import bench
    bench.CONFIGS.update(bench.EXTRA)
    dev = torch.device("cuda:0")
    flush = bench.L2Flush(dev)
    for cfg in args.configs.split(","):
        r, st = [], []
        for _ in range(args.rounds):
            t = bench.time_config(cfg, args.steps, 3, dev, flush)
            r.append(statistics.mean(t["kern_ms"]) * 1e3)
            st.append(statistics.mean(t["step_ms"]) * 1e3)
        print(f"{args.name:8s} {cfg:4s} kernel us {min(r):8.1f}  step us {min(st):8.1f}  "
              f"(rounds {[round(x, 1) for x in r]})", flush=True)


if __name__ == "__main__":
    main()
