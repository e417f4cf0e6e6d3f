"""A/B the pipeline's experiment flags with the bench's timing (L2 flushed
between steps, events around the merge kernel): mean kernel us per flags.

    python tools/ab.py C2 0,292 [--steps 20] [--rounds 3]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("flags")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--static-pct", type=int, default=0)
    ap.add_argument("--lookahead", default="0", help="comma list: A/B the tail look-ahead instead of flags")
    args = ap.parse_args()
    import torch
    import bench
    import paper_1303_4312_b200._native as N
    bench.CONFIGS.update(bench.EXTRA)
    dev = torch.device("cuda:0")
    flags = [int(x) for x in args.flags.split(",")]
    las = [int(x) for x in args.lookahead.split(",")]
    if len(las) > 1:  # A/B the look-ahead at flags[0]
        flags = las
    res = {f: [] for f in flags}
    for r in range(args.rounds):
        for f in flags:
            if len(las) > 1:
                N.lib.comerge_cuda_set_tuning(args.static_pct, int(args.flags.split(",")[0]), f)
            else:
                N.lib.comerge_cuda_set_tuning(args.static_pct, f, las[0])
            t = bench.time_config(args.config, args.steps, 3, dev)
            res[f].append(statistics.mean(t["kern_ms"]) * 1e3)
    N.lib.comerge_cuda_set_tuning(0, 0, 0)
    for f in flags:
        print(f"{args.config} {'lookahead' if len(las) > 1 else 'flags'}={f}: kernel us per round {[round(x, 1) for x in res[f]]} "
              f"mean {statistics.mean(res[f]):.1f}")


if __name__ == "__main__":
    main()
