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
    ap.add_argument("--static", default="", help="comma list: A/B the static share (%%) instead of flags")
    args = ap.parse_args()
    import torch
    import bench
    import paper_1303_4312_b200._native as N
    bench.CONFIGS.update(bench.EXTRA)
    dev = torch.device("cuda:0")
    flags = [int(x) for x in args.flags.split(",")]
    las = [int(x) for x in args.lookahead.split(",")]
    sts = [int(x) for x in args.static.split(",")] if args.static else []
    if len(las) > 1:  # A/B the look-ahead at flags[0]
        flags = las
    if sts:  # A/B the static share at flags[0]
        flags = sts
    flush = bench.L2Flush(dev)
    inp = bench.make_inputs(args.config, device=dev)
    out = bench.alloc_outputs(args.config, inp)
    res = {f: [] for f in flags}
    for r in range(args.rounds):
        for f in flags:
            if sts:
                N.lib.comerge_cuda_set_tuning(f, int(args.flags.split(",")[0]), las[0])
            elif len(las) > 1:
                N.lib.comerge_cuda_set_tuning(args.static_pct, int(args.flags.split(",")[0]), f)
            else:
                N.lib.comerge_cuda_set_tuning(args.static_pct, f, las[0])
            t = bench.time_steps(lambda: bench.run_config(args.config, inp, out), args.steps, 3,
                                 dev, flush)
            res[f].append(statistics.mean(t["kern_ms"]) * 1e3)
    N.lib.comerge_cuda_set_tuning(0, 0, 0)
    for f in flags:
        what = "static" if sts else ("lookahead" if len(las) > 1 else "flags")
        print(f"{args.config} {what}={f}: kernel us per round {[round(x, 1) for x in res[f]]} "
              f"mean {statistics.mean(res[f]):.1f}")


if __name__ == "__main__":
    main()
