"""Run one BASELINE config a few times (for ncu / tracing on the GPU box).

    python tools/run_config.py C2 [--path auto|tile|pipe] [--reps 3] [--trace]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1303_4312_b200 as P  # noqa: E402
from paper_1303_4312_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--path", default="auto")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--static-pct", type=int, default=0)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--lookahead", type=int, default=0)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    bench.CONFIGS.update(bench.EXTRA)
    inp = bench.make_inputs(args.config, device=dev)
    out = bench.alloc_outputs(args.config, inp)
    P.set_kernel_path(args.path)
    N.lib.comerge_cuda_set_tuning(args.static_pct, args.flags, args.lookahead)
    flush = bench.L2Flush(dev)
    trace = torch.zeros(20 * 4096, dtype=torch.int64, device=dev) if args.trace else None
    for r in range(args.reps):
        flush()
        if trace is not None and r == args.reps - 1:
            N.lib.comerge_cuda_set_trace(C.c_void_p(trace.data_ptr()))
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        bench.run_config(args.config, inp, out)
        e.record()
        torch.cuda.synchronize()
        N.lib.comerge_cuda_set_trace(None)
        print(f"{args.config} rep {r}: {s.elapsed_time(e) * 1e3:.1f} us "
              f"(path {N.lib.comerge_cuda_last_path()})")
    if trace is not None:
        report(trace)


def report(trace):
    """Per-CTA phase summary of a traced pipeline launch."""
    if True:
        rows = trace[: 8 * 4096].view(-1, 8).cpu()
        live = rows[:, 0] > 0
        ext_raw = trace[8 * 4096: 8 * 4096 + 4 * 4096].view(-1, 4).cpu()[live]
        ext = ext_raw.double() / 1e3
        full = rows[live]
        t = full[:, :4]
        t0 = t[:, 0].min()
        rel = (t - t0).double() / 1e3
        q = lambda x: [round(float(x.quantile(p)), 2) for p in (0.0, 0.5, 0.9, 1.0)]  # noqa: E731
        print(f"CTAs {t.shape[0]}; us from first CTA start [min, p50, p90, max]:")
        print("  start      ", q(rel[:, 0]))
        sched = full[:, 1]
        print("  sched claims", q((sched >> 48).double()), "rounds", q(((sched >> 32) & 0xffff).double()),
              "search us", q((sched & 0xffffffff).double()))
        print("  first tile ", q(rel[:, 2]))
        print("  end        ", q(rel[:, 3]))

        dur = rel[:, 3] - rel[:, 2]
        sm = full[:, 4]
        order = torch.argsort(dur)
        print("  stream dur ", q(dur))
        print("  startup done", q((full[:, 5] - t0).double() / 1e3))
        print("  consumer us: merge", q(ext[:, 0]), "bar1", q(ext[:, 1]), "stage+bar2", q(ext[:, 2]))
        print("  stores drained after consumer end us", q((ext_raw[:, 3] - full[:, 3]).double() / 1e3))
        print("  producer starved us", q(full[:, 6].double() / 1e3))
        r3 = trace[12 * 4096: 12 * 4096 + 4 * 4096].view(-1, 4).cpu()[live]
        print("    static range us", q(r3[:, 0].double() / 1e3), "waits", q(r3[:, 2].double()),
              "| tail us", q(r3[:, 1].double() / 1e3), "waits", q(r3[:, 3].double()))
        r4 = trace[16 * 4096: 16 * 4096 + 4 * 4096].view(-1, 4).cpu()[live]
        print("  tail slots co-ranked by the scheduler (not yet published)", q(r4[:, 0].double()),
              "tail warp done us", q((r4[:, 1] - t0).double() / 1e3),
              "first tail claim us", q((r4[:, 2] - t0).double() / 1e3))
        fb = r4[:, 0] > 0
        if fb.any():
            print("  last fallback tile index (of NT)", q(r4[fb, 3].double()))
        print("  consumer data-wait us", q(full[:, 7].double() / 1e3))
        print("  slowest 12 (cta, smid, us):",
              [(int(i), int(sm[i]), round(float(dur[i]), 1)) for i in order[-12:]])
        print("  fastest 6  (cta, smid, us):",
              [(int(i), int(sm[i]), round(float(dur[i]), 1)) for i in order[:6]])
        by_sm = {}
        for i in range(len(sm)):
            by_sm.setdefault(int(sm[i]), []).append(round(float(rel[i, 3]), 1))
        ends = sorted(((max(v), k, v) for k, v in by_sm.items()))
        print("  latest-finishing SMs:", [(k, v) for _, k, v in ends[-8:]])
        print("  earliest-finishing SMs:", [(k, v) for _, k, v in ends[:4]])


if __name__ == "__main__":
    main()
