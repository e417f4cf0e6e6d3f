#!/usr/bin/env python3
"""Benchmark of the B200 stable merge on the BASELINE.json configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One "step" is one stable merge of one config's full synthetic input (already
resident in HBM), timed with CUDA events on the launching stream; L2 is
flushed (512 MiB write) between steps, outside the events.  The headline
line is configs[1] of BASELINE.json (C2: key-value stability stress,
m = n = 2^24); every other config is measured too and reported under
"configs".  Metric: merged elements/s (+ achieved HBM GB/s vs the measured
copy peak).

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libcomerge_ref.so = /root/reference compiled unmodified:
comerge::merge_parallel with hardware_concurrency threads) on the same
config and prints the same JSON line with "impl": "reference".

Under torchrun (N > 1) every rank merges its own instance (seed + rank):
weak scaling, no collective on the data path; times are the max over ranks.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "C1": dict(kind="keys", dtype="int32", m=2**20, n=2**20, width=2**31,
               desc="int32 keys only, m=n=2^20, uniform [0,2^31)"),
    "C2": dict(kind="pairs", dtype="int32", m=2**24, n=2**24, width=16,
               desc="stability stress key-value, m=n=2^24, int32 keys in [0,16), uint32 "
                    "payload (A: i, B: i|2^31)"),
    "C3": dict(kind="keys", dtype="int32", m=2**12, n=2**28, width=2**31,
               desc="skewed int32, m=2^12, n=2^28"),
    "C3s": dict(kind="keys", dtype="int32", m=2**28, n=2**12, width=2**31, swapped=True,
                desc="skewed int32 swapped, m=2^28, n=2^12 (same arrays as C3)"),
    "C4": dict(kind="pairs", dtype="uint64", m=2**27, n=2**27, width=0,
               desc="uint64 keys (full range) + uint32 payload, m=n=2^27"),
    "C5": dict(kind="segmented", dtype="int32", nseg=2**14, maxlen=4096, width=2**20,
               desc="segmented batch: 2^14 pairs, m_s,n_s in [1,4096], int32 keys in [0,2^20)"),
}
# diagnostic shapes (not BASELINE configs; run only when named explicitly)
EXTRA = {
    "X1": dict(kind="keys", dtype="int32", m=2**26, n=2**26, width=2**31,
               desc="diagnostic: int32 keys only, m=n=2^26, uniform [0,2^31)"),
    "X2": dict(kind="pairs", dtype="int32", m=2**26, n=2**26, width=2**31,
               desc="diagnostic: int32 keys + payload, m=n=2^26, uniform [0,2^31)"),
    "X3": dict(kind="segmented", dtype="int32", nseg=2**20, maxlen=64, width=2**20,
               desc="diagnostic: segmented batch of 2^20 small pairs, m_s,n_s in [1,64]"),
    "X4": dict(kind="segmented", dtype="int32", nseg=2**21, maxlen=16, width=2**20,
               desc="diagnostic: segmented batch of 2^21 tiny pairs, m_s,n_s in [1,16]"),
}
HEADLINE = "C2"
SEED = 5


def key_bytes(cfg):
    return 8 if CONFIGS[cfg]["dtype"] == "uint64" else 4


def elem_bytes(cfg):
    c = CONFIGS[cfg]
    return key_bytes(cfg) + (4 if c["kind"] == "pairs" else 0)


# ------------------------------------------------------------------ inputs

def make_inputs(cfg, seed=SEED, device="cuda"):
    """Seeded inputs on the device (splitmix64 recipe of generate.cpp:17-29)."""
    import torch
    from paper_1303_4312_b200 import testkit as tk
    c = CONFIGS[cfg]
    tdt = {"int32": torch.int32, "uint64": torch.uint64}[c["dtype"]]
    with torch.cuda.device(device):
        if c["kind"] == "segmented":
            sizes = tk.generate_raw(seed, 2, 2 * c["nseg"], c["maxlen"], device=device)
            sizes = sizes.view(torch.int64) + 1          # m_s, n_s = 1 + below(4096)
            ms, ns = sizes[0::2], sizes[1::2]
            zero = torch.zeros(1, dtype=torch.int64, device=device)
            a_off = torch.cat([zero, torch.cumsum(ms, 0)]).view(torch.uint64)
            b_off = torch.cat([zero, torch.cumsum(ns, 0)]).view(torch.uint64)
            a = tk.generate_runs(tdt, seed, 0, a_off, c["width"])
            b = tk.generate_runs(tdt, seed, 1, b_off, c["width"])
            return dict(a=a, b=b, a_off=a_off, b_off=b_off)
        if c.get("swapped"):
            a = tk.generate_sorted(tdt, seed, 1, c["m"], c["width"], device=device)
            b = tk.generate_sorted(tdt, seed, 0, c["n"], c["width"], device=device)
        else:
            a = tk.generate_sorted(tdt, seed, 0, c["m"], c["width"], device=device)
            b = tk.generate_sorted(tdt, seed, 1, c["n"], c["width"], device=device)
        inp = dict(a=a, b=b)
        if c["kind"] == "pairs":
            inp["av"] = tk.iota(c["m"], 0, device=device)
            inp["bv"] = tk.iota(c["n"], 1 << 31, device=device)
        return inp


def alloc_outputs(cfg, inp):
    """Outputs plus the merge's scratch workspace (queried, CUB-style)."""
    import torch
    import paper_1303_4312_b200._native as N
    total = inp["a"].numel() + inp["b"].numel()
    dev = inp["a"].device
    out = dict(keys=torch.empty(total, dtype=inp["a"].dtype, device=dev))
    kind = {"int32": N.KEY_I32, "uint64": N.KEY_U64}[CONFIGS[cfg]["dtype"]]
    if CONFIGS[cfg]["kind"] == "segmented":
        wsb = N.lib.comerge_cuda_segmented_workspace_bytes(total, inp["a_off"].numel() - 1, kind)
    else:
        wsb = N.lib.comerge_cuda_merge_workspace_bytes(inp["a"].numel(), inp["b"].numel(), kind,
                                                       int(CONFIGS[cfg]["kind"] == "pairs"))
    out["ws"] = torch.empty(max(int(wsb), 256), dtype=torch.uint8, device=dev)
    if CONFIGS[cfg]["kind"] == "pairs":
        out["vals"] = torch.empty(total, dtype=torch.uint32, device=dev)
    return out


def run_config(cfg, inp, out=None):
    """One merge of the config through the public API (async, current stream)."""
    import paper_1303_4312_b200 as P
    if out is None:
        out = alloc_outputs(cfg, inp)
    kind = CONFIGS[cfg]["kind"]
    ws = out.get("ws")
    if kind == "keys":
        P.stable_merge(inp["a"], inp["b"], out["keys"], workspace=ws)
    elif kind == "pairs":
        P.merge_pairs(inp["a"], inp["av"], inp["b"], inp["bv"], out["keys"], out["vals"],
                      workspace=ws)
    else:
        P.merge_segmented(inp["a"], inp["a_off"], inp["b"], inp["b_off"], out["keys"],
                          workspace=ws)
    return out


KERNEL_NAMES = {1: "merge_tile_kernel (+ partition_kernel)", 2: "merge_stream_kernel",
                3: "merge_pipe_kernel", 4: "seg_merge_tile_kernel (+ seg_partition_kernel)",
                5: "merge_pipe_kernel (segmented)"}


def launches_per_step(path):
    return 1 if path in (2, 3, 5) else 2  # persistent kernels: one launch; tile paths: two


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ timing

_CUDART = None


def _cudart():
    """The CUDA runtime the merge library itself uses (for raw event handles)."""
    global _CUDART
    if _CUDART is None:
        import paper_1303_4312_b200._native  # noqa: F401  (loads libcudart first)
        _CUDART = C.CDLL("libcudart.so.12")
        _CUDART.cudaEventCreate.argtypes = [C.POINTER(C.c_void_p)]
        _CUDART.cudaEventElapsedTime.argtypes = [C.POINTER(C.c_float), C.c_void_p, C.c_void_p]
    return _CUDART


def raw_events(k):
    rt = _cudart()
    out = []
    for _ in range(k):
        e = C.c_void_p()
        assert rt.cudaEventCreate(C.byref(e)) == 0
        out.append(e)
    return out


def raw_elapsed_ms(e0, e1):
    ms = C.c_float()
    rc = _cudart().cudaEventElapsedTime(C.byref(ms), e0, e1)
    assert rc == 0, f"cudaEventElapsedTime failed ({rc})"
    return float(ms.value)


def peak_hbm():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_for(cfg):
    """DRAM bytes per launch of the merge kernel from the committed ncu capture."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            v = json.load(f).get(cfg)
        return v if isinstance(v, (int, float)) else None
    except Exception:
        return None


def time_config(cfg, steps, warmup, device, seed=SEED, dist_ctx=None, clocks=False):
    import torch
    import paper_1303_4312_b200._native as N
    inp = make_inputs(cfg, seed=seed, device=device)
    out = alloc_outputs(cfg, inp)
    total = inp["a"].numel() + inp["b"].numel()
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device=device)
    stream = torch.cuda.current_stream(device)
    # warm-up steps are the timed step exactly (flush, events, merge), untimed:
    # the first flush launch of a process otherwise lands in timed step 0
    # (seen: +113 us on the first step of a fresh process, lazy module load)
    wev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for k in range(max(warmup, 0)):
        flush.fill_(k)
        wev[0].record(stream)
        run_config(cfg, inp, out)
        wev[1].record(stream)
    torch.cuda.synchronize(device)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] + list(raw_events(2))
          for _ in range(steps)]
    sampler = ClockSampler(device.index or 0) if clocks else None
    if dist_ctx:
        dist_ctx.barrier()
    torch.cuda.synchronize(device)
    if sampler:
        sampler.__enter__()
    # hold the GPU behind a spin so the host enqueues every step before the
    # device starts them: step events then time device work, not host enqueue
    torch.cuda._sleep(int(2e8))
    for k in range(steps):
        flush.fill_(k)  # evict L2 (> 126 MB) outside the timed events
        s0, s1 = ev[k][0], ev[k][1]
        s0.record(stream)
        run_config(cfg, inp, out)
        s1.record(stream)
    torch.cuda.synchronize(device)
    if dist_ctx:
        dist_ctx.barrier()
    if sampler:
        sampler.__exit__()
    # the same steps again with events recorded by the library right around
    # the merge kernel (the roofline's kernel time; kept out of the steps
    # above because every extra event costs ~2.7 us on this platform)
    torch.cuda._sleep(int(2e8))
    for k in range(steps):
        flush.fill_(k)
        k0, k1 = ev[k][2], ev[k][3]
        N.lib.comerge_cuda_set_kernel_events(k0, k1)
        run_config(cfg, inp, out)
        N.lib.comerge_cuda_set_kernel_events(None, None)
    torch.cuda.synchronize(device)
    path = N.lib.comerge_cuda_last_path()
    step_ms = [e[0].elapsed_time(e[1]) for e in ev]
    kern_ms = [raw_elapsed_ms(e[2], e[3]) for e in ev]
    res = dict(total=total, step_ms=step_ms, kern_ms=kern_ms, path=path,
               clocks=sampler.summary() if sampler else None, inp=inp, out=out)
    return res


def summarize(cfg, res, peak, n_gpus=1, max_step_total_ms=None):
    total = res["total"]
    balg = 2 * total * elem_bytes(cfg)
    step_total = max_step_total_ms if max_step_total_ms is not None else sum(res["step_ms"])
    steps = len(res["step_ms"])
    ms_step = step_total / steps
    kern = statistics.mean(res["kern_ms"])
    return dict(
        workload=CONFIGS[cfg]["desc"], m=int(res["inp"]["a"].numel()),
        n=int(res["inp"]["b"].numel()), elements=total,
        elements_per_s=n_gpus * total * steps / (step_total * 1e-3),
        ms_per_step=ms_step, step_gbs=balg / (ms_step * 1e-3) / 1e9,
        merge_kernel_ms=kern, merge_kernel_gbs=balg / (kern * 1e-3) / 1e9,
        frac_of_peak=balg / (kern * 1e-3) / 1e9 / peak,
        step_frac_of_peak=balg / (ms_step * 1e-3) / 1e9 / peak,
        frac_of_8tbs=balg / (kern * 1e-3) / 8e12, algorithmic_bytes=balg,
        kernel=KERNEL_NAMES.get(res["path"], "?"), launches_per_step=launches_per_step(res["path"]))


# ------------------------------------------------------------- CPU legs

def host_arrays(cfg, inp):
    """Device inputs -> host numpy (+ AoS {key,val} for key-value configs)."""
    from oracle.py import to_aos
    h = {k: v.cpu().numpy() for k, v in inp.items()}
    if CONFIGS[cfg]["kind"] == "pairs":
        h["a_aos"] = to_aos(h["a"], h["av"])
        h["b_aos"] = to_aos(h["b"], h["bv"])
    return h


def cpu_reference_run(cfg, h, threads):
    """One run of the reference's CPU path on host arrays; returns wall ns
    (merge_report.wall_ns: the parallel region only, parallel.hpp:252-267)."""
    from oracle.py import Ref, available_ref, Port
    kind = CONFIGS[cfg]["kind"]
    if available_ref():
        ref = Ref()
        if kind == "segmented":
            return ref.merge_segmented(h["a"], h["a_off"], h["b"], h["b_off"], threads=threads,
                                       out=h.setdefault("out", np.empty(len(h["a"]) + len(h["b"]),
                                                                        h["a"].dtype)))[1], "reference"
        if kind == "pairs":
            o = h.setdefault("out_aos", np.zeros(len(h["a_aos"]) + len(h["b_aos"]),
                                                 h["a_aos"].dtype))
            return ref.merge_parallel_kv(h["a_aos"], h["b_aos"], threads, out=o)[1].wall_ns, \
                "reference"
        o = h.setdefault("out", np.zeros(len(h["a"]) + len(h["b"]), h["a"].dtype))
        return ref.merge_parallel(h["a"], h["b"], threads, out=o)[1].wall_ns, "reference"
    port = Port()
    t0 = time.perf_counter_ns()
    if kind == "segmented":
        port.merge_segmented(h["a"], h["a_off"], h["b"], h["b_off"], threads=threads)
    elif kind == "pairs":
        port.merge_parallel(h["a"], h["b"], threads, h["av"], h["bv"], threads=threads)
    else:
        port.merge_parallel(h["a"], h["b"], threads, threads=threads)
    return time.perf_counter_ns() - t0, "port"


def cpu_threads():
    from oracle.py import Ref, available_ref
    if available_ref():
        return Ref().hardware_concurrency()
    return os.cpu_count() or 1


def cpu_baseline(cfg, inp, budget_s=20.0, min_reps=3, max_reps=15):
    h = host_arrays(cfg, inp)
    threads = cpu_threads()
    cpu_reference_run(cfg, h, threads)  # touch output pages
    walls, kind = [], "reference"
    t_start = time.time()
    while len(walls) < max_reps and (len(walls) < min_reps or time.time() - t_start < budget_s / 4):
        w, kind = cpu_reference_run(cfg, h, threads)
        walls.append(w)
        if time.time() - t_start > budget_s:
            break
    total = len(h["a"]) + len(h["b"])
    med = statistics.median(walls)
    return dict(value=total / (med * 1e-9), unit="elements/s", cores=threads, kind=kind,
                sample=f"full {cfg} workload ({total} elements), median of {len(walls)} runs of "
                       f"the reference's merge_report.wall_ns, {threads} threads "
                       f"(std::thread::hardware_concurrency)",
                median_ms=med / 1e6, min_ms=min(walls) / 1e6)


# ------------------------------------------------------------------- e2e

def e2e_measure(cfg, inp, steps, warmup):
    """Same metric through the host-buffer C ABI (comerge_merge_parallel_*):
    pinned host inputs, H2D + merge + D2H inside every timed call."""
    import torch
    import paper_1303_4312_b200._native as N
    c = CONFIGS[cfg]
    if c["kind"] == "segmented":
        return None
    suf = {"int32": "i32", "uint64": "u64"}[c["dtype"]]
    pin = {k: v.cpu().pin_memory() for k, v in inp.items()}
    total = inp["a"].numel() + inp["b"].numel()
    ok = torch.empty(total, dtype=inp["a"].dtype).pin_memory()
    ov = torch.empty(total, dtype=torch.uint32).pin_memory() if c["kind"] == "pairs" else None
    rep = N.MergeReport()
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

    def call():
        if c["kind"] == "pairs":
            rc = getattr(N.lib, f"comerge_merge_parallel_pairs_{suf}")(
                p(pin["a"]), p(pin["av"]), pin["a"].numel(), p(pin["b"]), p(pin["bv"]),
                pin["b"].numel(), p(ok), p(ov), total, 1, C.byref(rep))
        else:
            rc = getattr(N.lib, f"comerge_merge_parallel_{suf}")(
                p(pin["a"]), pin["a"].numel(), p(pin["b"]), pin["b"].numel(), p(ok), total, 1, 0,
                C.byref(rep), None, None)
        N.check(rc)

    for _ in range(max(1, warmup)):
        call()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    # the e2e result must equal the device-path result
    dev_keys = run_config(cfg, inp)["keys"].cpu()
    assert bool((ok.view(torch.uint8) == dev_keys.view(torch.uint8)).all()), "e2e mismatch"
    # median call: one slow call (a PCIe hiccup, seen up to +20%) would move a
    # mean of a handful of calls by several percent
    return dict(value=total / statistics.median(times), unit="elements/s", stat=f"median of {steps} calls",
                h2d_bytes_per_step=int(rep.h2d_bytes), d2h_bytes_per_step=int(rep.d2h_bytes),
                ms_per_step=1e3 * statistics.median(times),
                path=f"comerge_merge_parallel{'_pairs' if c['kind'] == 'pairs' else ''}_{suf} "
                     "(host pinned buffers)")


# ------------------------------------------------------------------ main

def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1:
        return None, 0, 1, 0
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return dist, dist.get_rank(), world, local


def reference_arm(args):
    dist, rank, world, local = dist_setup()
    if rank != 0:
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return
    import torch
    device = torch.device("cuda", local)
    cfg = args.config
    inp = make_inputs(cfg, device=device)
    h = host_arrays(cfg, inp)
    threads = cpu_threads()
    for _ in range(max(args.warmup, 1)):
        cpu_reference_run(cfg, h, threads)
    walls, kind = [], "reference"
    for _ in range(args.steps):
        w, kind = cpu_reference_run(cfg, h, threads)
        walls.append(w)
    total = len(h["a"]) + len(h["b"])
    value = total * len(walls) / (sum(walls) * 1e-9)
    line = dict(metric="merged elements/s", value=value, unit="elements/s", n_gpus=world,
                steps=args.steps, warmup=args.warmup,
                ms_per_step=sum(walls) / len(walls) / 1e6, higher_is_better=True,
                scaling="weak", vs_baseline=None, dtype=CONFIGS[cfg]["dtype"], data="synthetic",
                impl="reference",
                config=dict(workload=f"{cfg}: {CONFIGS[cfg]['desc']}", elements=total,
                            l2="n/a (CPU)"),
                cpu_baseline=dict(value=value, unit="elements/s", cores=threads, kind=kind,
                                  sample=f"full {cfg} workload per step, reference "
                                         "comerge::merge_parallel, merge_report.wall_ns"),
                e2e=dict(value=value, unit="elements/s", h2d_bytes_per_step=0,
                         d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def sort_extras(device, reps=5):
    """SURVEY 8f row 1 (not a BASELINE config): the stable merge sorts on
    2^26 int32 keys (uniform 31-bit, seeded) with and without uint32 payloads,
    median device time (events, L2 flushed before each rep)."""
    import torch
    import paper_1303_4312_b200 as P
    import paper_1303_4312_b200._native as N
    n = 1 << 26
    raw = torch.empty(n, dtype=torch.int64, device=device)
    N.check(N.tk().comerge_testkit_generate_raw(SEED, 0, n, 1 << 31, raw.data_ptr(), None), True)
    k = raw.to(torch.int32)
    del raw
    v = torch.arange(n, dtype=torch.int32, device=device).view(torch.uint32)
    ok, ov = torch.empty_like(k), torch.empty_like(v)
    ws = torch.empty(max(P.sort_workspace_bytes(n, torch.int32),
                         P.sort_pairs_workspace_bytes(n, torch.int32)), dtype=torch.uint8,
                     device=device)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.int32, device=device)

    def med(fn):
        ts = []
        for r in range(reps + 2):
            flush.fill_(r)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(e0.elapsed_time(e1))
        return statistics.median(ts)

    t_keys = med(lambda: P.sort(k, out=ok, workspace=ws))
    t_pairs = med(lambda: P.sort_pairs(k, v, out_keys=ok, out_vals=ov, workspace=ws))
    out = {"workload": "2^26 int32 keys, uniform [0, 2^31), seeded; stable merge sort",
           "keys_ms": t_keys, "keys_per_s": n / (t_keys * 1e-3),
           "pairs_ms": t_pairs, "pairs_per_s": n / (t_pairs * 1e-3)}
    del k, v, ok, ov, ws, flush
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--only-headline", action="store_true",
                    help="skip the per-config table")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    dist, rank, world, local = dist_setup()
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    peak, peak_src = peak_hbm()

    class Ctx:
        def barrier(self):
            if dist:
                dist.barrier()

    ctx = Ctx() if dist else None
    cfg = args.config
    res = time_config(cfg, args.steps, args.warmup, device, seed=SEED + rank, dist_ctx=ctx,
                      clocks=(rank == 0))
    step_total = sum(res["step_ms"])
    if dist:
        t = torch.tensor([step_total], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_total = float(t.item())
    head = summarize(cfg, res, peak, n_gpus=world, max_step_total_ms=step_total)

    per_config = {}
    if not args.only_headline:
        for other in CONFIGS:
            if other == cfg:
                per_config[other] = {k: v for k, v in head.items()}
                per_config[other]["elements_per_s"] = head["elements_per_s"] / world
                continue
            r = time_config(other, min(args.steps, 10), 3, device, seed=SEED + rank)
            per_config[other] = summarize(other, r, peak)
            del r
            torch.cuda.empty_cache()

    sorts = None if args.only_headline else sort_extras(device)
    e2e = None if args.no_e2e or rank != 0 else e2e_measure(cfg, res["inp"], max(5, min(args.steps, 9)), 1)
    cpu = None if args.no_cpu or rank != 0 else cpu_baseline(cfg, res["inp"])
    if rank == 0:
        line = dict(
            metric="merged elements/s", value=head["elements_per_s"], unit="elements/s",
            n_gpus=world, steps=args.steps, warmup=args.warmup, ms_per_step=head["ms_per_step"],
            higher_is_better=True, scaling="weak", vs_baseline=None,
            dtype=CONFIGS[cfg]["dtype"] + ("+u32 payload" if CONFIGS[cfg]["kind"] == "pairs" else ""),
            data="synthetic (seeded splitmix64, generate.cpp recipe)",
            config=dict(workload=f"{cfg}: {CONFIGS[cfg]['desc']}", elements=head["elements"],
                        parallelism=f"{world} GPU(s), independent instance per GPU",
                        l2="flushed between steps (512 MiB write, outside the events)"),
            roofline=dict(bound="hbm", achieved=head["merge_kernel_gbs"], peak=peak,
                          unit="GB/s", frac=head["frac_of_peak"], traffic=traffic_for(cfg),
                          kernel=head["kernel"], peak_source=peak_src,
                          algorithmic_bytes_per_launch=head["algorithmic_bytes"],
                          step_gbs=head["step_gbs"], frac_of_8tbs=head["frac_of_8tbs"]),
            cpu_baseline=cpu, e2e=e2e, clocks=res["clocks"],
            gpu_launches=args.steps * head["launches_per_step"],
            configs=per_config, sorts=sorts)
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
