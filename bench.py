#!/usr/bin/env python3
"""Benchmark of the B200 stable merge on the BASELINE.json configs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4]
                    [--impl ours|reference] [--replicas]

One "step" is one stable merge of one config's full synthetic input (already
resident in HBM), timed with CUDA events on the launching stream; L2 is
flushed between steps (a 512 MiB read, outside the events, so no dirty flush
lines are written back inside the timed merge).  The headline line is the
largest BASELINE config (C4: uint64 keys + uint32 payload, m = n = 2^27;
BASELINE's metric is per config, so the largest one is quoted); every other
config is measured too and reported under "configs", each with its own CPU
baseline (the reference at p = hardware_concurrency and p = 1) and its own
end-to-end number through the host-buffer API.  Metric: merged elements/s
(+ achieved HBM GB/s vs the measured copy peak).

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libcomerge_ref.so = /root/reference compiled unmodified:
comerge::merge_parallel with hardware_concurrency threads, timed by its
merge_report.wall_ns) on the same config, with inputs generated on the host by
the reference's seeded recipe; that arm never loads this package or the GPU.

N > 1 (torchrun, or `--gpus N`, which relaunches itself under torchrun): by
default ONE merge of the config is split across the N GPUs (Algorithm 2 with a
worker per GPU; each rank merges its output range reading its peers' input
pieces over NVLink; strong scaling); `--replicas` runs an independent instance
per GPU instead (weak scaling).  Times are the max over ranks.
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
# the key-value configs in the reference's own call shape: records {key, val}
# (8 bytes; 16 with the uint64 key's padding) merged by key (oracle.hpp:22-37)
CONFIGS["C2r"] = dict(kind="records", base="C2", dtype="int32", m=2**24, n=2**24, width=16,
                      desc="C2 as 8-byte {int32 key, uint32 val} records (the reference's "
                           "struct + key-only less)")
CONFIGS["C4r"] = dict(kind="records", base="C4", dtype="uint64", m=2**27, n=2**27, width=0,
                      desc="C4 as 16-byte {uint64 key, uint32 val, pad} records (the "
                           "reference's struct + key-only less)")
# C2 as the reference's OWN tagged<int32_t> (12 bytes: key, origin byte +
# padding, uint32 index) merged with its tagged_key_less
CONFIGS["C2t"] = dict(kind="records", base="C2", dtype="int32", m=2**24, n=2**24, width=16,
                      rec=12, desc="C2 as the reference's tagged<int32_t> (12-byte {int32 key, "
                                   "origin, uint32 index} records, tagged_key_less)")
# diagnostic shapes (not BASELINE configs; tools/run_config.py only)
EXTRA = {
    "X1": dict(kind="keys", dtype="int32", m=2**26, n=2**26, width=2**31,
               desc="diagnostic: int32 keys only, m=n=2^26, uniform [0,2^31)"),
    "X2": dict(kind="pairs", dtype="int32", m=2**26, n=2**26, width=2**31,
               desc="diagnostic: int32 keys + payload, m=n=2^26, uniform [0,2^31)"),
    "X3": dict(kind="segmented", dtype="int32", nseg=2**20, maxlen=64, width=2**20,
               desc="diagnostic: segmented batch of 2^20 small pairs, m_s,n_s in [1,64]"),
    "X4": dict(kind="segmented", dtype="int32", nseg=2**21, maxlen=16, width=2**20,
               desc="diagnostic: segmented batch of 2^21 tiny pairs, m_s,n_s in [1,16]"),
    "X5": dict(kind="keys", dtype="uint64", m=2**26, n=2**26, width=0,
               desc="diagnostic: uint64 keys only (the reference's key_t), m=n=2^26, full range"),
}
HEADLINE = "C4"
SEED = 5
METRIC = "merged elements/s"


def key_bytes(cfg):
    return 8 if CONFIGS[cfg]["dtype"] == "uint64" else 4


def elem_bytes(cfg):
    c = CONFIGS[cfg]
    if c["kind"] == "records":
        return c.get("rec", 2 * key_bytes(cfg))
    return key_bytes(cfg) + (4 if c["kind"] == "pairs" else 0)


def dtype_str(cfg):
    c = CONFIGS[cfg]
    k = {"int32": "int32", "uint64": "u64"}[c["dtype"]]
    if c["kind"] == "records":
        if c.get("rec") == 12:
            return f"12-byte tagged<{k}> records ({k} key, origin byte, u32 index)"
        return f"{elem_bytes(cfg)}-byte records ({k} key + u32 payload)"
    return k + ("+u32 payload" if c["kind"] == "pairs" else "")


def count(cfg, inp):
    """Elements (records) of one merge of the config."""
    if CONFIGS[cfg]["kind"] == "records":
        return inp["m"] + inp["n"]
    return inp["a"].numel() + inp["b"].numel()


def pack_records(keys, vals, rec=None):
    """Device {key, val} records as a (len, 2) tensor: int32 words for 32-bit
    keys, int64 words {key, val | pad << 32} (pad 0) for uint64 keys; rec=12:
    the reference's tagged<int32_t> as (len, 3) int32 words {key, origin (0 for
    A, 1 for B: the payload's top bit), index (the payload's low 31 bits)}."""
    import torch
    if rec == 12:
        v = vals.view(torch.int32)
        return torch.stack([keys.view(torch.int32), (v >> 31) & 1, v & 0x7FFFFFFF], 1).contiguous()
    if keys.dtype == torch.uint64:
        return torch.stack([keys.view(torch.int64), vals.to(torch.int64)], 1).contiguous()
    return torch.stack([keys.view(torch.int32), vals.view(torch.int32)], 1).contiguous()


def scaling_of(world, replicas):
    return "strong" if world > 1 and not replicas else "weak"


def config_dict(cfg, elements, world, split):
    """The `config` object of both arms' lines (identical by construction)."""
    if world == 1:
        par = "1 GPU"
    elif split:
        par = (f"{world} GPUs, one merge split by output rank (Algorithm 2, a worker per GPU, "
               "peer windows over NVLink)")
    else:
        par = f"{world} GPUs, independent instance per GPU"
    balg = 2 * elements * elem_bytes(cfg)
    return dict(workload=f"{cfg}: {CONFIGS[cfg]['desc']}", elements=int(elements),
                parallelism=par,
                l2=(f"inputs+outputs {balg / 2**30:.2f} GiB per step (> 126 MB L2); L2 also "
                    if balg > 126e6 else
                    f"inputs+outputs {balg / 2**20:.1f} MiB per step (fit in L2); L2 ")
                + "flushed between steps (512 MiB read, outside the timed events)")


# ------------------------------------------------------------------ inputs

def make_inputs(cfg, seed=SEED, device="cuda"):
    """Seeded inputs on the device (splitmix64 recipe of generate.cpp:17-29,
    the testkit library's generator, pinned to the reference's by test)."""
    import torch
    from paper_1303_4312_b200 import testkit as tk
    c = CONFIGS[cfg]
    tdt = {"int32": torch.int32, "uint64": torch.uint64}[c["dtype"]]
    if c["kind"] == "records":
        base = make_inputs(c["base"], seed, device)
        rec = dict(a=pack_records(base["a"], base["av"], c.get("rec")),
                   b=pack_records(base["b"], base["bv"], c.get("rec")),
                   m=base["a"].numel(), n=base["b"].numel())
        del base
        return rec
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


def make_host_inputs(cfg, seed=SEED):
    """The same seeded inputs generated on the host (the reference arm: no GPU,
    no package import) by the C restatement of the reference's generator
    (oracle/comerge_oracle.c, pinned against the reference's own generator by
    tests/test_oracle.py)."""
    from oracle.py import Port
    port = Port()
    c = CONFIGS[cfg]
    if c["kind"] == "records":  # the reference's own form of the key-value configs
        return make_host_inputs(c["base"], seed)
    dt = {"int32": np.int32, "uint64": np.uint64}[c["dtype"]]
    if c["kind"] == "segmented":
        sizes = port.generate_raw(seed, 2, 2 * c["nseg"], c["maxlen"]).astype(np.int64) + 1
        ms, ns = sizes[0::2], sizes[1::2]
        a_off = np.concatenate([[0], np.cumsum(ms)]).astype(np.uint64)
        b_off = np.concatenate([[0], np.cumsum(ns)]).astype(np.uint64)
        out = {"a_off": a_off, "b_off": b_off}
        for side, off, lane in (("a", a_off, 0), ("b", b_off, 1)):
            raw = port.generate_raw(seed, lane, int(off[-1]), c["width"]).astype(dt)
            for s in range(c["nseg"]):
                raw[int(off[s]):int(off[s + 1])].sort()
            out[side] = raw
        return out
    la, lb = (1, 0) if c.get("swapped") else (0, 1)
    h = dict(a=port.generate_sorted(dt, seed, la, c["m"], c["width"]),
             b=port.generate_sorted(dt, seed, lb, c["n"], c["width"]))
    if c["kind"] == "pairs":
        h["av"] = np.arange(c["m"], dtype=np.uint32)
        h["bv"] = np.arange(c["n"], dtype=np.uint32) | np.uint32(1 << 31)
    return h


def alloc_outputs(cfg, inp):
    """Outputs plus the merge's scratch workspace (queried, CUB-style)."""
    import torch
    import paper_1303_4312_b200._native as N
    total = count(cfg, inp)
    dev = inp["a"].device
    kind = {"int32": N.KEY_I32, "uint64": N.KEY_U64}[CONFIGS[cfg]["dtype"]]
    if CONFIGS[cfg]["kind"] == "records":
        if CONFIGS[cfg].get("rec") == 12:
            wsb = N.lib.comerge_cuda_records12_workspace_bytes(inp["m"], inp["n"])
        else:
            wsb = N.lib.comerge_cuda_records_workspace_bytes(inp["m"], inp["n"], kind)
        return dict(keys=torch.empty((total, inp["a"].shape[1]), dtype=inp["a"].dtype, device=dev),
                    ws=torch.empty(max(int(wsb), 256), dtype=torch.uint8, device=dev))
    out = dict(keys=torch.empty(total, dtype=inp["a"].dtype, device=dev))
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
    elif kind == "records":
        P.merge_records(inp["a"], inp["b"], out["keys"], key_dtype=CONFIGS[cfg]["dtype"],
                        workspace=ws, record_bytes=CONFIGS[cfg].get("rec"))
    else:
        P.merge_segmented(inp["a"], inp["a_off"], inp["b"], inp["b_off"], out["keys"],
                          workspace=ws)
    return out


KERNEL_NAMES = {1: "merge_tile_kernel (+ partition_kernel)", 3: "merge_pipe_kernel",
                4: "seg_merge_tile_kernel (+ seg_partition_kernel)",
                5: "merge_pipe_kernel (segmented)", 7: "merge_pipe_kernel (pieced range)",
                8: "merge_small_kernel"}


def launches_per_step(path):
    return 2 if path in (1, 4) else 1  # persistent / single kernels: one launch


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


class L2Flush:
    """Evicts L2 (126 MB) between steps by READING a 512 MiB buffer: the lines
    left in L2 are clean, so the next merge does not pay for writing back
    dirty flush lines (a write-based flush left up to ~126 MB dirty)."""

    def __init__(self, device):
        import torch
        self.buf = torch.zeros(512 * 2**20 // 8, dtype=torch.int64, device=device)
        self.sink = torch.zeros((), dtype=torch.int64, device=device)

    def __call__(self):
        import torch
        torch.sum(self.buf, dim=0, out=self.sink)


def time_steps(step, steps, warmup, device, flush, dist_ctx=None, clocks=False,
               kernel_events=True):
    """Device time of `step` (enqueues one unit of work on the current stream):
    per-step events on the launching stream, L2 flushed outside them; then the
    same steps with events recorded by the library right around the merge
    kernel (the roofline's kernel time)."""
    import torch
    import paper_1303_4312_b200._native as N
    stream = torch.cuda.current_stream(device)
    wev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    # warm-up steps are the timed step exactly (flush, events, merge), untimed
    for _ in range(max(warmup, 0)):
        flush()
        wev[0].record(stream)
        step()
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
        flush()
        ev[k][0].record(stream)
        step()
        ev[k][1].record(stream)
    torch.cuda.synchronize(device)
    if dist_ctx:
        dist_ctx.barrier()
    if sampler:
        sampler.__exit__()
    kern_ms = None
    if kernel_events:
        torch.cuda._sleep(int(2e8))
        for k in range(steps):
            flush()
            N.lib.comerge_cuda_set_kernel_events(ev[k][2], ev[k][3])
            step()
            N.lib.comerge_cuda_set_kernel_events(None, None)
        torch.cuda.synchronize(device)
        kern_ms = [raw_elapsed_ms(e[2], e[3]) for e in ev]
    step_ms = [e[0].elapsed_time(e[1]) for e in ev]
    return dict(step_ms=step_ms, kern_ms=kern_ms, path=N.lib.comerge_cuda_last_path(),
                clocks=sampler.summary() if sampler else None)


def time_config(cfg, steps, warmup, device, flush, seed=SEED, dist_ctx=None, clocks=False):
    inp = make_inputs(cfg, seed=seed, device=device)
    out = alloc_outputs(cfg, inp)
    res = time_steps(lambda: run_config(cfg, inp, out), steps, warmup, device, flush, dist_ctx,
                     clocks)
    res.update(total=count(cfg, inp), inp=inp, out=out)
    return res


def summarize(cfg, res, peak, n_units=1, max_step_total_ms=None):
    """n_units: instances merged per step over the whole job (replicas)."""
    total = res["total"]
    balg = 2 * total * elem_bytes(cfg)
    step_total = max_step_total_ms if max_step_total_ms is not None else sum(res["step_ms"])
    steps = len(res["step_ms"])
    ms_step = step_total / steps
    kern = statistics.mean(res["kern_ms"])
    return dict(
        workload=CONFIGS[cfg]["desc"], elements=total,
        elements_per_s=n_units * total * steps / (step_total * 1e-3),
        ms_per_step=ms_step, step_gbs=balg / (ms_step * 1e-3) / 1e9,
        merge_kernel_ms=kern, merge_kernel_gbs=balg / (kern * 1e-3) / 1e9,
        frac_of_peak=balg / (kern * 1e-3) / 1e9 / peak,
        step_frac_of_peak=balg / (ms_step * 1e-3) / 1e9 / peak,
        frac_of_8tbs=balg / (kern * 1e-3) / 8e12, algorithmic_bytes=balg,
        kernel=KERNEL_NAMES.get(res["path"], "?"), launches_per_step=launches_per_step(res["path"]))


# ------------------------------------------------------------- CPU legs

def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def with_aos(cfg, h):
    """Key-value configs in the reference's own call shape: {key, val} structs
    with a key-only less (oracle.hpp:22-37)."""
    if CONFIGS[cfg]["kind"] in ("pairs", "records") and "a_aos" not in h:
        from oracle.py import to_aos
        h["a_aos"] = to_aos(h["a"], h["av"])
        h["b_aos"] = to_aos(h["b"], h["bv"])
    return h


def cpu_reference_run(cfg, h, threads):
    """One run of the reference's CPU path on host arrays; returns (wall ns,
    kind): merge_report.wall_ns, the parallel region only (parallel.hpp:252-267).
    C5: the reference has no batched API -- pairs round-robin over `threads`
    std::threads, each calling comerge::stable_merge (merge.hpp:52-68)."""
    from oracle.py import Ref, available_ref, Port
    kind = CONFIGS[cfg]["kind"]
    if kind == "records" and CONFIGS[cfg].get("rec") == 12 and available_ref():
        # the reference's own tagged<int32_t> with tagged_key_less
        from oracle.py import KIND, tagged_dtype
        if "a_tag" not in h:
            for side, v in (("a", "av"), ("b", "bv")):
                t = np.zeros(len(h[side]), tagged_dtype(KIND[np.dtype(h[side].dtype)]))
                t["key"] = h[side]
                t["origin"] = (h[v] >> 31).astype(np.uint8)
                t["index"] = h[v] & np.uint32(0x7FFFFFFF)
                h[side + "_tag"] = t
        ref = Ref()
        o = h.setdefault("out_tag", np.zeros(len(h["a_tag"]) + len(h["b_tag"]), h["a_tag"].dtype))
        return ref.merge_parallel_tagged(h["a_tag"], h["b_tag"], threads, out=o)[1].wall_ns, \
            "reference"
    if kind == "records":
        kind = "pairs"
    if available_ref():
        ref = Ref()
        if kind == "segmented":
            o = h.setdefault("out", np.empty(len(h["a"]) + len(h["b"]), h["a"].dtype))
            return ref.merge_segmented(h["a"], h["a_off"], h["b"], h["b_off"], threads=threads,
                                       out=o)[1], "reference"
        if kind == "pairs":
            with_aos(cfg, h)
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


def cpu_sample(cfg, h, threads, budget_s, min_reps=3, max_reps=15):
    cpu_reference_run(cfg, h, threads)  # warm: touch output pages
    walls, kind = [], "reference"
    t_start = time.time()
    while len(walls) < max_reps and (len(walls) < min_reps or time.time() - t_start < budget_s):
        w, kind = cpu_reference_run(cfg, h, threads)
        walls.append(w)
    return walls, kind


def cpu_baseline(cfg, h, budget_s=4.0, p1_budget_s=8.0):
    """The reference at p = hardware_concurrency (the baseline) and p = 1 on
    the full workload: median (primary) and min of >= 3
    runs of merge_report.wall_ns."""
    total = len(h["a"]) + len(h["b"])
    threads = cpu_threads()
    walls, kind = cpu_sample(cfg, h, threads, budget_s)
    walls1, _ = cpu_sample(cfg, h, 1, p1_budget_s, min_reps=1, max_reps=5)
    med, med1 = statistics.median(walls), statistics.median(walls1)
    return dict(value=total / (med * 1e-9), unit="elements/s", cores=threads, kind=kind,
                sample=f"full {cfg} workload ({total} elements), median of {len(walls)} runs of "
                       f"the reference's merge_report.wall_ns at {threads} threads "
                       "(std::thread::hardware_concurrency)"
                       + ("; pairs round-robin over the threads, stable_merge each (no batched "
                          "reference API)" if CONFIGS[cfg]["kind"] == "segmented" else ""),
                median_ms=med / 1e6, min_ms=min(walls) / 1e6,
                p1=dict(value=total / (med1 * 1e-9), median_ms=med1 / 1e6,
                        min_ms=min(walls1) / 1e6, runs=len(walls1)),
                cpu_model=cpu_model())


# ------------------------------------------------------------------- e2e

def e2e_measure(cfg, inp, steps, warmup):
    """The same metric through the host-buffer C ABI (comerge_merge_parallel_*
    / comerge_merge_segmented_host_*): pinned host inputs, H2D + merge + D2H
    inside every timed call; the result must equal the device path's."""
    import torch
    import paper_1303_4312_b200._native as N
    c = CONFIGS[cfg]
    suf = {"int32": "i32", "uint64": "u64"}[c["dtype"]]
    pin = {k: v.cpu().pin_memory() for k, v in inp.items() if hasattr(v, "cpu")}
    total = inp["a"].numel() + inp["b"].numel()
    ok = torch.empty(total, dtype=inp["a"].dtype).pin_memory()
    ov = torch.empty(total, dtype=torch.uint32).pin_memory() if c["kind"] == "pairs" else None
    rep = N.MergeReport()
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

    if c["kind"] == "records":
        total = count(cfg, inp)
        fname = f"comerge_merge_parallel_records{'12' if c.get('rec') == 12 else ''}_{suf}"
        path = f"{fname} (host pinned buffers)"
        ok = torch.empty((total, inp["a"].shape[1]), dtype=inp["a"].dtype).pin_memory()

        def call():
            N.check(getattr(N.lib, fname)(
                p(pin["a"]), inp["m"], p(pin["b"]), inp["n"], p(ok), total, 1, 0, C.byref(rep),
                None, None))
    elif c["kind"] == "segmented":
        fn = getattr(N.lib, f"comerge_merge_segmented_host_{suf}", None)
        if fn is None:
            return None
        nseg = pin["a_off"].numel() - 1
        path = f"comerge_merge_segmented_host_{suf} (host pinned buffers)"

        def call():
            N.check(fn(p(pin["a"]), p(pin["a_off"]), pin["a"].numel(), p(pin["b"]),
                       p(pin["b_off"]), pin["b"].numel(), nseg, p(ok), total, C.byref(rep)))
    elif c["kind"] == "pairs":
        path = f"comerge_merge_parallel_pairs_{suf} (host pinned buffers)"

        def call():
            N.check(getattr(N.lib, f"comerge_merge_parallel_pairs_{suf}")(
                p(pin["a"]), p(pin["av"]), pin["a"].numel(), p(pin["b"]), p(pin["bv"]),
                pin["b"].numel(), p(ok), p(ov), total, 1, C.byref(rep)))
    else:
        path = f"comerge_merge_parallel_{suf} (host pinned buffers)"

        def call():
            N.check(getattr(N.lib, f"comerge_merge_parallel_{suf}")(
                p(pin["a"]), pin["a"].numel(), p(pin["b"]), pin["b"].numel(), p(ok), total, 1,
                0, C.byref(rep), None, None))

    # warm-up: at least `warmup` calls and 200 ms of them -- the first calls
    # of a process on small configs ran ~2x slower (C1: 0.78 vs 0.37 ms for
    # the first ~10 calls; copy engines / clocks ramping after the device
    # benches), which a single warm-up call left inside the timed calls
    t_w = time.perf_counter()
    n_w = 0
    while n_w < max(1, warmup) or time.perf_counter() - t_w < 0.2:
        call()
        n_w += 1
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    dev = run_config(cfg, inp)
    torch.cuda.synchronize()
    assert bool((ok.view(torch.uint8) == dev["keys"].cpu().view(torch.uint8)).all()), "e2e keys"
    if ov is not None:
        assert bool((ov == dev["vals"].cpu()).all()), "e2e payloads"
    med = statistics.median(times)
    return dict(value=total / med, unit="elements/s", stat=f"median of {steps} calls",
                h2d_bytes_per_step=int(rep.h2d_bytes), d2h_bytes_per_step=int(rep.d2h_bytes),
                ms_per_step=1e3 * med, path=path, calls_ms=[round(1e3 * t, 3) for t in times])


# ------------------------------------------------------------------ main

def dist_setup():
    """One process per GPU (NCCL for the control plane: barriers and the
    max-over-ranks of the step times; the data path has no collective).  With
    fewer GPUs than ranks (a test run of the multi-GPU line on one GPU) ranks
    share devices and the control plane runs over gloo (NCCL refuses two ranks
    on one device); the ranks' kernels never wait on each other."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world <= 1:
        return None, 0, 1, 0
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = torch.cuda.device_count()
    dev_index = local % ndev
    torch.cuda.set_device(dev_index)
    if ndev >= world:
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev_index))
    else:
        dist.init_process_group("gloo")
    return dist, dist.get_rank(), world, dev_index


def shared_devices(dist):
    """Ranks share GPUs (fewer devices than ranks: a functional run of the
    multi-GPU line).  Their kernels then time-slice one device, so a job time
    is the SUM of the ranks' times, not the max."""
    import torch
    return dist is not None and torch.cuda.device_count() < dist.get_world_size()


def allreduce_time(dist, values, device):
    """Job time of a few per-rank times: max over ranks, or the sum when ranks
    share a device (on the device under NCCL, host under gloo)."""
    import torch
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor(values, dtype=torch.float64, device=device if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM if shared_devices(dist) else dist.ReduceOp.MAX)
    return [float(x) for x in t.cpu().tolist()]


def relaunch_under_torchrun(n):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def reference_arm(args):
    """CPU only: the compiled reference on host-generated inputs (this arm
    never imports the package, torch or CUDA)."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    cfg = args.config
    h = make_host_inputs(cfg)
    threads = cpu_threads()
    for _ in range(max(args.warmup, 1)):
        cpu_reference_run(cfg, h, threads)
    walls, kind = [], "reference"
    for _ in range(args.steps):
        w, kind = cpu_reference_run(cfg, h, threads)
        walls.append(w)
    total = len(h["a"]) + len(h["b"])
    # same statistic as the GPU arm: total work / total time of the K steps
    value = total * len(walls) / (sum(walls) * 1e-9)
    line = dict(metric=METRIC, value=value, unit="elements/s", n_gpus=world,
                steps=args.steps, warmup=args.warmup,
                ms_per_step=sum(walls) / len(walls) / 1e6, higher_is_better=True,
                scaling=scaling_of(world, args.replicas),
                vs_baseline=None, dtype=dtype_str(cfg), data="synthetic (seeded splitmix64, "
                "generate.cpp recipe)", impl="reference",
                config=config_dict(cfg, total, world, world > 1 and not args.replicas),
                cpu_baseline=dict(value=value, unit="elements/s", cores=threads, kind=kind,
                                  sample=f"full {cfg} workload per step: reference "
                                         "comerge::merge_parallel"
                                         + (" ({key,val} structs, key-only less)"
                                            if CONFIGS[cfg]["kind"] == "pairs" else "")
                                         + f" at {threads} threads, merge_report.wall_ns",
                                  cpu_model=cpu_model()),
                e2e=dict(value=value, unit="elements/s", h2d_bytes_per_step=0,
                         d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


def sort_extras(device, flush, reps=5):
    """SURVEY 8f row 1 (not a BASELINE config): the stable merge sorts on
    2^26 int32 keys (uniform 31-bit, seeded) with and without uint32 payloads,
    median device time (events, L2 flushed before each rep), next to CUB's
    merge and radix sorts of the same keys (library baselines, testkit)."""
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

    def med(fn):
        ts = []
        for r in range(reps + 2):
            flush()
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
    # library baselines on the same keys (CUB, in the testkit library)
    tkl = N.tk()
    need = int(tkl.comerge_testkit_cub_sort_bytes(n))
    tmp = torch.empty(max(need, 1), dtype=torch.uint8, device=device)
    for alg, name in {0: "cub_radix_keys", 1: "cub_radix_pairs", 2: "cub_merge_keys",
                      3: "cub_merge_pairs"}.items():
        def run(alg=alg):
            N.check(tkl.comerge_testkit_cub_sort(
                alg, C.c_void_p(k.data_ptr()), C.c_void_p(v.data_ptr()), C.c_void_p(ok.data_ptr()),
                C.c_void_p(ov.data_ptr()), n, C.c_void_p(tmp.data_ptr()), need, None), True)
        out[f"{name}_ms"] = med(run)
    del tmp
    del k, v, ok, ov, ws
    torch.cuda.empty_cache()
    return out


def split_e2e(dm, local, dist, device, calls, total_bytes):
    """End to end at N GPUs: every call copies each rank's input pieces from
    pinned host memory to its GPU, waits until every rank's pieces are in place
    (the peers read them over NVLink), runs the rank's range merge and copies
    its output range back to pinned host memory.  Wall clock between barriers,
    max over ranks; median of the calls after two warm-up calls."""
    import torch
    host = [x.cpu().pin_memory() for x in local]
    outs = [dm.out] + ([dm.out_vals] if dm.out_vals is not None else [])
    hout = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]
    times = []
    for it in range(calls + 2):
        torch.cuda.synchronize(device)
        dist.barrier()
        t0 = time.perf_counter()
        for d, h in zip(local, host):
            d.copy_(h, non_blocking=True)
        torch.cuda.synchronize(device)
        dist.barrier()  # every rank's pieces are resident before any rank's kernel reads them
        dm.run()
        for h, o in zip(hout, outs):
            h.copy_(o, non_blocking=True)
        torch.cuda.synchronize(device)
        dt = time.perf_counter() - t0
        # wall clock between barriers spans every rank's work: max over ranks
        on_dev = dist.get_backend() == "nccl"
        w = torch.tensor([dt], dtype=torch.float64, device=device if on_dev else "cpu")
        dist.all_reduce(w, op=dist.ReduceOp.MAX)
        job = float(w.cpu()[0])
        if it >= 2:
            times.append(job)
    med = statistics.median(times)
    return dict(value=dm.total / med, unit="elements/s",
                stat=f"median of {calls} calls, max over ranks",
                h2d_bytes_per_step=int(total_bytes), d2h_bytes_per_step=int(total_bytes),
                ms_per_step=1e3 * med,
                path="per rank: H2D of its pieces, range merge over peer windows "
                     "(comerge_cuda_merge_*_pieces_*), D2H of its output range")


def run_split(args, dist, rank, world, device, peak, flush):
    """ONE merge of the config split across the ranks (Algorithm 2 with a
    worker per GPU): rank r holds the r-th piece of A and B (cut at r/world,
    a multiple of 4 elements) and merges its output range, reading the peers'
    pieces over NVLink.  value = the whole merge / the max over ranks."""
    import torch
    from paper_1303_4312_b200.shard import DistributedMerge
    cfg = args.config
    if CONFIGS[cfg]["kind"] in ("segmented", "records"):
        raise SystemExit("--split: plain keys / key-value merges only (use --replicas)")
    full = make_inputs(cfg, seed=SEED, device=device)

    def piece(t, length):
        lo = (length * rank // world) // 4 * 4
        hi = length if rank == world - 1 else (length * (rank + 1) // world) // 4 * 4
        return t[lo:hi].clone()

    m, n = full["a"].numel(), full["b"].numel()
    pa, pb = piece(full["a"], m), piece(full["b"], n)
    pav = piece(full["av"], m) if "av" in full else None
    pbv = piece(full["bv"], n) if "bv" in full else None
    del full
    torch.cuda.empty_cache()
    try:  # CUDA IPC / peer access between the ranks' GPUs
        dm, err = DistributedMerge(pa, pb, a_vals=pav, b_vals=pbv), None
    except Exception as e:  # noqa: BLE001 -- every rank must learn of any rank's failure
        dm, err = None, repr(e)
    if allreduce_time(dist, [0.0 if err is None else 1.0], device)[0] > 0:
        if dm is not None:
            dm.close()
        print(f"bench.py rank {rank}: split setup failed ({err or 'on a peer rank'}); "
              "falling back to replicas", file=sys.stderr, flush=True)
        return False

    class Ctx:
        def barrier(self):
            dist.barrier()

    res = time_steps(dm.run, args.steps, args.warmup, device, flush, Ctx(), clocks=(rank == 0))
    step_total, kern = allreduce_time(dist, [sum(res["step_ms"]), statistics.mean(res["kern_ms"])],
                                      device)
    if shared_devices(dist):  # per-rank kernel time: the summed one over the ranks
        kern /= world
    e2e = split_e2e(dm, [x for x in (pa, pb, pav, pbv) if x is not None], dist, device,
                    max(3, min(args.steps, 9)), (m + n) * elem_bytes(cfg))
    dm.close()
    total = m + n
    balg = 2 * total * elem_bytes(cfg)
    if rank == 0:
        ms = step_total / args.steps
        line = dict(
            metric=METRIC, value=total * args.steps / (step_total * 1e-3), unit="elements/s",
            n_gpus=world, steps=args.steps, warmup=args.warmup, ms_per_step=ms,
            higher_is_better=True, scaling="strong", vs_baseline=None, dtype=dtype_str(cfg),
            data="synthetic (seeded splitmix64, generate.cpp recipe)",
            config=config_dict(cfg, total, world, True),
            roofline=dict(bound="hbm", achieved=balg / world / (kern * 1e-3) / 1e9, peak=peak,
                          unit="GB/s", frac=balg / world / (kern * 1e-3) / 1e9 / peak,
                          traffic=None, kernel="merge_pipe_kernel (pieced range, per rank)",
                          algorithmic_bytes_per_launch=balg // world),
            cpu_baseline=None, e2e=e2e, clocks=res["clocks"],
            gpu_launches=args.steps * launches_per_step(res["path"]))
        if shared_devices(dist):
            line["note"] = (f"{world} ranks on {torch.cuda.device_count()} GPU(s): a functional run "
                            "of the split; ranks time-slice the device, job time = sum of ranks")
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    # defaults: a 50-step timed region (~55 ms for C4) keeps one host-side hiccup
    # of a millisecond or two (seen once: 20 steps at 1.090 instead of 1.004 ms)
    # within a few percent of the whole-job figure
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default=HEADLINE, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: an independent instance per GPU instead of one split merge")
    ap.add_argument("--only-headline", action="store_true", help="skip the per-config table")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline legs")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sorts", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return reference_arm(args)
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        return sys.exit(relaunch_under_torchrun(args.gpus))
    if env_world is not None and int(env_world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}")

    import torch
    dist, rank, world, local = dist_setup()
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    peak, peak_src = peak_hbm()
    flush = L2Flush(device)
    split_failed = False
    if world > 1 and not args.replicas:
        if run_split(args, dist, rank, world, device, peak, flush) is not False:
            dist.barrier()
            dist.destroy_process_group()
            return
        split_failed = True

    class Ctx:
        def barrier(self):
            if dist:
                dist.barrier()

    ctx = Ctx() if dist else None
    cfg = args.config
    res = time_config(cfg, args.steps, args.warmup, device, flush, seed=SEED + rank,
                      dist_ctx=ctx, clocks=(rank == 0))
    step_total = sum(res["step_ms"])
    if dist:
        step_total = allreduce_time(dist, [step_total], device)[0]
    head = summarize(cfg, res, peak, n_units=world, max_step_total_ms=step_total)
    legs = rank == 0 and world == 1  # CPU / e2e legs: rank 0 at N = 1 only

    def extras(c, r):
        d = {}
        if legs and not args.no_e2e:
            d["e2e"] = e2e_measure(c, r["inp"], max(5, min(args.steps, 9)), 1)
        if legs and not args.no_cpu:
            if CONFIGS[c].get("rec") == 12:  # the reference's own tagged<int32_t> merge
                d["cpu_baseline"] = cpu_baseline(c, make_host_inputs(CONFIGS[c]["base"]))
            elif CONFIGS[c]["kind"] == "records":  # the reference's call is this record form
                d["cpu_baseline"] = f"same as {CONFIGS[c]['base']} (the reference merges its " \
                                    "{key, val} structs there)"
            else:
                d["cpu_baseline"] = cpu_baseline(c, {k: v.cpu().numpy()
                                                     for k, v in r["inp"].items()})
        return d

    head_extras = extras(cfg, res)
    per_config = {}
    if not args.only_headline:
        for other in CONFIGS:
            if other == cfg:
                per_config[other] = dict(head, elements_per_s=head["elements_per_s"] / world,
                                         **head_extras)
                continue
            r = time_config(other, min(args.steps, 10), 3, device, flush, seed=SEED + rank)
            per_config[other] = dict(summarize(other, r, peak), **extras(other, r))
            del r
            torch.cuda.empty_cache()
    del res["inp"], res["out"]
    torch.cuda.empty_cache()
    sorts = None if args.only_headline or args.no_sorts else sort_extras(device, flush)
    if rank == 0:
        line = dict(
            metric=METRIC, value=head["elements_per_s"], unit="elements/s",
            n_gpus=world, steps=args.steps, warmup=args.warmup, ms_per_step=head["ms_per_step"],
            higher_is_better=True, scaling="weak", vs_baseline=None, dtype=dtype_str(cfg),
            data="synthetic (seeded splitmix64, generate.cpp recipe)",
            config=config_dict(cfg, head["elements"], world, False),
            roofline=dict(bound="hbm", achieved=head["merge_kernel_gbs"], peak=peak,
                          unit="GB/s", frac=head["frac_of_peak"], traffic=traffic_for(cfg),
                          kernel=head["kernel"], peak_source=peak_src,
                          algorithmic_bytes_per_launch=head["algorithmic_bytes"],
                          step_gbs=head["step_gbs"], frac_of_8tbs=head["frac_of_8tbs"]),
            cpu_baseline=head_extras.get("cpu_baseline"), e2e=head_extras.get("e2e"),
            clocks=res["clocks"], gpu_launches=args.steps * head["launches_per_step"],
            configs=per_config, sorts=sorts)
        if world > 1:
            line["scaling_note"] = "replicas: an independent instance per GPU (seed + rank)"
            if split_failed:
                line["scaling_note"] += "; the split of one merge could not set up peer access"
            if shared_devices(dist):
                line["note"] = (f"{world} ranks on {torch.cuda.device_count()} GPU(s): a functional "
                                "run; ranks time-slice the device, job time = sum of ranks")
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
