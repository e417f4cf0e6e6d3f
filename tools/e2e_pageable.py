"""The host-buffer merge (comerge_merge_parallel_pairs_* / _i32 ...) with
PAGEABLE host arrays (what a reference caller's std::vector is) next to pinned
ones.     python tools/e2e_pageable.py C4 C2"""
import ctypes as C
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1303_4312_b200._native as N  # noqa: E402

p = lambda t: C.c_void_p(t.ctypes.data if isinstance(t, np.ndarray) else t.data_ptr())  # noqa: E731
for cfg in sys.argv[1:]:
    c = bench.CONFIGS[cfg]
    inp = bench.make_inputs(cfg, device=torch.device("cuda:0"))
    suf = {"int32": "i32", "uint64": "u64"}[c["dtype"]]
    for kind in ("pageable", "pinned"):
        h = {k: (v.cpu().numpy() if kind == "pageable" else v.cpu().pin_memory())
             for k, v in inp.items()}
        if "a_off" in h and kind == "pinned":  # offsets: host arrays either way
            h["a_off"], h["b_off"] = inp["a_off"].cpu().numpy(), inp["b_off"].cpu().numpy()
        total = len(h["a"]) + len(h["b"])
        mk = (lambda n, dt: np.empty(n, dt)) if kind == "pageable" else \
            (lambda n, dt: torch.empty(n, dtype={np.int32: torch.int32, np.uint64: torch.uint64,
                                                 np.uint32: torch.uint32}[dt]).pin_memory())
        kdt = np.uint64 if c["dtype"] == "uint64" else np.int32
        ok = mk(total, kdt)
        rep = N.MergeReport()
        if c["kind"] == "segmented":
            fn = getattr(N.lib, f"comerge_merge_segmented_host_{suf}")
            nseg = len(h["a_off"]) - 1
            call = lambda: N.check(fn(p(h["a"]), p(h["a_off"]), len(h["a"]), p(h["b"]),  # noqa: E731
                                      p(h["b_off"]), len(h["b"]), nseg, p(ok), total, C.byref(rep)))
        elif c["kind"] == "pairs":
            ov = mk(total, np.uint32)
            fn = getattr(N.lib, f"comerge_merge_parallel_pairs_{suf}")
            call = lambda: N.check(fn(p(h["a"]), p(h["av"]), len(h["a"]), p(h["b"]), p(h["bv"]),  # noqa: E731
                                      len(h["b"]), p(ok), p(ov), total, 1, C.byref(rep)))
        else:
            fn = getattr(N.lib, f"comerge_merge_parallel_{suf}")
            call = lambda: N.check(fn(p(h["a"]), len(h["a"]), p(h["b"]), len(h["b"]), p(ok), total,  # noqa: E731
                                      1, 0, C.byref(rep), None, None))
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.3:
            call()
        ts = []
        for _ in range(5):
            t = time.perf_counter()
            call()
            ts.append(time.perf_counter() - t)
        print(f"{cfg} {kind:8s} e2e {1e3 * statistics.median(ts):8.2f} ms", flush=True)
