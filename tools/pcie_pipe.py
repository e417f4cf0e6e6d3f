"""Copy-engine pipeline floor: chunked H2D (stream 1) overlapped with D2H
(stream 2), C2's bytes (268 MB each way), uniform and ramped chunk sizes."""
import time
import torch

n = 268435456  # bytes each way (C2: 2^25 x (4+4) B)
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def ramp(parts, ends):
    """parts equal middle chunks; `ends` halvings at both ends"""
    w = [2.0 ** -(ends - k) for k in range(ends)] + [1.0] * parts + [2.0 ** -(k + 1) for k in range(ends)]
    s = sum(w)
    cuts = [0]
    acc = 0.0
    for x in w:
        acc += x
        cuts.append(min(n, int(round(acc / s * n / 4096)) * 4096))
    cuts[-1] = n
    return cuts


def timeit(cuts, split=1):
    C = len(cuts) - 1
    evs = [torch.cuda.Event() for _ in range(C)]

    def run():
        for c in range(C):
            lo, hi = cuts[c], cuts[c + 1]
            with torch.cuda.stream(s1):
                step = (hi - lo) // split
                for q in range(split):
                    a, b = lo + q * step, (hi if q == split - 1 else lo + (q + 1) * step)
                    d_in[a:b].copy_(h_in[a:b], non_blocking=True)
                evs[c].record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(evs[c])
                h_out[lo:hi].copy_(d_out[lo:hi], non_blocking=True)
        torch.cuda.synchronize()

    run()
    t0 = time.perf_counter()
    for _ in range(5):
        run()
    return (time.perf_counter() - t0) / 5 * 1e3


for C in (4, 8, 16, 32):
    print(f"uniform chunks {C}: {timeit([n * c // C for c in range(C + 1)]):.2f} ms")
print(f"uniform 8, 4 copies in per chunk: {timeit([n * c // 8 for c in range(9)], split=4):.2f} ms")
for parts, ends in ((4, 3), (6, 3), (8, 4), (6, 5)):
    cuts = ramp(parts, ends)
    print(f"ramp parts {parts} ends {ends} ({len(cuts) - 1} chunks): {timeit(cuts):.2f} ms")
