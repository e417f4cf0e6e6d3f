"""Copy-engine pipeline floor: chunked H2D (stream 1) overlapped with D2H (stream 2)."""
import time, torch
n = 268435456  # bytes each way (C2: 2^25 x (4+4) B)
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda"); d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for C in (4, 8, 16, 32):
    ch = n // C
    evs = [torch.cuda.Event() for _ in range(C)]
    def run():
        for c in range(C):
            with torch.cuda.stream(s1):
                d_in[c*ch:(c+1)*ch].copy_(h_in[c*ch:(c+1)*ch], non_blocking=True); evs[c].record(s1)
            with torch.cuda.stream(s2):
                s2.wait_event(evs[c]); h_out[c*ch:(c+1)*ch].copy_(d_out[c*ch:(c+1)*ch], non_blocking=True)
        torch.cuda.synchronize()
    run()
    t0 = time.perf_counter(); [run() for _ in range(5)]; t = (time.perf_counter() - t0) / 5
    print(f"chunks {C}: {t*1e3:.2f} ms for {n/1e6:.0f} MB each way")
