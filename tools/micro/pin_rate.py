"""H2D / D2H rates of torch-pinned tensors vs cudaHostAlloc'd memory (one large copy each)."""
import ctypes as C
import time
import torch

n = 268435456
rt = C.CDLL("libcudart.so.12") if False else None
dev = torch.empty(n, dtype=torch.uint8, device="cuda")
dev2 = torch.empty(n, dtype=torch.uint8, device="cuda")
pinned = torch.empty(n, dtype=torch.uint8).pin_memory()
pinned2 = torch.empty(n, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(name, fn):
    best = 1e9
    for r in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if r:
            best = min(best, dt)
    print(f"{name:40s} {best * 1e3:7.3f} ms  {n / best / 1e9:6.1f} GB/s")


t("torch pinned H2D", lambda: dev.copy_(pinned, non_blocking=True))
t("torch pinned D2H", lambda: pinned2.copy_(dev2, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        dev.copy_(pinned, non_blocking=True)
    with torch.cuda.stream(s2):
        pinned2.copy_(dev2, non_blocking=True)


t("torch pinned H2D || D2H", both)
