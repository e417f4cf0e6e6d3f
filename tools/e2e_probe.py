"""Time the host-buffer C-ABI merge (C2 shape) end to end."""
import ctypes as C, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1303_4312_b200._native as N
dev = torch.device("cuda:0")
inp = bench.make_inputs("C2", device=dev)
tot = inp["a"].numel() + inp["b"].numel()
if os.environ.get("HOSTALLOC"):  # cudaHostAlloc'd host arrays instead of torch's pinned allocator
    import numpy as np
    rt = C.CDLL("libcudart.so.12")
    def halloc(n, dt):
        p_ = C.c_void_p()
        assert rt.cudaHostAlloc(C.byref(p_), C.c_size_t(n * 4), 0) == 0
        arr = np.ctypeslib.as_array(C.cast(p_, C.POINTER(C.c_uint32)), shape=(n,))
        return torch.from_numpy(arr).view(dt)
    pin = {}
    for k, v in inp.items():
        pin[k] = halloc(v.numel(), v.dtype); pin[k].copy_(v.cpu())
    ok = halloc(tot, torch.int32); ov = halloc(tot, torch.uint32)
else:
    pin = {k: v.cpu().pin_memory() for k, v in inp.items()}
    ok = torch.empty(tot, dtype=torch.int32).pin_memory(); ov = torch.empty(tot, dtype=torch.uint32).pin_memory()
p = lambda t: C.c_void_p(t.data_ptr())
rep = N.MergeReport()
def call():
    N.check(N.lib.comerge_merge_parallel_pairs_i32(p(pin["a"]), p(pin["av"]), pin["a"].numel(), p(pin["b"]), p(pin["bv"]), pin["b"].numel(), p(ok), p(ov), tot, 1, C.byref(rep)))
N.lib.comerge_cuda_set_host_mode(int(os.environ.get("HOST_MODE", "0")))
call()
ts = []
for _ in range(5):
    t0 = time.perf_counter(); call(); ts.append(time.perf_counter() - t0)
ref = bench.run_config("C2", inp)
torch.cuda.synchronize()
assert torch.equal(ok, ref["keys"].cpu()) and torch.equal(ov.view(torch.int32), ref["vals"].cpu().view(torch.int32)), "e2e mismatch"
print(os.environ.get("HOST_MODE"), os.environ.get("COMERGE_HOST_CHUNKS"), "e2e ms", [round(t*1e3, 2) for t in ts], "merge span ms", rep.wall_ns/1e6, "e2e_ns", rep.e2e_ns/1e6)
