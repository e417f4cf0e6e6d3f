import ctypes as C, time, numpy as np
rt = C.CDLL("libcudart.so.12")
rt.cudaFree(None)
for gb in (0.25, 1, 2):
    a = np.ones(int(gb * 2**30), np.uint8)  # touched
    t = time.perf_counter(); rc = rt.cudaHostRegister(C.c_void_p(a.ctypes.data), C.c_size_t(a.nbytes), 0); t1 = time.perf_counter()
    rc2 = rt.cudaHostUnregister(C.c_void_p(a.ctypes.data)); t2 = time.perf_counter()
    print(f"{gb} GB: register {1e3*(t1-t):.1f} ms ({a.nbytes/(t1-t)/1e9:.1f} GB/s) rc={rc}, unregister {1e3*(t2-t1):.1f} ms")
