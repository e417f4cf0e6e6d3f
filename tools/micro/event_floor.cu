// Event-timed floor of a kernel launch in the bench's pattern (L2-flush
// kernel, event, kernel, event): empty kernels of several grid / block /
// shared-memory shapes, vs the small-merge kernel's C1 time.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/micro/event_floor tools/micro/event_floor.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void flush_read(const int4* p, size_t n, int* sink) {
    int acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        acc ^= p[i].x;
    if (acc == 0x7fffffff) *sink = acc;
}
__global__ void empty_k(int* p) {
    extern __shared__ int sm[];
    if (threadIdx.x == 0 && p == nullptr) sm[0] = 1;
}
__global__ void write_k(int4* out, size_t per_cta) {
    int4* o = out + blockIdx.x * per_cta;
    for (size_t i = threadIdx.x; i < per_cta; i += blockDim.x) o[i] = make_int4(int(i), 1, 2, 3);
}

int main() {
    int4* buf;
    const size_t n = size_t(512) << 16;  // 512 MiB of int4
    cudaMalloc(&buf, n * 16);
    cudaMemset(buf, 0, n * 16);
    int* sink;
    cudaMalloc(&sink, 64);
    int4* wbuf;
    cudaMalloc(&wbuf, size_t(64) << 20);
    cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct cfg { int grid, block, smem_kb, write_mb; };
    for (cfg c : {cfg{1, 32, 0, 0}, cfg{148, 256, 0, 0}, cfg{265, 256, 40, 0}, cfg{296, 384, 100, 0},
                  cfg{265, 256, 40, 8}, cfg{265, 256, 0, 8}}) {
        std::vector<float> t;
        for (int r = 0; r < 30; ++r) {
            flush_read<<<1184, 512>>>(buf, n, sink);
            cudaEventRecord(e0);
            if (c.write_mb)
                write_k<<<c.grid, c.block>>>(wbuf, ((size_t(c.write_mb) << 20) / 16) / c.grid);
            else
                empty_k<<<c.grid, c.block, c.smem_kb * 1024>>>(sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r >= 5) t.push_back(ms * 1e3f);
        }
        std::sort(t.begin(), t.end());
        printf("grid %3d block %3d smem %3d KB write %d MB: event time median %.2f us, min %.2f (%s)\n",
               c.grid, c.block, c.smem_kb, c.write_mb, t[t.size() / 2], t[0],
               cudaGetErrorString(cudaGetLastError()));
    }
}
