// Launch/teardown gaps of a persistent-grid kernel vs its configuration:
// marker kernel -> probe kernel (296 CTAs x 384 threads, first-CTA start and
// last-CTA end by globaltimer) -> marker kernel, optionally after a fill
// kernel (the bench's L2 flush).  Does the dynamic shared memory size (and the
// carve-out switch it forces after a kernel without shared memory) matter?
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/micro/launch_cfg tools/micro/launch_cfg.cu
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>

__global__ void marker(unsigned long long* t) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    *t = g;
}
__global__ void fill(int* p, size_t n, int v) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
        p[i] = v;
}
__global__ void writer(unsigned long long* t, uint4* out, size_t per_cta16) {
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    uint4* o = out + blockIdx.x * per_cta16;
    for (size_t i = threadIdx.x; i < per_cta16; i += blockDim.x) o[i] = make_uint4(unsigned(i), 1, 2, 3);
    __syncthreads();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (threadIdx.x == 0) {
        t[2 * blockIdx.x] = g0;
        t[2 * blockIdx.x + 1] = g1;
    }
}
__global__ void probe(unsigned long long* t, int work_ns) {
    extern __shared__ unsigned char smem[];
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    if (work_ns) {
        for (;;) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
            if (g1 - g0 >= (unsigned long long)work_ns) break;
        }
    }
    if (threadIdx.x == 0) smem[0] = 1;
    __syncthreads();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    if (threadIdx.x == 0) {
        t[2 * blockIdx.x] = g0;
        t[2 * blockIdx.x + 1] = g1 + smem[0] - 1;
    }
}

int main() {
    unsigned long long *t, *mk;
    cudaMalloc(&t, 2 * 4096 * 8);
    cudaMalloc(&mk, 64);
    int* buf;
    const size_t nfill = size_t(512) << 18;  // 512 MiB of int
    cudaMalloc(&buf, nfill * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    uint4* wbuf;
    cudaMalloc(&wbuf, size_t(600) << 20);
    for (int withfill : {0, 1})
        for (size_t mb : {size_t(0), size_t(9), size_t(100), size_t(537)}) {
            std::vector<double> a, b, c, ev;
            for (int r = 0; r < 8; ++r) {
                if (withfill) fill<<<1184, 512>>>(buf, nfill, r);
                cudaEventRecord(e0);
                marker<<<1, 1>>>(mk);
                writer<<<296, 384>>>(t, wbuf, ((mb << 20) / 296) / 16);
                marker<<<1, 1>>>(mk + 1);
                cudaEventRecord(e1);
                cudaDeviceSynchronize();
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                std::vector<unsigned long long> h(2 * 296), hm(2);
                cudaMemcpy(h.data(), t, h.size() * 8, cudaMemcpyDeviceToHost);
                cudaMemcpy(hm.data(), mk, 16, cudaMemcpyDeviceToHost);
                unsigned long long s0 = ~0ull, e_max = 0;
                for (int k = 0; k < 296; ++k) {
                    s0 = std::min(s0, h[2 * k]);
                    e_max = std::max(e_max, h[2 * k + 1]);
                }
                if (r >= 2) {
                    a.push_back((s0 - hm[0]) / 1e3);
                    b.push_back((e_max - s0) / 1e3);
                    c.push_back((hm[1] - e_max) / 1e3);
                    ev.push_back(ms * 1e3);
                }
            }
            auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
            printf("fill %d writes %3zu MB: marker->first CTA %.2f us, span %.2f, last end->marker %.2f, events %.2f (%s)\n",
                   withfill, mb, med(a), med(b), med(c), med(ev), cudaGetErrorString(cudaGetLastError()));
        }
}
