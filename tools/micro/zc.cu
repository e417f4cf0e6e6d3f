// PCIe paths on this box: kernel-driven writes to / reads from pinned host
// memory (zero-copy), alone and concurrently with a copy-engine transfer.
#include <cstdio>
#include <cstdint>
#include <chrono>
#include <cuda_runtime.h>
__global__ void zc_write(uint4* dst, size_t n16) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
        dst[i] = make_uint4(uint32_t(i), 1, 2, 3);
}
__global__ void zc_read(const uint4* src, size_t n16, uint32_t* sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
        uint4 v = src[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}
__global__ void zc_copy(const uint4* src, uint4* dst, size_t n16) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}
int main() {
    const size_t B = size_t(256) << 20;
    void *h1, *h2, *d1, *d2; uint32_t* sink;
    cudaHostAlloc(&h1, B, cudaHostAllocMapped); cudaHostAlloc(&h2, B, cudaHostAllocMapped);
    cudaMalloc(&d1, B); cudaMalloc(&d2, B); cudaMalloc(&sink, 4);
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const size_t n16 = B / 16;
    auto t = [&](const char* name, auto fn) {
        float best = 1e9;
        for (int r = 0; r < 4; ++r) {
            cudaDeviceSynchronize();
            auto t0 = std::chrono::steady_clock::now();
            fn();
            cudaDeviceSynchronize();
            float ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (r) best = ms < best ? ms : best;
        }
        printf("%-52s %7.3f ms  %6.1f GB/s per 256 MiB\n", name, best, B / best / 1e6);
    };
    for (int grid : {148, 296, 592, 1184}) {
        char nm[96];
        snprintf(nm, sizeof nm, "kernel writes host (grid %d x 256)", grid);
        t(nm, [&] { zc_write<<<grid, 256, 0, s1>>>((uint4*)h1, n16); });
        snprintf(nm, sizeof nm, "kernel reads host (grid %d x 256)", grid);
        t(nm, [&] { zc_read<<<grid, 256, 0, s1>>>((const uint4*)h1, n16, sink); });
    }
    t("copy engine H2D", [&] { cudaMemcpyAsync(d1, h1, B, cudaMemcpyHostToDevice, s1); });
    t("copy engine D2H", [&] { cudaMemcpyAsync(h2, d2, B, cudaMemcpyDeviceToHost, s1); });
    t("copy engine H2D || D2H (both, time for both)", [&] {
        cudaMemcpyAsync(d1, h1, B, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync(h2, d2, B, cudaMemcpyDeviceToHost, s2);
    });
    t("CE H2D || kernel writes host 592 (both)", [&] {
        cudaMemcpyAsync(d1, h1, B, cudaMemcpyHostToDevice, s1);
        zc_write<<<592, 256, 0, s2>>>((uint4*)h2, n16);
    });
    t("kernel reads host 592 || CE D2H (both)", [&] {
        zc_read<<<592, 256, 0, s1>>>((const uint4*)h1, n16, sink);
        cudaMemcpyAsync(h2, d2, B, cudaMemcpyDeviceToHost, s2);
    });
    t("kernel copies host->dev 592 || CE D2H (both)", [&] {
        zc_copy<<<592, 256, 0, s1>>>((const uint4*)h1, (uint4*)d1, n16);
        cudaMemcpyAsync(h2, d2, B, cudaMemcpyDeviceToHost, s2);
    });
    t("kernel copies dev->host (592)", [&] { zc_copy<<<592, 256, 0, s1>>>((const uint4*)d2, (uint4*)h2, n16); });
    t("kernel copies host->host (592) [read+write]", [&] { zc_copy<<<592, 256, 0, s1>>>((const uint4*)h1, (uint4*)h2, n16); });
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
