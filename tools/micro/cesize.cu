// Copy-engine rate vs copy size and source interleaving (H2D only, D2H only).
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t B = size_t(256) << 20;
    unsigned char *h, *d, *h2;
    cudaHostAlloc(&h, B, 0); cudaHostAlloc(&h2, B, 0); cudaMalloc(&d, B);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    auto t = [&](const char* nm, auto fn) {
        double best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaDeviceSynchronize();
            auto t0 = std::chrono::steady_clock::now();
            fn();
            cudaDeviceSynchronize();
            double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (r) best = ms < best ? ms : best;
        }
        printf("%-60s %7.3f ms %6.1f GB/s\n", nm, best, B / best / 1e6);
    };
    for (size_t piece : {size_t(256) << 20, size_t(32) << 20, size_t(8) << 20, size_t(2) << 20, size_t(512) << 10}) {
        char nm[128];
        snprintf(nm, sizeof nm, "H2D sequential pieces of %zu KiB", piece >> 10);
        t(nm, [&] { for (size_t o = 0; o < B; o += piece) cudaMemcpyAsync(d + o, h + o, piece, cudaMemcpyHostToDevice, s); });
        snprintf(nm, sizeof nm, "H2D 4 interleaved regions, pieces of %zu KiB", piece >> 10);
        t(nm, [&] {
            const size_t R = B / 4;
            for (size_t o = 0; o < R; o += piece / 4 ? piece / 4 : 1)
                for (int q = 0; q < 4; ++q) cudaMemcpyAsync(d + q * R + o, h + q * R + o, piece / 4, cudaMemcpyHostToDevice, s);
        });
        snprintf(nm, sizeof nm, "D2H sequential pieces of %zu KiB", piece >> 10);
        t(nm, [&] { for (size_t o = 0; o < B; o += piece) cudaMemcpyAsync(h2 + o, d + o, piece, cudaMemcpyDeviceToHost, s); });
    }
}
