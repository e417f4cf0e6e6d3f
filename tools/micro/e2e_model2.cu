// Copy model of the host pipeline with the library's exact command pattern
// (C2: four separately pinned 64 MiB input arrays, two 128 MiB output arrays;
// chunk c: A keys, A vals, B keys, B vals in; out windows back), with and
// without a kernel between the directions and with different stream layouts.
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/micro/e2e_model2 tools/micro/e2e_model2.cu
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void spin(unsigned long long ns) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 >= ns) break;
    }
}

int main() {
    const size_t M = size_t(1) << 24, N = M, T = M + N;
    unsigned *ha, *hav, *hb, *hbv, *ho, *hov;
    CK(cudaHostAlloc(&ha, M * 4, 0)); CK(cudaHostAlloc(&hb, N * 4, 0));
    CK(cudaHostAlloc(&hav, M * 4, 0)); CK(cudaHostAlloc(&hbv, N * 4, 0));
    CK(cudaHostAlloc(&ho, T * 4, 0)); CK(cudaHostAlloc(&hov, T * 4, 0));
    for (auto p : {ha, hav, hb, hbv}) memset(p, 1, M * 4);
    memset(ho, 0, T * 4); memset(hov, 0, T * 4);
    unsigned* d;
    CK(cudaMalloc(&d, T * 4 * 4));
    unsigned *da = d, *dav = d + M, *db = d + 2 * M, *dbv = d + 3 * M, *dout = d + T * 2, *doutv = d + T * 3;
    cudaStream_t s1, s2, s3;
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> ev(64), ev2(64);
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (auto& e : ev2) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    auto timed = [&](const char* name, int C, auto body) {
        double best = 1e9, sum = 0;
        for (int r = 0; r < 6; ++r) {
            cudaDeviceSynchronize();
            auto t0 = std::chrono::steady_clock::now();
            body(C);
            cudaDeviceSynchronize();
            double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (r) { best = ms < best ? ms : best; sum += ms; }
        }
        cudaError_t e = cudaGetLastError();
        printf("%-70s chunks %3d  best %6.2f ms  mean %6.2f ms %s\n", name, C, best, sum / 5,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    // granularity of chunk cuts and window starts (elements), non-power-of-two chunk counts
    for (int C : {8, 12}) for (long G : {64L, 1024L, 16384L, 524288L}) {
        char nm[128];
        snprintf(nm, sizeof nm, "G grid %ld elements, 4 matched, skew 0.47, no kernel", G);
        timed(nm, C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                auto cutf = [&](int q) { return q == C ? T : (T * q / C) / G * G; };
                auto jf = [&](int q) { return q == C ? M : size_t(double(cutf(q)) * 0.47) / G * G; };
                size_t i0 = cutf(c), i1 = cutf(c + 1), j0 = jf(c), j1 = jf(c + 1);
                size_t k0 = i0 - j0, k1 = i1 - j1, wa = j1 - j0, wb = k1 - k0;
                size_t sk0 = k0 / G * G, ek1 = std::min(N, (k1 + G - 1) / G * G);
                cudaMemcpyAsync(da + j0, ha + j0, wa * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(dav + j0, hav + j0, wa * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(db + sk0, hb + sk0, (ek1 - sk0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(dbv + sk0, hbv + sk0, (ek1 - sk0) * 4, cudaMemcpyHostToDevice, s1);
                cudaEventRecord(ev[c], s1);
                cudaStreamWaitEvent(s3, ev[c], 0);
                size_t h = std::min(i1 - i0, (wa + G / 2) / G * G);
                cudaMemcpyAsync(ho + i0, dout + i0, h * 4, cudaMemcpyDeviceToHost, s3);
                cudaMemcpyAsync(hov + i0, doutv + i0, h * 4, cudaMemcpyDeviceToHost, s3);
                cudaMemcpyAsync(ho + i0 + h, dout + i0 + h, (i1 - i0 - h) * 4, cudaMemcpyDeviceToHost, s3);
                cudaMemcpyAsync(hov + i0 + h, doutv + i0 + h, (i1 - i0 - h) * 4, cudaMemcpyDeviceToHost, s3);
            }
        });
    }
    return 0;
}
