// Copy-command cost on this box's PCIe: C2's bytes (4 input arrays of 64 MiB,
// 2 output arrays of 128 MiB) through an 8/16-chunk H2D/D2H pipeline issued
// as (1) separate copies per array, (2) 2-row cudaMemcpy2DAsync per array
// pair, (3) one copy per direction from single contiguous buffers (floor).
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void busy(unsigned char* p, size_t n) {  // ~a chunk merge: read+write n bytes
    for (size_t i = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) * 16; i + 16 <= n; i += size_t(gridDim.x) * blockDim.x * 16) {
        uint4 v = *reinterpret_cast<uint4*>(p + i);
        v.x += 1;
        *reinterpret_cast<uint4*>(p + i) = v;
    }
}
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)
int main() {
    const size_t E = size_t(1) << 24, EB = E * 4;  // elements per input array
    unsigned char *h, *d;
    // one pinned slab so the 2D pitch between paired arrays is small and fixed
    CK(cudaHostAlloc(&h, 8 * EB, 0));
    CK(cudaMalloc(&d, 8 * EB));
    unsigned char *ha = h, *hav = h + EB, *hb = h + 2 * EB, *hbv = h + 3 * EB;
    unsigned char *ho = h + 4 * EB, *hov = h + 6 * EB;
    unsigned char *da = d, *dav = d + EB, *db = d + 2 * EB, *dbv = d + 3 * EB;
    unsigned char *dO = d + 4 * EB, *dov = d + 6 * EB;
    cudaStream_t s1, s2, s3; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking);
    cudaEvent_t ev2[64]; for (auto& e : ev2) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEvent_t ev[64]; for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    for (int C : {8, 16}) {
        for (int mode = 0; mode < 5; ++mode) {
            double best = 1e9;
            for (int rep = 0; rep < 6; ++rep) {
                cudaDeviceSynchronize();
                auto t0 = std::chrono::steady_clock::now();
                for (int c = 0; c < C; ++c) {
                    const size_t lo = EB * c / C, hi = EB * (c + 1) / C, w = hi - lo;
                    if (mode == 0) {
                        cudaMemcpyAsync(da + lo, ha + lo, w, cudaMemcpyHostToDevice, s1);
                        cudaMemcpyAsync(db + lo, hb + lo, w, cudaMemcpyHostToDevice, s1);
                        cudaMemcpyAsync(dav + lo, hav + lo, w, cudaMemcpyHostToDevice, s1);
                        cudaMemcpyAsync(dbv + lo, hbv + lo, w, cudaMemcpyHostToDevice, s1);
                    } else if (mode == 1) {
                        cudaMemcpy2DAsync(da + lo, EB, ha + lo, EB, w, 2, cudaMemcpyHostToDevice, s1);
                        cudaMemcpy2DAsync(db + lo, EB, hb + lo, EB, w, 2, cudaMemcpyHostToDevice, s1);
                    } else if (mode == 2 || mode == 3) {
                        cudaMemcpyAsync(da + 4 * lo, ha + 4 * lo, 4 * w, cudaMemcpyHostToDevice, s1);
                    } else {
                        cudaMemcpy2DAsync(da + lo, EB, ha + lo, EB, w, 2, cudaMemcpyHostToDevice, s1);
                        cudaMemcpy2DAsync(db + lo, EB, hb + lo, EB, w, 2, cudaMemcpyHostToDevice, s1);
                    }
                    cudaEventRecord(ev[c], s1);
                    if (mode >= 3) {  // a merge-like kernel between the two copies
                        cudaStreamWaitEvent(s3, ev[c], 0);
                        busy<<<296, 512, 0, s3>>>(dO + 4 * lo, 4 * w);
                        cudaEventRecord(ev2[c], s3);
                        cudaStreamWaitEvent(s2, ev2[c], 0);
                    } else {
                        cudaStreamWaitEvent(s2, ev[c], 0);
                    }
                    const size_t olo = 2 * lo, ow = 2 * w;
                    if (mode == 0) {
                        cudaMemcpyAsync(ho + olo, dO + olo, ow, cudaMemcpyDeviceToHost, s2);
                        cudaMemcpyAsync(hov + olo, dov + olo, ow, cudaMemcpyDeviceToHost, s2);
                    } else if (mode == 1 || mode == 4) {
                        cudaMemcpy2DAsync(ho + olo, 2 * EB, dO + olo, 2 * EB, ow, 2, cudaMemcpyDeviceToHost, s2);
                    } else {
                        cudaMemcpyAsync(ho + 2 * olo, dO + 2 * olo, 2 * ow, cudaMemcpyDeviceToHost, s2);
                    }
                }
                CK(cudaStreamSynchronize(s2));
                CK(cudaStreamSynchronize(s3));
                CK(cudaStreamSynchronize(s1));
                const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                if (rep) best = ms < best ? ms : best;
            }
            printf("chunks %2d mode %d (%s): %.2f ms\n", C, mode,
                   mode == 0 ? "6 copies/chunk" : mode == 1 ? "3 2D copies/chunk" : mode == 2 ? "2 copies/chunk" : mode == 3 ? "2 copies + kernel/chunk" : "3 2D copies + kernel/chunk", best);
        }
    }
    // per-array streams: 4 H2D streams x C copies, 2 D2H streams x C copies, no dependencies
    cudaStream_t hs[4], ds[2];
    for (auto& x : hs) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    for (auto& x : ds) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    for (int C : {1, 8, 16, 32}) {
        for (int variant = 0; variant < 2; ++variant) {
            double best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaDeviceSynchronize();
                auto t0 = std::chrono::steady_clock::now();
                for (int c = 0; c < C; ++c) {
                    const size_t lo = EB * c / C, w = EB * (c + 1) / C - lo;
                    unsigned char* hin[4] = {ha, hav, hb, hbv};
                    unsigned char* din[4] = {da, dav, db, dbv};
                    for (int q = 0; q < 4; ++q)
                        cudaMemcpyAsync(din[q] + lo, hin[q] + lo, w, cudaMemcpyHostToDevice, variant ? hs[q] : hs[0]);
                    cudaMemcpyAsync(ho + 2 * lo, dO + 2 * lo, 2 * w, cudaMemcpyDeviceToHost, ds[0]);
                    cudaMemcpyAsync(hov + 2 * lo, dov + 2 * lo, 2 * w, cudaMemcpyDeviceToHost, variant ? ds[1] : ds[0]);
                }
                cudaDeviceSynchronize();
                const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                if (rep) best = ms < best ? ms : best;
            }
            printf("independent copies, %2d chunks per array, %s: %.2f ms\n", C,
                   variant ? "one stream per array (4 H2D + 2 D2H)" : "1 H2D + 1 D2H stream", best);
        }
    }
    return 0;
}
