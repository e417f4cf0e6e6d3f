// Copy-only model of the host pipeline for C2's shape (2^24 + 2^24 int32 keys
// with uint32 payloads in four pinned host arrays; 2^25 keys + payloads out in
// two): chunk c moves A[j0,j1), B[k0,k1) (keys + payloads) in and out[i0,i1)
// back, H2D and D2H on separate streams, D2H of chunk c after its H2D.
// Variants differ only in how the copies are expressed.
//   nvcc -O2 -arch=sm_100a -o tools/micro/e2e_model tools/micro/e2e_model.cu
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void copy2(const uint4* s0, uint4* d0, const uint4* s1, uint4* d1, size_t n16) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x) {
        d0[i] = s0[i];
        d1[i] = s1[i];
    }
}

int main() {
    const size_t M = size_t(1) << 24, N = M, T = M + N;
    unsigned *ha, *hav, *hb, *hbv, *ho, *hov, *h1in, *h1out;
    unsigned* hslab;  // host arrays from one pinned slab: two-row pitches are valid
    CK(cudaHostAlloc(&hslab, (2 * M + 2 * N + 2 * T) * 4, cudaHostAllocMapped));
    ha = hslab; hav = ha + M; hb = hav + M; hbv = hb + N; ho = hbv + N; hov = ho + T;
    CK(cudaHostAlloc(&h1in, T * 8, 0)); CK(cudaHostAlloc(&h1out, T * 8, 0));
    for (auto p : {ha, hav, hb, hbv}) memset(p, 1, M * 4);
    memset(h1in, 1, T * 8);
    unsigned *da, *dav, *db, *dbv, *dout, *doutv, *dslab;
    CK(cudaMalloc(&dslab, (2 * M + 2 * N + 2 * T) * 4));
    da = dslab; dav = da + M; db = dav + M; dbv = db + N; dout = dbv + N; doutv = dout + T;
    unsigned *mo, *mov;  // device aliases of the mapped host output
    CK(cudaHostGetDevicePointer((void**)&mo, ho, 0));
    CK(cudaHostGetDevicePointer((void**)&mov, hov, 0));
    // two-row device layouts (rows P apart) for the 2D variants
    unsigned char* slab;
    CK(cudaMalloc(&slab, T * 8 * 2));
    cudaStream_t s1, s2, s3, p1, p2;
    int plo = 0, phi = 0;
    cudaDeviceGetStreamPriorityRange(&plo, &phi);
    CK(cudaStreamCreateWithPriority(&p1, cudaStreamNonBlocking, plo));
    CK(cudaStreamCreateWithPriority(&p2, cudaStreamNonBlocking, phi));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
    std::vector<cudaEvent_t> ev(256), ev2(256);
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
        printf("%-58s chunks %3d  best %6.2f ms  mean %6.2f ms %s\n", name, C, best, sum / 5,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
    };
    auto cut = [&](int C, int c, size_t& i0, size_t& i1, size_t& j0, size_t& j1) {
        i0 = T * c / C; i1 = T * (c + 1) / C; j0 = i0 / 2; j1 = i1 / 2;
    };
    for (int C : {8}) {
        timed("V0 one 1D copy per chunk per direction (8 B/elem slab)", C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                size_t i0 = T * 8 * c / C, i1 = T * 8 * (c + 1) / C;
                cudaMemcpyAsync(slab + i0, (char*)h1in + i0, i1 - i0, cudaMemcpyHostToDevice, s1);
                cudaEventRecord(ev[c], s1);
                cudaStreamWaitEvent(s2, ev[c], 0);
                cudaMemcpyAsync((char*)h1out + i0, slab + T * 8 + i0, i1 - i0, cudaMemcpyDeviceToHost, s2);
            }
        });
        timed("V1 2 two-row 2D H2D + 1 two-row 2D D2H per chunk", C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                size_t i0, i1, j0, j1; cut(C, c, i0, i1, j0, j1);
                size_t k0 = i0 - j0, k1 = i1 - j1;
                cudaMemcpy2DAsync(da + j0, (char*)dav - (char*)da, ha + j0, (char*)hav - (char*)ha,
                                  (j1 - j0) * 4, 2, cudaMemcpyHostToDevice, s1);
                cudaMemcpy2DAsync(db + k0, (char*)dbv - (char*)db, hb + k0, (char*)hbv - (char*)hb,
                                  (k1 - k0) * 4, 2, cudaMemcpyHostToDevice, s1);
                cudaEventRecord(ev[c], s1);
                cudaStreamWaitEvent(s2, ev[c], 0);
                cudaMemcpy2DAsync(ho + i0, (char*)hov - (char*)ho, dout + i0, (char*)doutv - (char*)dout,
                                  (i1 - i0) * 4, 2, cudaMemcpyDeviceToHost, s2);
            }
        });
        timed("V2 4 1D H2D + 2 1D D2H per chunk", C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                size_t i0, i1, j0, j1; cut(C, c, i0, i1, j0, j1);
                size_t k0 = i0 - j0, k1 = i1 - j1;
                cudaMemcpyAsync(da + j0, ha + j0, (j1 - j0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(dav + j0, hav + j0, (j1 - j0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(db + k0, hb + k0, (k1 - k0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(dbv + k0, hbv + k0, (k1 - k0) * 4, cudaMemcpyHostToDevice, s1);
                cudaEventRecord(ev[c], s1);
                cudaStreamWaitEvent(s2, ev[c], 0);
                cudaMemcpyAsync(ho + i0, dout + i0, (i1 - i0) * 4, cudaMemcpyDeviceToHost, s2);
                cudaMemcpyAsync(hov + i0, doutv + i0, (i1 - i0) * 4, cudaMemcpyDeviceToHost, s2);
            }
        });
        timed("V3 V2 with A side / B side on two H2D streams", C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                size_t i0, i1, j0, j1; cut(C, c, i0, i1, j0, j1);
                size_t k0 = i0 - j0, k1 = i1 - j1;
                cudaMemcpyAsync(da + j0, ha + j0, (j1 - j0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(dav + j0, hav + j0, (j1 - j0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(db + k0, hb + k0, (k1 - k0) * 4, cudaMemcpyHostToDevice, s3);
                cudaMemcpyAsync(dbv + k0, hbv + k0, (k1 - k0) * 4, cudaMemcpyHostToDevice, s3);
                cudaEventRecord(ev[c], s1);
                cudaEventRecord(ev2[c], s3);
                cudaStreamWaitEvent(s2, ev[c], 0);
                cudaStreamWaitEvent(s2, ev2[c], 0);
                cudaMemcpyAsync(ho + i0, dout + i0, (i1 - i0) * 4, cudaMemcpyDeviceToHost, s2);
                cudaMemcpyAsync(hov + i0, doutv + i0, (i1 - i0) * 4, cudaMemcpyDeviceToHost, s2);
            }
        });
        timed("V5 H2D only, V2 command shape", C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                size_t i0, i1, j0, j1; cut(C, c, i0, i1, j0, j1);
                size_t k0 = i0 - j0, k1 = i1 - j1;
                cudaMemcpyAsync(da + j0, ha + j0, (j1 - j0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(dav + j0, hav + j0, (j1 - j0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(db + k0, hb + k0, (k1 - k0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(dbv + k0, hbv + k0, (k1 - k0) * 4, cudaMemcpyHostToDevice, s1);
            }
        });
        timed("V6 D2H only, V2 command shape", C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                size_t i0, i1, j0, j1; cut(C, c, i0, i1, j0, j1);
                cudaMemcpyAsync(ho + i0, dout + i0, (i1 - i0) * 4, cudaMemcpyDeviceToHost, s2);
                cudaMemcpyAsync(hov + i0, doutv + i0, (i1 - i0) * 4, cudaMemcpyDeviceToHost, s2);
            }
        });
        timed("V7 V2 with the D2H stream issuing both output rows on 2 streams", C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                size_t i0, i1, j0, j1; cut(C, c, i0, i1, j0, j1);
                size_t k0 = i0 - j0, k1 = i1 - j1;
                cudaMemcpyAsync(da + j0, ha + j0, (j1 - j0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(dav + j0, hav + j0, (j1 - j0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(db + k0, hb + k0, (k1 - k0) * 4, cudaMemcpyHostToDevice, s1);
                cudaMemcpyAsync(dbv + k0, hbv + k0, (k1 - k0) * 4, cudaMemcpyHostToDevice, s1);
                cudaEventRecord(ev[c], s1);
                cudaStreamWaitEvent(s2, ev[c], 0);
                cudaStreamWaitEvent(s3, ev[c], 0);
                cudaMemcpyAsync(ho + i0, dout + i0, (i1 - i0) * 4, cudaMemcpyDeviceToHost, s2);
                cudaMemcpyAsync(hov + i0, doutv + i0, (i1 - i0) * 4, cudaMemcpyDeviceToHost, s3);
            }
        });
        timed("W5 V1 with the D2H stream at high priority", C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                size_t i0, i1, j0, j1; cut(C, c, i0, i1, j0, j1);
                size_t k0 = i0 - j0, k1 = i1 - j1;
                cudaMemcpy2DAsync(da + j0, (char*)dav - (char*)da, ha + j0, (char*)hav - (char*)ha,
                                  (j1 - j0) * 4, 2, cudaMemcpyHostToDevice, p1);
                cudaMemcpy2DAsync(db + k0, (char*)dbv - (char*)db, hb + k0, (char*)hbv - (char*)hb,
                                  (k1 - k0) * 4, 2, cudaMemcpyHostToDevice, p1);
                cudaEventRecord(ev[c], p1);
                cudaStreamWaitEvent(p2, ev[c], 0);
                cudaMemcpy2DAsync(ho + i0, (char*)hov - (char*)ho, dout + i0, (char*)doutv - (char*)dout,
                                  (i1 - i0) * 4, 2, cudaMemcpyDeviceToHost, p2);
            }
        });
        for (int grid : {32, 64, 148}) {
            char nm[96];
            snprintf(nm, sizeof nm, "W4 2 two-row 2D H2D + D2H by a copy kernel (grid %d)", grid);
            timed(nm, C, [&](int C) {
                for (int c = 0; c < C; ++c) {
                    size_t i0, i1, j0, j1; cut(C, c, i0, i1, j0, j1);
                    size_t k0 = i0 - j0, k1 = i1 - j1;
                    cudaMemcpy2DAsync(da + j0, (char*)dav - (char*)da, ha + j0, (char*)hav - (char*)ha,
                                      (j1 - j0) * 4, 2, cudaMemcpyHostToDevice, s1);
                    cudaMemcpy2DAsync(db + k0, (char*)dbv - (char*)db, hb + k0, (char*)hbv - (char*)hb,
                                      (k1 - k0) * 4, 2, cudaMemcpyHostToDevice, s1);
                    cudaEventRecord(ev[c], s1);
                    cudaStreamWaitEvent(s2, ev[c], 0);
                    copy2<<<grid, 512, 0, s2>>>((const uint4*)(dout + i0), (uint4*)(mo + i0),
                                               (const uint4*)(doutv + i0), (uint4*)(mov + i0), (i1 - i0) / 4);
                }
            });
        }
    }
    // which direction's command count costs under bidirectional load
    for (int C : {8, 16}) for (int hin : {1, 2, 4}) for (int hout : {1, 2, 4}) {
        char nm[96];
        snprintf(nm, sizeof nm, "Y contiguous slab, %d H2D + %d D2H commands per chunk", hin, hout);
        timed(nm, C, [&](int C) {
            for (int c = 0; c < C; ++c) {
                size_t i0 = T * 8 * c / C, i1 = T * 8 * (c + 1) / C, w = (i1 - i0);
                for (int q = 0; q < hin; ++q)
                    cudaMemcpyAsync(slab + i0 + w * q / hin, (char*)h1in + i0 + w * q / hin,
                                    w * (q + 1) / hin - w * q / hin, cudaMemcpyHostToDevice, s1);
                cudaEventRecord(ev[c], s1);
                cudaStreamWaitEvent(s2, ev[c], 0);
                for (int q = 0; q < hout; ++q)
                    cudaMemcpyAsync((char*)h1out + i0 + w * q / hout, slab + T * 8 + i0 + w * q / hout,
                                    w * (q + 1) / hout - w * q / hout, cudaMemcpyDeviceToHost, s2);
            }
        });
    }
    return 0;
}
