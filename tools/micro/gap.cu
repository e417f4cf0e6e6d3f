// Where does event time go around one pipeline launch?  marker kernel ->
// merge (traced) -> marker kernel, all on one stream; prints GPU-clock gaps.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>
#include "comerge_cuda.h"
#include "comerge_cuda_testkit.h"
__global__ void marker(unsigned long long* t) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    *t = g;
}
int main(int argc, char** argv) {
    const size_t m = 1 << 24, n = 1 << 24;
    int *a, *b, *o; uint32_t *av, *bv, *ov;
    cudaMalloc(&a, m * 4); cudaMalloc(&b, n * 4); cudaMalloc(&o, (m + n) * 4);
    cudaMalloc(&av, m * 4); cudaMalloc(&bv, n * 4); cudaMalloc(&ov, (m + n) * 4);
    comerge_testkit_generate_sorted(COMERGE_KEY_I32, 1, 0, m, 16, a, 0);
    comerge_testkit_generate_sorted(COMERGE_KEY_I32, 1, 1, n, 16, b, 0);
    size_t wsb = comerge_cuda_merge_workspace_bytes(m, n, COMERGE_KEY_I32, 1);
    void* ws; cudaMalloc(&ws, wsb);
    unsigned long long *tr, *mk; cudaMalloc(&tr, 20 * 4096 * 8); cudaMalloc(&mk, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int r = 0; r < 6; ++r) {
        cudaMemset(tr, 0, 20 * 4096 * 8);
        comerge_cuda_set_trace(tr);
        cudaEventRecord(e0);
        marker<<<1, 1>>>(mk);
        int rc = comerge_cuda_merge_pairs_i32(a, av, m, b, bv, n, o, ov, ws, wsb, 0);
        marker<<<1, 1>>>(mk + 1);
        cudaEventRecord(e1);
        cudaDeviceSynchronize();
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<unsigned long long> h(8 * 4096), hm(2);
        cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(hm.data(), mk, 16, cudaMemcpyDeviceToHost);
        std::vector<unsigned long long> hx(4 * 4096);
        cudaMemcpy(hx.data(), tr + 8 * 4096, hx.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long s0 = ~0ull, e_max = 0, st_max = 0;
        for (int c = 0; c < 4096; ++c) {
            if (!h[8 * c]) continue;
            s0 = std::min(s0, h[8 * c]);
            e_max = std::max(e_max, h[8 * c + 3]);
            st_max = std::max(st_max, hx[4 * c + 3]);
        }
        printf("stores drained %.2f us after the last consumer end; ", (st_max - e_max) / 1e3);
        printf("rc %d events %.1f us | marker0->first CTA %.2f  span %.2f  last end->marker1 %.2f\n", rc,
               ms * 1e3, (s0 - hm[0]) / 1e3, (e_max - s0) / 1e3, (hm[1] - e_max) / 1e3);
    }
    comerge_cuda_set_trace(nullptr);
}
