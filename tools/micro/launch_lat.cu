// Launch-latency microbenchmark: event-timed empty persistent kernels with and
// without a large dynamic shared-memory carveout, after a small-smem kernel.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void small_kernel(float* p, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] += 1.f;
}
__global__ void empty_kernel(unsigned long long* t) {
    extern __shared__ char s[];
    if (threadIdx.x == 0 && t) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        if (blockIdx.x == 0) t[0] = g;
        if (g == 0) s[0] = 1;
    }
}
int main() {
    float* p; cudaMalloc(&p, 64 << 20);
    unsigned long long* t; cudaMalloc(&t, 64);
    cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    int sizes[4] = {0, 48 * 1024, 120 * 1024, 220 * 1024};
    for (int pre = 0; pre < 2; ++pre)
        for (int si = 0; si < 4; ++si) {
            float best = 1e9, sum = 0;
            for (int r = 0; r < 20; ++r) {
                if (pre) small_kernel<<<16384, 1024>>>(p, 16 << 20);
                cudaEventRecord(a);
                empty_kernel<<<296, 352, sizes[si]>>>(t);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (r >= 3) { best = ms < best ? ms : best; sum += ms; }
            }
            printf("pre_small=%d smem=%6d  event us: min %.2f mean %.2f\n", pre, sizes[si], best * 1e3,
                   sum / 17 * 1e3);
        }
    // two back-to-back big-smem kernels: second one's cost
    for (int r = 0; r < 5; ++r) {
        small_kernel<<<16384, 1024>>>(p, 16 << 20);
        empty_kernel<<<296, 352, 220 * 1024>>>(t);
        cudaEventRecord(a);
        empty_kernel<<<296, 352, 220 * 1024>>>(t);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("after big-smem predecessor: %.2f us\n", ms * 1e3);
    }
    // grid size and graph variants
    int grids[3] = {1, 148, 296};
    for (int gi = 0; gi < 3; ++gi) {
        float best = 1e9;
        for (int r = 0; r < 20; ++r) {
            cudaEventRecord(a);
            empty_kernel<<<grids[gi], 32, 0>>>(nullptr);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) best = ms < best ? ms : best;
        }
        printf("grid %d: min %.2f us\n", grids[gi], best * 1e3);
    }
    {
        cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        empty_kernel<<<296, 352, 220 * 1024, s>>>(t);
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        float best = 1e9;
        for (int r = 0; r < 20; ++r) {
            cudaEventRecord(a, s);
            cudaGraphLaunch(ge, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) best = ms < best ? ms : best;
        }
        printf("graph launch: min %.2f us\n", best * 1e3);
        // two events back to back
        best = 1e9;
        for (int r = 0; r < 20; ++r) {
            cudaEventRecord(a, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) best = ms < best ? ms : best;
        }
        printf("empty event pair: min %.2f us\n", best * 1e3);
        // 10 kernels back to back
        cudaEventRecord(a, s);
        for (int r = 0; r < 10; ++r) empty_kernel<<<296, 352, 220 * 1024, s>>>(t);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("10 kernels: %.2f us\n", ms * 1e3);
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
