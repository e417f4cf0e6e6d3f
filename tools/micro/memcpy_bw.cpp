// host copy bandwidth: T threads copying a 1 GiB buffer in 2 MiB pieces, std::memcpy
// against non-temporal AVX2 stores (the host pipeline's staging copies)
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <atomic>
#include <immintrin.h>
__attribute__((target("avx2"))) static void nt_copy(char* d, const char* s, size_t n) {
    size_t i = 0;
    for (; i < n && ((uintptr_t)(d + i) & 31); ++i) d[i] = s[i];
    for (; i + 128 <= n; i += 128) {
        __m256i a = _mm256_loadu_si256((const __m256i*)(s + i));
        __m256i b = _mm256_loadu_si256((const __m256i*)(s + i + 32));
        __m256i c = _mm256_loadu_si256((const __m256i*)(s + i + 64));
        __m256i e = _mm256_loadu_si256((const __m256i*)(s + i + 96));
        _mm256_stream_si256((__m256i*)(d + i), a);
        _mm256_stream_si256((__m256i*)(d + i + 32), b);
        _mm256_stream_si256((__m256i*)(d + i + 64), c);
        _mm256_stream_si256((__m256i*)(d + i + 96), e);
    }
    for (; i < n; ++i) d[i] = s[i];
    _mm_sfence();
}
int main() {
    const size_t N = size_t(1) << 30;
    char* a = (char*)aligned_alloc(4096, N);
    char* b = (char*)aligned_alloc(4096, N);
    memset(a, 1, N); memset(b, 2, N);
    const size_t P = size_t(2) << 20;
    for (int mode = 0; mode < 2; ++mode)
    for (int T : {1, 4, 8, 16}) {
        double best = 1e9;
        for (int r = 0; r < 3; ++r) {
            std::atomic<size_t> next{0};
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t) th.emplace_back([&] {
                for (;;) { size_t o = next.fetch_add(P); if (o >= N) break;
                           size_t len = std::min(P, N - o);
                           if (mode) nt_copy(b + o, a + o, len); else std::memcpy(b + o, a + o, len); } });
            for (auto& x : th) x.join();
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (s < best) best = s;
        }
        std::printf("%s threads %2d: %.1f GB/s copied\n", mode ? "nt    " : "memcpy", T, N / best / 1e9);
    }
}
