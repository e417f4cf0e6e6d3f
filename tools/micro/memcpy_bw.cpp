// host memcpy bandwidth: T threads copying a 1 GiB buffer in 4 MiB pieces
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
#include <atomic>
int main() {
    const size_t N = size_t(1) << 30;
    char* a = (char*)aligned_alloc(4096, N);
    char* b = (char*)aligned_alloc(4096, N);
    memset(a, 1, N); memset(b, 2, N);
    for (int T : {1, 2, 4, 8, 12, 16}) {
        double best = 1e9;
        for (int r = 0; r < 3; ++r) {
            std::atomic<size_t> next{0};
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t) th.emplace_back([&] {
                for (;;) { size_t o = next.fetch_add(size_t(4) << 20); if (o >= N) break;
                           std::memcpy(b + o, a + o, std::min(size_t(4) << 20, N - o)); } });
            for (auto& x : th) x.join();
            double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (s < best) best = s;
        }
        std::printf("threads %2d: %.1f GB/s copied\n", T, N / best / 1e9);
    }
}
