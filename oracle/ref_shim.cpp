// ref_shim.cpp -- TEST ORACLE glue: exposes the UNMODIFIED reference
// library (header-only core under /root/reference/proj/include plus
// /root/reference/proj/src/generate.cpp) through a C ABI so Python tests
// and bench.py's reference arm can call it.  Built by oracle/Makefile into
// oracle/_ref/libcomerge_ref.so; no reference source is copied into this
// repository.  Only tests/, smoke() and bench.py's CPU legs load it.
//
// Entry points wrap, one to one:
//   comerge::co_rank                  corank.hpp:128-133
//   comerge::stable_merge             merge.hpp:52-68
//   comerge::merge_parallel(_synced)  parallel.hpp:304-336
//   comerge::plan                     parallel.hpp:94-115
//   comerge::partition_output         parallel.hpp:60-67
//   comerge::oracle_merge_tagged      oracle.hpp:65-93
//   comerge::generate                 generate.cpp:69-97
//   comerge::multiset_checksum        keys.hpp:50-55
// Key-value merges use a {key, uint32 val} struct with a key-only less,
// the reference's own tagged<K>/tagged_key_less pattern (oracle.hpp:22-37).

#include <chrono>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "comerge/corank.hpp"
#include "comerge/generate.hpp"
#include "comerge/keys.hpp"
#include "comerge/merge.hpp"
#include "comerge/oracle.hpp"
#include "comerge/parallel.hpp"

namespace {

thread_local std::string g_error;

enum { K_I32 = 0, K_U32 = 1, K_U64 = 2 };
enum { OK = 0, E_INVALID = 1, E_RANGE = 2, E_LENGTH = 3, E_OTHER = 4 };

struct kv_i32 {
    std::int32_t key;
    std::uint32_t val;
};
struct kv_u32 {
    std::uint32_t key;
    std::uint32_t val;
};
struct kv_u64 {
    std::uint64_t key;
    std::uint32_t val;
};
struct key_less {
    template <typename T>
    bool operator()(const T& x, const T& y) const {
        return x.key < y.key;
    }
};

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return OK;
    } catch (const std::invalid_argument& e) {
        g_error = e.what();
        return E_INVALID;
    } catch (const std::out_of_range& e) {
        g_error = e.what();
        return E_RANGE;
    } catch (const std::length_error& e) {
        g_error = e.what();
        return E_LENGTH;
    } catch (const std::exception& e) {
        g_error = e.what();
        return E_OTHER;
    }
}

template <typename Fn>
int dispatch_key(int kind, Fn&& fn) {
    switch (kind) {
    case K_I32: return fn(std::int32_t{});
    case K_U32: return fn(std::uint32_t{});
    case K_U64: return fn(std::uint64_t{});
    default: g_error = "unknown key kind"; return E_INVALID;
    }
}

struct ref_report {
    std::uint64_t m, n, workers, wall_ns, comparisons;
    std::int32_t has_comparisons;
    std::int32_t pad;
};

template <typename T>
void fill_report(const comerge::merge_report& r, ref_report* rep, std::uint64_t* block_sizes,
                 std::uint32_t* iters) {
    if (rep) {
        rep->m = r.m;
        rep->n = r.n;
        rep->workers = r.workers;
        rep->wall_ns = r.wall_ns;
        rep->has_comparisons = r.comparisons.has_value();
        rep->comparisons = r.comparisons.value_or(0);
    }
    if (block_sizes)
        for (std::size_t i = 0; i < r.block_sizes.size(); ++i) block_sizes[i] = r.block_sizes[i];
    if (iters)
        for (std::size_t i = 0; i < r.corank_iterations.size(); ++i)
            iters[i] = r.corank_iterations[i];
}

template <typename T>
int run_merge_parallel(const void* a, std::size_t m, const void* b, std::size_t n, void* out,
                       std::size_t out_len, std::size_t workers, int simulated, int synced,
                       int count_cmp, ref_report* rep, std::uint64_t* block_sizes,
                       std::uint32_t* iters) {
    return guarded([&] {
        const std::span<const T> av(static_cast<const T*>(a), m);
        const std::span<const T> bv(static_cast<const T*>(b), n);
        std::span<T> ov(static_cast<T*>(out), out_len);
        const comerge::merge_options opts{
            simulated ? comerge::run_mode::simulated : comerge::run_mode::threads,
            count_cmp != 0};
        comerge::merge_report r;
        if constexpr (requires(T t) { t.key; }) {
            r = synced ? comerge::merge_parallel_synced(av, bv, ov, workers, key_less{}, opts)
                       : comerge::merge_parallel(av, bv, ov, workers, key_less{}, opts);
        } else {
            r = synced ? comerge::merge_parallel_synced(av, bv, ov, workers, std::less<>{}, opts)
                       : comerge::merge_parallel(av, bv, ov, workers, std::less<>{}, opts);
        }
        fill_report<T>(r, rep, block_sizes, iters);
    });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

std::size_t ref_report_size() { return sizeof(ref_report); }

std::size_t ref_kv_size(int kind) {
    return kind == K_I32 ? sizeof(kv_i32) : kind == K_U32 ? sizeof(kv_u32) : sizeof(kv_u64);
}

int ref_co_rank(int kind, std::uint64_t target, const void* a, std::size_t m, const void* b,
                std::size_t n, std::uint64_t* j, std::uint64_t* k, std::uint32_t* iterations,
                std::uint32_t* comparisons) {
    return dispatch_key(kind, [&](auto tag) {
        using K = decltype(tag);
        return guarded([&] {
            const std::span<const K> av(static_cast<const K*>(a), m);
            const std::span<const K> bv(static_cast<const K*>(b), n);
            comerge::co_rank_stats stats;
            const comerge::co_ranks r = comerge::co_rank(target, av, bv, std::less<>{}, &stats);
            *j = r.a;
            *k = r.b;
            if (iterations) *iterations = stats.iterations;
            if (comparisons) *comparisons = stats.comparisons;
        });
    });
}

int ref_partition_output(std::size_t total, std::size_t workers, std::size_t r,
                         std::uint64_t* out) {
    return guarded([&] { *out = comerge::partition_output(total, workers, r); });
}

int ref_stable_merge(int kind, const void* a, std::size_t m, const void* b, std::size_t n,
                     void* out, std::size_t out_len) {
    return dispatch_key(kind, [&](auto tag) {
        using K = decltype(tag);
        return guarded([&] {
            const std::span<const K> av(static_cast<const K*>(a), m);
            const std::span<const K> bv(static_cast<const K*>(b), n);
            comerge::stable_merge(av, bv, std::span<K>(static_cast<K*>(out), out_len));
        });
    });
}

// keys-only merge_parallel / merge_parallel_synced
int ref_merge_parallel(int kind, const void* a, std::size_t m, const void* b, std::size_t n,
                       void* out, std::size_t out_len, std::size_t workers, int simulated,
                       int synced, int count_cmp, ref_report* rep, std::uint64_t* block_sizes,
                       std::uint32_t* iters) {
    return dispatch_key(kind, [&](auto tag) {
        using K = decltype(tag);
        return run_merge_parallel<K>(a, m, b, n, out, out_len, workers, simulated, synced,
                                     count_cmp, rep, block_sizes, iters);
    });
}

// key-value merge_parallel over AoS {key, val} structs (see ref_kv_size)
int ref_merge_parallel_kv(int kind, const void* a, std::size_t m, const void* b, std::size_t n,
                          void* out, std::size_t out_len, std::size_t workers, int simulated,
                          int synced, ref_report* rep, std::uint64_t* block_sizes,
                          std::uint32_t* iters) {
    switch (kind) {
    case K_I32:
        return run_merge_parallel<kv_i32>(a, m, b, n, out, out_len, workers, simulated, synced,
                                          0, rep, block_sizes, iters);
    case K_U32:
        return run_merge_parallel<kv_u32>(a, m, b, n, out, out_len, workers, simulated, synced,
                                          0, rep, block_sizes, iters);
    case K_U64:
        return run_merge_parallel<kv_u64>(a, m, b, n, out, out_len, workers, simulated, synced,
                                          0, rep, block_sizes, iters);
    }
    g_error = "unknown key kind";
    return E_INVALID;
}

// plan(): 7 uint64 per block {worker, out_begin, out_end, a_begin, a_end, b_begin, b_end}
int ref_plan(int kind, const void* a, std::size_t m, const void* b, std::size_t n,
             std::size_t workers, std::uint64_t* blocks) {
    return dispatch_key(kind, [&](auto tag) {
        using K = decltype(tag);
        return guarded([&] {
            const std::span<const K> av(static_cast<const K*>(a), m);
            const std::span<const K> bv(static_cast<const K*>(b), n);
            const comerge::merge_plan p = comerge::plan(av, bv, workers);
            for (std::size_t r = 0; r < p.blocks.size(); ++r) {
                const auto& x = p.blocks[r];
                const std::uint64_t v[7] = {x.worker,  x.out_begin, x.out_end, x.a_begin,
                                            x.a_end,   x.b_begin,   x.b_end};
                std::memcpy(blocks + 7 * r, v, sizeof(v));
            }
        });
    });
}

// Segmented batch: the reference has no batched API, so pairs are spread
// round-robin over `threads` std::threads, each calling stable_merge per
// pair.  Returns the wall time of the parallel region.
int ref_merge_segmented(int kind, const void* a, const std::uint64_t* a_off, const void* b,
                        const std::uint64_t* b_off, std::size_t nseg, void* out, int threads,
                        std::uint64_t* wall_ns) {
    return dispatch_key(kind, [&](auto tag) {
        using K = decltype(tag);
        return guarded([&] {
            const K* ap = static_cast<const K*>(a);
            const K* bp = static_cast<const K*>(b);
            K* op = static_cast<K*>(out);
            auto work = [&](std::size_t first, std::size_t step) {
                for (std::size_t p = first; p < nseg; p += step) {
                    const std::size_t ma = a_off[p + 1] - a_off[p];
                    const std::size_t nb = b_off[p + 1] - b_off[p];
                    comerge::stable_merge(std::span<const K>(ap + a_off[p], ma),
                                          std::span<const K>(bp + b_off[p], nb),
                                          std::span<K>(op + a_off[p] + b_off[p], ma + nb));
                }
            };
            const std::size_t t = threads < 1 ? 1 : static_cast<std::size_t>(threads);
            const auto t0 = std::chrono::steady_clock::now();
            if (t == 1) {
                work(0, 1);
            } else {
                std::vector<std::thread> pool;
                for (std::size_t i = 1; i < t; ++i) pool.emplace_back(work, i, t);
                work(0, t);
                for (auto& th : pool) th.join();
            }
            const auto t1 = std::chrono::steady_clock::now();
            if (wall_ns)
                *wall_ns = static_cast<std::uint64_t>(
                    std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
        });
    });
}

// merge_parallel over the reference's OWN tagged<K> with its tagged_key_less
// (oracle.hpp:22-37; parallel.hpp:304-317): 12-byte records for 32-bit keys,
// 16-byte for uint64 (see ref_tagged_size)
std::size_t ref_tagged_size(int kind) {
    return kind == K_U64 ? sizeof(comerge::tagged<std::uint64_t>)
                         : kind == K_U32 ? sizeof(comerge::tagged<std::uint32_t>)
                                         : sizeof(comerge::tagged<std::int32_t>);
}

int ref_merge_parallel_tagged(int kind, const void* a, std::size_t m, const void* b,
                              std::size_t n, void* out, std::size_t out_len, std::size_t workers,
                              int synced, ref_report* rep) {
    return dispatch_key(kind, [&](auto tag) {
        using T = comerge::tagged<decltype(tag)>;
        return guarded([&] {
            const std::span<const T> av(static_cast<const T*>(a), m);
            const std::span<const T> bv(static_cast<const T*>(b), n);
            std::span<T> ov(static_cast<T*>(out), out_len);
            const comerge::merge_report r =
                synced ? comerge::merge_parallel_synced(av, bv, ov, workers, comerge::tagged_key_less{})
                       : comerge::merge_parallel(av, bv, ov, workers, comerge::tagged_key_less{});
            fill_report<T>(r, rep, nullptr, nullptr);
        });
    });
}

// oracle_merge_tagged over uint64 keys: origin 0 = a, 1 = b
int ref_oracle_merge_tagged(const std::uint64_t* a, std::size_t m, const std::uint64_t* b,
                            std::size_t n, std::uint64_t* keys, std::uint8_t* origin,
                            std::uint32_t* index) {
    return guarded([&] {
        const auto r = comerge::oracle_merge_tagged(std::span<const std::uint64_t>(a, m),
                                                    std::span<const std::uint64_t>(b, n));
        for (std::size_t i = 0; i < r.size(); ++i) {
            keys[i] = r[i].key;
            origin[i] = static_cast<std::uint8_t>(r[i].from);
            index[i] = r[i].index;
        }
    });
}

// comerge::generate (uint64 keys) for dist token kinds 0..6 in dist_kind order
int ref_generate(int dist, std::uint64_t seed, std::uint64_t param, std::size_t m, std::size_t n,
                 std::uint64_t* a, std::uint64_t* b) {
    return guarded([&] {
        comerge::distribution d;
        d.kind = static_cast<comerge::dist_kind>(dist);
        d.seed = seed;
        d.param = param;
        const auto [ga, gb] = comerge::generate(d, m, n);
        std::memcpy(a, ga.data(), m * sizeof(std::uint64_t));
        std::memcpy(b, gb.data(), n * sizeof(std::uint64_t));
    });
}

std::uint64_t ref_multiset_checksum(const std::uint64_t* keys, std::size_t len) {
    return comerge::multiset_checksum(std::span<const std::uint64_t>(keys, len));
}

}  // extern "C"
