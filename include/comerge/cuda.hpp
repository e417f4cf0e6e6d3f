// comerge/cuda.hpp -- C++ drop-in for the reference's co-rank / merge API on
// the B200 (sm_100a) kernels of libcomerge_cuda.so.
//
// Mirrors /root/reference/proj/include/comerge/{corank,merge,parallel}.hpp:
//
//   comerge::cuda::co_rank            <- comerge::co_rank            corank.hpp:128-133
//   comerge::cuda::co_rank_counted    <- comerge::co_rank_counted    corank.hpp:138-147
//   comerge::cuda::stable_merge       <- comerge::stable_merge       merge.hpp:52-68
//   comerge::cuda::partition_output   <- comerge::partition_output   parallel.hpp:60-67
//   comerge::cuda::plan               <- comerge::plan               parallel.hpp:94-115
//   comerge::cuda::merge_parallel     <- comerge::merge_parallel     parallel.hpp:304-317
//   comerge::cuda::merge_parallel_synced <- merge_parallel_synced   parallel.hpp:323-336
//   comerge::cuda::merge_report       <- comerge::merge_report       parallel.hpp:44-55
//
// Same argument meaning and the same exception types / message substrings
// (std::invalid_argument, std::out_of_range, std::length_error).  Element
// types: int32_t, uint32_t, uint64_t with std::less<> -- any other comparator
// or type is a compile-time error: there is no CPU fallback.  Ranges may live
// in host memory (copied through the device inside the call) or be device
// spans (comerge::cuda::device_span).  Key-value merges take the reference's
// own shape -- ranges of a {key, payload} struct with a key-only comparator
// (merge_parallel(a, b, out, workers, key_less{}); the pattern of tagged<K> /
// tagged_key_less, oracle.hpp:22-37): any trivially copyable standard-layout
// struct whose first member `key` is int32_t / uint32_t (8- or 12-byte struct:
// the reference's own tagged<int32_t> is 12 bytes) or uint64_t (16-byte
// struct), the rest of the struct moving with its key byte for byte.  A caller's own key-only comparator is accepted once declared
// key-only by specialising comerge::cuda::is_key_less.  The SoA overload
// merge_parallel_pairs (payload uint32_t arrays) is the other form.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <new>
#include <optional>
#include <ranges>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../comerge_cuda.h"

namespace comerge::cuda {

using rank_t = std::size_t;

struct co_ranks {
    std::size_t a = 0;
    std::size_t b = 0;
    friend bool operator==(const co_ranks&, const co_ranks&) = default;
};

struct co_rank_stats {
    std::uint32_t iterations = 0;
    std::uint32_t comparisons = 0;
};

struct comparison_counter {
    std::uint64_t count = 0;
};

enum class run_mode { threads, simulated };

// `mode` is accepted for API compatibility (the device schedule does not
// depend on it); count_comparisons fills merge_report::comparisons with the
// reference's total (co-ranks + every block's merge_into), computed exactly.
struct merge_options {
    run_mode mode = run_mode::threads;
    bool count_comparisons = false;
};

struct merge_report {
    std::size_t m = 0;
    std::size_t n = 0;
    std::size_t workers = 0;
    std::uint64_t wall_ns = 0;  // device merge time
    std::vector<std::size_t> block_sizes;
    std::vector<std::uint32_t> corank_iterations;
    std::optional<std::uint64_t> comparisons;
    std::optional<bool> verified;
    std::optional<double> speedup_vs_p1;
    std::string note;
    // B200 extras
    std::uint64_t e2e_ns = 0;
    std::uint64_t h2d_bytes = 0;
    std::uint64_t d2h_bytes = 0;
    std::uint64_t tiles = 0;
};

struct block_assignment {
    std::size_t worker = 0;
    std::size_t out_begin = 0;
    std::size_t out_end = 0;
    std::size_t a_begin = 0;
    std::size_t a_end = 0;
    std::size_t b_begin = 0;
    std::size_t b_end = 0;
    std::size_t out_size() const { return out_end - out_begin; }
    std::size_t a_size() const { return a_end - a_begin; }
    std::size_t b_size() const { return b_end - b_begin; }
    friend bool operator==(const block_assignment&, const block_assignment&) = default;
};

struct merge_plan {
    std::size_t workers = 0;
    std::vector<block_assignment> blocks;
};

// A contiguous range in device memory (the entry points detect host vs device
// pointers themselves; this type just carries a pointer and a length).
template <typename T>
struct device_span {
    T* ptr = nullptr;
    std::size_t len = 0;
    T* data() const { return ptr; }
    std::size_t size() const { return len; }
    T* begin() const { return ptr; }
    T* end() const { return ptr + len; }
};

namespace detail {

[[noreturn]] inline void throw_status(int rc) {
    const std::string msg = comerge_cuda_last_error();
    switch (rc) {
    case COMERGE_E_INVALID: throw std::invalid_argument(msg);
    case COMERGE_E_RANGE: throw std::out_of_range(msg);
    case COMERGE_E_LENGTH: throw std::length_error(msg);
    default: throw std::runtime_error(msg);
    }
}

inline void check(int rc) {
    if (rc != COMERGE_OK) throw_status(rc);
}

template <typename T>
concept key_type = std::same_as<T, std::int32_t> || std::same_as<T, std::uint32_t> ||
                   std::same_as<T, std::uint64_t>;

template <typename R>
concept key_range = std::ranges::contiguous_range<R> && std::ranges::sized_range<R> &&
                    key_type<std::remove_cv_t<std::ranges::range_value_t<R>>>;

template <typename R>
using key_of = std::remove_cv_t<std::ranges::range_value_t<R>>;

// key-value records (see the header comment)
template <typename T>
concept record_type =
    std::is_trivially_copyable_v<T> && std::is_standard_layout_v<T> &&
    requires(T t) { t.key; } && key_type<std::remove_cv_t<decltype(T::key)>> &&
    (offsetof(T, key) == 0) &&
    ((sizeof(T) == 8 && sizeof(T::key) == 4) || (sizeof(T) == 12 && sizeof(T::key) == 4) ||
     (sizeof(T) == 16 && sizeof(T::key) == 8));

template <typename R>
concept record_range = std::ranges::contiguous_range<R> && std::ranges::sized_range<R> &&
                       record_type<std::remove_cv_t<std::ranges::range_value_t<R>>>;

template <typename R>
using elem_of = std::remove_cv_t<std::ranges::range_value_t<R>>;

template <typename K>
struct abi;

#define COMERGE_CUDA_ABI(K, SUF)                                                                \
    template <>                                                                                 \
    struct abi<K> {                                                                             \
        static int merge_parallel(const K* a, std::size_t m, const K* b, std::size_t n, K* out, \
                                  std::size_t out_len, std::size_t workers, int synced,         \
                                  comerge_merge_report* rep, std::uint64_t* bs,                 \
                                  std::uint32_t* its) {                                         \
            return comerge_merge_parallel_##SUF(a, m, b, n, out, out_len, workers, synced, rep, \
                                                bs, its);                                       \
        }                                                                                       \
        static int merge_ex(const K* a, const std::uint32_t* av, std::size_t m, const K* b,    \
                            const std::uint32_t* bv, std::size_t n, K* out, std::uint32_t* ov, \
                            std::size_t out_len, std::size_t workers,                          \
                            const comerge_merge_options* o, comerge_merge_report* rep,         \
                            std::uint64_t* bs, std::uint32_t* its, std::uint64_t* cmp) {       \
            return comerge_merge_parallel_ex_##SUF(a, av, m, b, bv, n, out, ov, out_len,        \
                                                   workers, o, rep, bs, its, cmp);              \
        }                                                                                       \
        static int merge_pairs(const K* ak, const std::uint32_t* av, std::size_t m,            \
                               const K* bk, const std::uint32_t* bv, std::size_t n, K* ok,      \
                               std::uint32_t* ov, std::size_t out_len, std::size_t workers,     \
                               comerge_merge_report* rep) {                                     \
            return comerge_merge_parallel_pairs_##SUF(ak, av, m, bk, bv, n, ok, ov, out_len,    \
                                                      workers, rep);                            \
        }                                                                                       \
        static int plan(const K* a, std::size_t m, const K* b, std::size_t n, std::size_t w,    \
                        std::uint64_t* blocks) {                                                \
            return comerge_plan_##SUF(a, m, b, n, w, blocks);                                   \
        }                                                                                       \
        static int co_rank(std::uint64_t t, const K* a, std::size_t m, const K* b,             \
                           std::size_t n, std::uint64_t* j, std::uint64_t* k,                   \
                           std::uint32_t* it, std::uint32_t* cmp) {                             \
            return comerge_co_rank_##SUF(t, a, m, b, n, j, k, it, cmp);                          \
        }                                                                                       \
    };
COMERGE_CUDA_ABI(std::int32_t, i32)
COMERGE_CUDA_ABI(std::uint32_t, u32)
COMERGE_CUDA_ABI(std::uint64_t, u64)
#undef COMERGE_CUDA_ABI

inline merge_report to_report(const comerge_merge_report& r) {
    merge_report out;
    out.m = r.m;
    out.n = r.n;
    out.workers = r.workers;
    out.wall_ns = r.wall_ns;
    out.e2e_ns = r.e2e_ns;
    out.h2d_bytes = r.h2d_bytes;
    out.d2h_bytes = r.d2h_bytes;
    out.tiles = r.tiles;
    return out;
}

template <typename A, typename B, typename Out>
merge_report run_merge_parallel(const A& a, const B& b, Out& out, std::size_t workers,
                                merge_options opts, bool synced) {
    using K = key_of<A>;
    comerge_merge_report rep{};
    const comerge_merge_options o{synced ? 1 : 0, opts.count_comparisons ? 1 : 0};
    std::vector<std::uint64_t> bs(workers ? workers : 1);
    std::vector<std::uint32_t> its(2 * (workers ? workers : 1));
    std::uint64_t cmp = 0;
    check(abi<K>::merge_ex(std::ranges::data(a), nullptr, std::ranges::size(a),
                           std::ranges::data(b), nullptr, std::ranges::size(b),
                           std::ranges::data(out), nullptr, std::ranges::size(out), workers, &o,
                           &rep, bs.data(), its.data(), &cmp));
    merge_report r = to_report(rep);
    r.block_sizes.assign(bs.begin(), bs.begin() + workers);
    r.corank_iterations.assign(its.begin(), its.begin() + (synced ? workers : 2 * workers));
    if (opts.count_comparisons) r.comparisons = cmp;
    return r;
}

}  // namespace detail

/// Unique split (j, k), j + k = target, of the stable merge of a and b
/// (Algorithm 1, corank.hpp:72-121, run on the device).  Throws
/// std::out_of_range ("rank out of range") if target > m + n.
template <detail::key_range A, detail::key_range B>
    requires std::same_as<detail::key_of<A>, detail::key_of<B>>
co_ranks co_rank(rank_t target, const A& a, const B& b, std::less<> = {},
                 co_rank_stats* stats = nullptr) {
    using K = detail::key_of<A>;
    std::uint64_t j = 0, k = 0;
    std::uint32_t it = 0, cmp = 0;
    detail::check(detail::abi<K>::co_rank(target, std::ranges::data(a), std::ranges::size(a),
                                          std::ranges::data(b), std::ranges::size(b), &j, &k, &it,
                                          &cmp));
    if (stats) *stats = {it, cmp};
    return {static_cast<std::size_t>(j), static_cast<std::size_t>(k)};
}

template <detail::key_range A, detail::key_range B>
    requires std::same_as<detail::key_of<A>, detail::key_of<B>>
co_ranks co_rank_counted(rank_t target, const A& a, const B& b, std::less<> less,
                         comparison_counter& counter) {
    co_rank_stats st;
    const co_ranks r = co_rank(target, a, b, less, &st);
    counter.count += st.comparisons;
    return r;
}

/// floor(r * total / workers) without intermediate overflow.
inline rank_t partition_output(std::size_t total, std::size_t workers, std::size_t r) {
    std::uint64_t out = 0;
    detail::check(comerge_partition_output(total, workers, r, &out));
    return static_cast<rank_t>(out);
}

/// Stable merge of a and b into out (ties A-first); out must have length
/// |a| + |b| and must not alias an input (std::invalid_argument).
template <detail::key_range A, detail::key_range B, std::ranges::contiguous_range Out>
    requires std::same_as<detail::key_of<A>, detail::key_of<B>> &&
             std::same_as<detail::key_of<A>, std::ranges::range_value_t<Out>>
void stable_merge(const A& a, const B& b, Out&& out, std::less<> = {}) {
    if (std::ranges::size(out) != std::ranges::size(a) + std::ranges::size(b))
        throw std::invalid_argument("stable_merge: output length must equal |a| + |b|");
    try {
        detail::run_merge_parallel(a, b, out, 1, merge_options{}, false);
    } catch (const std::invalid_argument& e) {
        std::string msg = e.what();
        const auto pos = msg.find("merge_parallel");
        if (pos != std::string::npos) msg.replace(pos, 14, "stable_merge");
        throw std::invalid_argument(msg);
    }
}

/// Merge with the reference's `workers`-way report (block sizes, co-rank
/// iterations of every block boundary); the device merges in its own tiles,
/// so the output does not depend on `workers`.
template <detail::key_range A, detail::key_range B, std::ranges::contiguous_range Out>
    requires std::same_as<detail::key_of<A>, detail::key_of<B>> &&
             std::same_as<detail::key_of<A>, std::ranges::range_value_t<Out>>
merge_report merge_parallel(const A& a, const B& b, Out&& out, std::size_t workers,
                            std::less<> = {}, merge_options opts = {}) {
    return detail::run_merge_parallel(a, b, out, workers, opts, false);
}

template <detail::key_range A, detail::key_range B, std::ranges::contiguous_range Out>
    requires std::same_as<detail::key_of<A>, detail::key_of<B>> &&
             std::same_as<detail::key_of<A>, std::ranges::range_value_t<Out>>
merge_report merge_parallel_synced(const A& a, const B& b, Out&& out, std::size_t workers,
                                   std::less<> = {}, merge_options opts = {}) {
    return detail::run_merge_parallel(a, b, out, workers, opts, true);
}

/// std::allocator replacement handing out page-locked host memory
/// (comerge_cuda_host_alloc): host-buffer merges of vectors allocated with it
/// copy at PCIe rate (pageable storage goes through the library's staging
/// pool, ~1.9x slower on C4).  std::vector<T, comerge::cuda::pinned_allocator<T>> is a contiguous
/// range every overload here accepts.
template <typename T>
struct pinned_allocator {
    using value_type = T;
    pinned_allocator() noexcept = default;
    template <typename U>
    pinned_allocator(const pinned_allocator<U>&) noexcept {}
    T* allocate(std::size_t n) {
        if (n > std::size_t(-1) / sizeof(T)) throw std::bad_array_new_length();
        void* p = nullptr;
        if (comerge_cuda_host_alloc(n * sizeof(T), &p) != COMERGE_OK || (n && !p))
            throw std::bad_alloc();
        return static_cast<T*>(p);
    }
    void deallocate(T* p, std::size_t) noexcept { comerge_cuda_host_free(p); }
    template <typename U>
    friend bool operator==(const pinned_allocator&, const pinned_allocator<U>&) noexcept {
        return true;
    }
};

/// A key-value record (the shape of the reference's tagged<K>, oracle.hpp:22-37).
template <typename K>
struct record {
    K key{};
    std::uint32_t val = 0;
    friend bool operator==(const record&, const record&) = default;
};

/// Key-only ordering of records (the reference's tagged_key_less).
struct key_less {
    template <typename T>
    bool operator()(const T& x, const T& y) const {
        return x.key < y.key;
    }
};

/// Comparators the device may run as "compare the keys only": key_less, plus
/// any caller comparator declared key-only by specialising this trait, e.g.
///   template <> struct comerge::cuda::is_key_less<comerge::tagged_key_less>
///       : std::true_type {};
template <typename C>
struct is_key_less : std::false_type {};
template <>
struct is_key_less<key_less> : std::true_type {};

namespace detail {
// generic record entry points by key type (record size passed at run time)
template <typename K>
struct rec_generic;
#define COMERGE_CUDA_REC_GENERIC(K, SUF)                                                        \
    template <>                                                                                 \
    struct rec_generic<K> {                                                                     \
        static int merge_ex(const void* a, std::size_t m, const void* b, std::size_t n,        \
                            void* out, std::size_t len, std::size_t rb, std::size_t w,          \
                            const comerge_merge_options* o, comerge_merge_report* rep,         \
                            std::uint64_t* bs, std::uint32_t* its, std::uint64_t* cmp) {        \
            return comerge_merge_parallel_records_ex_##SUF(a, m, b, n, out, len, rb, w, o, rep, \
                                                           bs, its, cmp);                       \
        }                                                                                       \
        static int co_rank(std::uint64_t t, const void* a, std::size_t m, const void* b,       \
                           std::size_t n, std::size_t rb, std::uint64_t* j, std::uint64_t* k,   \
                           std::uint32_t* it, std::uint32_t* cmp) {                             \
            return comerge_co_rank_records_##SUF(t, a, m, b, n, rb, j, k, it, cmp);             \
        }                                                                                       \
        static int plan(const void* a, std::size_t m, const void* b, std::size_t n,            \
                        std::size_t rb, std::size_t w, std::uint64_t* blocks) {                 \
            return comerge_plan_records_##SUF(a, m, b, n, rb, w, blocks);                       \
        }                                                                                       \
    };
COMERGE_CUDA_REC_GENERIC(std::int32_t, i32)
COMERGE_CUDA_REC_GENERIC(std::uint32_t, u32)
COMERGE_CUDA_REC_GENERIC(std::uint64_t, u64)
#undef COMERGE_CUDA_REC_GENERIC

template <typename A, typename B, typename Out>
merge_report run_merge_records(const A& a, const B& b, Out& out, std::size_t workers,
                               bool synced, merge_options opts = {}) {
    using T = elem_of<A>;
    using K = std::remove_cv_t<decltype(T::key)>;
    comerge_merge_report rep{};
    const comerge_merge_options o{synced ? 1 : 0, opts.count_comparisons ? 1 : 0};
    std::vector<std::uint64_t> bs(workers ? workers : 1);
    std::vector<std::uint32_t> its(2 * (workers ? workers : 1));
    std::uint64_t cmp = 0;
    check(rec_generic<K>::merge_ex(std::ranges::data(a), std::ranges::size(a),
                                   std::ranges::data(b), std::ranges::size(b),
                                   std::ranges::data(out), std::ranges::size(out), sizeof(T),
                                   workers, &o, &rep, bs.data(), its.data(), &cmp));
    merge_report r = to_report(rep);
    r.block_sizes.assign(bs.begin(), bs.begin() + workers);
    r.corank_iterations.assign(its.begin(), its.begin() + (synced ? workers : 2 * workers));
    if (opts.count_comparisons) r.comparisons = cmp;
    return r;
}
}  // namespace detail

/// comerge::merge_parallel over key-value records with a key-only comparator
/// (parallel.hpp:304-317 instantiated with tagged<K> / tagged_key_less): ties
/// keep A first, then input order; records move whole.
template <detail::record_range A, detail::record_range B, std::ranges::contiguous_range Out,
          typename Less>
    requires std::same_as<detail::elem_of<A>, detail::elem_of<B>> &&
             std::same_as<detail::elem_of<A>, std::ranges::range_value_t<Out>> &&
             is_key_less<Less>::value
merge_report merge_parallel(const A& a, const B& b, Out&& out, std::size_t workers, Less,
                            merge_options opts = {}) {
    return detail::run_merge_records(a, b, out, workers, false, opts);
}

/// comerge::merge_parallel_synced over records (parallel.hpp:323-336).
template <detail::record_range A, detail::record_range B, std::ranges::contiguous_range Out,
          typename Less>
    requires std::same_as<detail::elem_of<A>, detail::elem_of<B>> &&
             std::same_as<detail::elem_of<A>, std::ranges::range_value_t<Out>> &&
             is_key_less<Less>::value
merge_report merge_parallel_synced(const A& a, const B& b, Out&& out, std::size_t workers, Less,
                                   merge_options opts = {}) {
    return detail::run_merge_records(a, b, out, workers, true, opts);
}

/// comerge::co_rank over records with a key-only comparator (corank.hpp:128-133;
/// the comparator known-answer test of corank_test.cpp:205-214).
template <detail::record_range A, detail::record_range B, typename Less>
    requires std::same_as<detail::elem_of<A>, detail::elem_of<B>> && is_key_less<Less>::value
co_ranks co_rank(rank_t target, const A& a, const B& b, Less, co_rank_stats* stats = nullptr) {
    using T = detail::elem_of<A>;
    using K = std::remove_cv_t<decltype(T::key)>;
    std::uint64_t j = 0, k = 0;
    std::uint32_t it = 0, cmp = 0;
    detail::check(detail::rec_generic<K>::co_rank(target, std::ranges::data(a),
                                                  std::ranges::size(a), std::ranges::data(b),
                                                  std::ranges::size(b), sizeof(T), &j, &k, &it,
                                                  &cmp));
    if (stats) *stats = {it, cmp};
    return {static_cast<std::size_t>(j), static_cast<std::size_t>(k)};
}

/// comerge::co_rank_counted over records (corank.hpp:138-147).
template <detail::record_range A, detail::record_range B, typename Less>
    requires std::same_as<detail::elem_of<A>, detail::elem_of<B>> && is_key_less<Less>::value
co_ranks co_rank_counted(rank_t target, const A& a, const B& b, Less less,
                         comparison_counter& counter) {
    co_rank_stats st;
    const co_ranks r = co_rank(target, a, b, less, &st);
    counter.count += st.comparisons;
    return r;
}

/// comerge::stable_merge over records (merge.hpp:52-68).
template <detail::record_range A, detail::record_range B, std::ranges::contiguous_range Out,
          typename Less>
    requires std::same_as<detail::elem_of<A>, detail::elem_of<B>> &&
             std::same_as<detail::elem_of<A>, std::ranges::range_value_t<Out>> &&
             is_key_less<Less>::value
void stable_merge(const A& a, const B& b, Out&& out, Less) {
    try {
        detail::run_merge_records(a, b, out, 1, false);
    } catch (const std::invalid_argument& e) {
        std::string msg = e.what();
        const auto pos = msg.find("merge_parallel");
        if (pos != std::string::npos) msg.replace(pos, 14, "stable_merge");
        throw std::invalid_argument(msg);
    }
}

/// Key-value merge over SoA arrays (keys + uint32 payload).
template <detail::key_range A, detail::key_range B, std::ranges::contiguous_range Out>
    requires std::same_as<detail::key_of<A>, detail::key_of<B>> &&
             std::same_as<detail::key_of<A>, std::ranges::range_value_t<Out>>
merge_report merge_parallel_pairs(const A& a_keys, std::span<const std::uint32_t> a_vals,
                                  const B& b_keys, std::span<const std::uint32_t> b_vals,
                                  Out&& out_keys, std::span<std::uint32_t> out_vals,
                                  std::size_t workers = 1) {
    using K = detail::key_of<A>;
    if (a_vals.size() != std::ranges::size(a_keys) || b_vals.size() != std::ranges::size(b_keys) ||
        out_vals.size() != std::ranges::size(out_keys))
        throw std::invalid_argument("merge_parallel_pairs: payload length must equal key length");
    comerge_merge_report rep{};
    detail::check(detail::abi<K>::merge_pairs(
        std::ranges::data(a_keys), a_vals.data(), std::ranges::size(a_keys),
        std::ranges::data(b_keys), b_vals.data(), std::ranges::size(b_keys),
        std::ranges::data(out_keys), out_vals.data(), std::ranges::size(out_keys), workers, &rep));
    return detail::to_report(rep);
}

/// Central per-worker assignment (two independent co-ranks per block), all
/// co-ranks in one batched device launch.
template <detail::key_range A, detail::key_range B>
    requires std::same_as<detail::key_of<A>, detail::key_of<B>>
merge_plan plan(const A& a, const B& b, std::size_t workers, std::less<> = {}) {
    using K = detail::key_of<A>;
    if (workers == 0) throw std::invalid_argument("plan: worker count must be positive");
    std::vector<std::uint64_t> raw(7 * workers);
    detail::check(detail::abi<K>::plan(std::ranges::data(a), std::ranges::size(a),
                                       std::ranges::data(b), std::ranges::size(b), workers,
                                       raw.data()));
    merge_plan p;
    p.workers = workers;
    for (std::size_t r = 0; r < workers; ++r) {
        const std::uint64_t* o = raw.data() + 7 * r;
        p.blocks.push_back({static_cast<std::size_t>(o[0]), static_cast<rank_t>(o[1]),
                            static_cast<rank_t>(o[2]), static_cast<std::size_t>(o[3]),
                            static_cast<std::size_t>(o[4]), static_cast<std::size_t>(o[5]),
                            static_cast<std::size_t>(o[6])});
    }
    return p;
}

/// comerge::plan over records with a key-only comparator (parallel.hpp:94-115).
template <detail::record_range A, detail::record_range B, typename Less>
    requires std::same_as<detail::elem_of<A>, detail::elem_of<B>> && is_key_less<Less>::value
merge_plan plan(const A& a, const B& b, std::size_t workers, Less) {
    using T = detail::elem_of<A>;
    using K = std::remove_cv_t<decltype(T::key)>;
    if (workers == 0) throw std::invalid_argument("plan: worker count must be positive");
    std::vector<std::uint64_t> raw(7 * workers);
    detail::check(detail::rec_generic<K>::plan(std::ranges::data(a), std::ranges::size(a),
                                               std::ranges::data(b), std::ranges::size(b),
                                               sizeof(T), workers, raw.data()));
    merge_plan p;
    p.workers = workers;
    for (std::size_t r = 0; r < workers; ++r) {
        const std::uint64_t* o = raw.data() + 7 * r;
        p.blocks.push_back({static_cast<std::size_t>(o[0]), static_cast<rank_t>(o[1]),
                            static_cast<rank_t>(o[2]), static_cast<std::size_t>(o[3]),
                            static_cast<std::size_t>(o[4]), static_cast<std::size_t>(o[5]),
                            static_cast<std::size_t>(o[6])});
    }
    return p;
}

}  // namespace comerge::cuda
