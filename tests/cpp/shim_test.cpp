// shim_test.cpp -- the reference's own unit-test cases (corank_test.cpp,
// merge_test.cpp, parallel_test.cpp; /root/reference/proj/tests), replayed
// against the B200 drop-in comerge::cuda (include/comerge/cuda.hpp), plus
// seeded sweeps checked against a naive two-finger merge (test-only oracle,
// written as plainly as the reference's oracle.hpp:98-119).
//
// Exit code = number of failed checks.  Needs a GPU (run by tests/test_cpp_shim.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <functional>
#include <random>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "comerge/cuda.hpp"

namespace cm = comerge::cuda;

static int g_fail = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            ++g_fail;                                                          \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                      \
    } while (0)

template <typename Ex, typename Fn>
static bool throws_with(Fn&& fn, const char* needle) {
    try {
        fn();
    } catch (const Ex& e) {
        return std::string(e.what()).find(needle) != std::string::npos;
    } catch (...) {
        return false;
    }
    return false;
}

template <typename K>
static std::vector<K> naive_merge(const std::vector<K>& a, const std::vector<K>& b) {
    std::vector<K> out;
    std::size_t x = 0, y = 0;
    while (x < a.size() && y < b.size()) out.push_back(a[x] <= b[y] ? a[x++] : b[y++]);
    while (x < a.size()) out.push_back(a[x++]);
    while (y < b.size()) out.push_back(b[y++]);
    return out;
}

using keys = std::vector<std::uint64_t>;

static void kats() {
    // corank_test.cpp:22-56
    cm::co_rank_stats st;
    CHECK((cm::co_rank(0, keys{1, 3, 5, 7}, keys{2, 4, 6, 8}, {}, &st) == cm::co_ranks{0, 0}));
    CHECK(st.iterations == 0 && st.comparisons == 0);
    CHECK((cm::co_rank(8, keys{1, 3, 5, 7}, keys{2, 4, 6, 8}, {}, &st) == cm::co_ranks{4, 4}));
    CHECK(st.iterations == 0 && st.comparisons == 0);
    CHECK((cm::co_rank(0, keys{}, keys{}) == cm::co_ranks{0, 0}));
    CHECK((cm::co_rank(4, keys{1, 3, 5, 7}, keys{2, 4, 6, 8}) == cm::co_ranks{2, 2}));
    CHECK((cm::co_rank(2, keys{2, 2}, keys{2, 2}) == cm::co_ranks{2, 0}));
    CHECK((cm::co_rank(3, keys{10, 20}, keys{1, 2, 3, 4, 5}) == cm::co_ranks{0, 3}));
    CHECK((cm::co_rank(1, keys{1}, keys{2}) == cm::co_ranks{1, 0}));
    for (std::size_t i = 0; i <= 3; ++i) {
        CHECK((cm::co_rank(i, keys{5, 6, 7}, keys{}, {}, &st) == cm::co_ranks{i, 0}));
        CHECK(st.comparisons == 0);
        CHECK((cm::co_rank(i, keys{}, keys{5, 6, 7}, {}, &st) == cm::co_ranks{0, i}));
    }
    // corank_test.cpp:58-63
    CHECK(throws_with<std::out_of_range>([] { cm::co_rank(4, keys{1, 2}, keys{3}); },
                                         "rank out of range"));
    CHECK(throws_with<std::out_of_range>([] { cm::co_rank(100, keys{1, 2}, keys{3}); },
                                         "rank out of range"));
    // merge_test.cpp:17-35, :53-70
    keys out(2);
    cm::stable_merge(keys{}, keys{1, 2}, out);
    CHECK((out == keys{1, 2}));
    keys out4(4);
    cm::stable_merge(keys{1, 3}, keys{2, 3}, out4);
    CHECK((out4 == keys{1, 2, 3, 3}));
    CHECK(throws_with<std::invalid_argument>(
        [] {
            keys small(2);
            cm::stable_merge(keys{1, 2}, keys{3}, small);
        },
        "output length must equal |a| + |b|"));
    // stability through payloads (merge_test.cpp:37-51)
    {
        const std::vector<std::uint32_t> ak{5, 5}, bk{5};
        const std::vector<std::uint32_t> av{0, 1}, bv{0x80000000u};
        std::vector<std::uint32_t> ok(3), ov(3);
        cm::merge_parallel_pairs(ak, av, bk, bv, ok, std::span<std::uint32_t>(ov));
        CHECK((ov == std::vector<std::uint32_t>{0, 1, 0x80000000u}));
    }
    // parallel_test.cpp:28-32, :63-71
    const std::vector<std::size_t> expect{0, 3, 6, 10};
    for (std::size_t r = 0; r <= 3; ++r) CHECK(cm::partition_output(10, 3, r) == expect[r]);
    const std::size_t big = std::size_t{1} << 62;
    CHECK(cm::partition_output(big, 3, 3) == big);
    CHECK(cm::partition_output(big, 3, 1) == big / 3);
    CHECK(throws_with<std::invalid_argument>([] { cm::partition_output(10, 0, 0); }, "worker"));
    // parallel_test.cpp:74-91
    {
        const auto p = cm::plan(keys{2, 2}, keys{2, 2}, 2);
        CHECK((p.blocks[0] == cm::block_assignment{0, 0, 2, 0, 2, 0, 0}));
        CHECK((p.blocks[1] == cm::block_assignment{1, 2, 4, 2, 2, 0, 2}));
        const auto q = cm::plan(keys{}, keys{0, 1, 2, 3, 4, 5, 6, 7, 8, 9}, 2);
        CHECK((q.blocks[0] == cm::block_assignment{0, 0, 5, 0, 0, 0, 5}));
    }
    // parallel_test.cpp:190-212
    {
        keys e;
        const auto rep = cm::merge_parallel(keys{}, keys{}, e, 4);
        CHECK((rep.block_sizes == std::vector<std::size_t>(4, 0)));
        keys o3(3);
        cm::merge_parallel(keys{1, 3}, keys{2}, o3, 9);
        CHECK((o3 == keys{1, 2, 3}));
        CHECK(throws_with<std::invalid_argument>(
            [] {
                keys w(3);
                cm::merge_parallel(keys{1}, keys{2}, w, 2);
            },
            "output length must equal"));
        CHECK(throws_with<std::invalid_argument>(
            [] {
                keys w(2);
                cm::merge_parallel(keys{1}, keys{2}, w, 0);
            },
            "worker count must be positive"));
    }
}

// merge_options::count_comparisons (parallel.hpp:41, :253-280): absent unless
// requested (parallel_test.cpp:186); when requested, the reference's total --
// here recomputed the reference's way: Algorithm 1's comparisons at both ends
// of every block plus a counted two-finger merge of every block.
static void comparisons() {
    std::mt19937_64 rng(11);
    keys a(3000), b(2000);
    for (auto& x : a) x = rng() % 50;
    for (auto& x : b) x = rng() % 50;
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    keys out(5000);
    CHECK(!cm::merge_parallel(a, b, out, 7).comparisons.has_value());
    for (std::size_t w : {std::size_t{1}, std::size_t{7}, std::size_t{64}}) {
        cm::merge_options opts;
        opts.count_comparisons = true;
        const auto rep = cm::merge_parallel(a, b, out, w, {}, opts);
        std::uint64_t expect = 0;
        for (std::size_t r = 0; r < w; ++r) {
            const auto lo = cm::partition_output(5000, w, r), hi = cm::partition_output(5000, w, r + 1);
            cm::co_rank_stats s0, s1;
            const auto c0 = cm::co_rank(lo, a, b, {}, &s0), c1 = cm::co_rank(hi, a, b, {}, &s1);
            std::size_t x = c0.a, y = c0.b;
            std::uint64_t kc = 0;
            while (x < c1.a && y < c1.b) {
                ++kc;
                if (b[y] < a[x]) ++y; else ++x;
            }
            expect += s0.comparisons + s1.comparisons + kc;
        }
        CHECK(rep.comparisons.has_value() && *rep.comparisons == expect);
    }
}

template <typename K>
static void sweep(std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    const std::vector<std::pair<std::size_t, std::size_t>> shapes = {
        {0, 5}, {7, 0}, {1, 1}, {3000, 20000}, {20000, 3}, {4096, 4096}, {100000, 77777},
        {1 << 20, 5000}};
    for (auto [m, n] : shapes) {
        for (std::uint64_t alphabet : {std::uint64_t{3}, std::uint64_t{1} << 20}) {
            std::vector<K> a(m), b(n);
            for (auto& x : a) x = K(rng() % alphabet);
            for (auto& x : b) x = K(rng() % alphabet);
            std::sort(a.begin(), a.end());
            std::sort(b.begin(), b.end());
            const std::vector<K> expect = naive_merge(a, b);
            for (std::size_t workers : {1, 3, 16}) {
                std::vector<K> out(m + n, K(0x5a));
                const auto rep = cm::merge_parallel(a, b, out, workers);
                CHECK(out == expect);
                CHECK(rep.block_sizes.size() == workers);
                CHECK(rep.corank_iterations.size() == 2 * workers);
            }
            // device spans through the same entry point
            K *da = nullptr, *db = nullptr, *dout = nullptr;
            cudaMalloc(&da, (m + 1) * sizeof(K));
            cudaMalloc(&db, (n + 1) * sizeof(K));
            cudaMalloc(&dout, (m + n + 1) * sizeof(K));
            cudaMemcpy(da, a.data(), m * sizeof(K), cudaMemcpyHostToDevice);
            cudaMemcpy(db, b.data(), n * sizeof(K), cudaMemcpyHostToDevice);
            cm::device_span<const K> sa{da, m}, sb{db, n};
            cm::device_span<K> so{dout, m + n};
            cm::merge_parallel_synced(sa, sb, so, 4);
            std::vector<K> back(m + n);
            cudaMemcpy(back.data(), dout, (m + n) * sizeof(K), cudaMemcpyDeviceToHost);
            CHECK(back == expect);
            cudaFree(da);
            cudaFree(db);
            cudaFree(dout);
        }
    }
}

// The reference's key-value shape as a caller holds it: tagged<K> with a
// key-only comparator (oracle.hpp:22-37), declared key-only for the device.
enum class origin : std::uint8_t { from_a, from_b };
template <typename K>
struct tagged {
    K key{};
    origin from = origin::from_a;
    std::uint32_t index = 0;
    friend bool operator==(const tagged&, const tagged&) = default;
};
struct tagged_key_less {
    template <typename K>
    bool operator()(const tagged<K>& x, const tagged<K>& y) const {
        return x.key < y.key;
    }
};
template <>
struct comerge::cuda::is_key_less<tagged_key_less> : std::true_type {};

template <typename T>
static std::vector<T> naive_merge_by_key(const std::vector<T>& a, const std::vector<T>& b) {
    std::vector<T> out;
    std::size_t x = 0, y = 0;
    while (x < a.size() && y < b.size()) out.push_back(b[y].key < a[x].key ? b[y++] : a[x++]);
    while (x < a.size()) out.push_back(a[x++]);
    while (y < b.size()) out.push_back(b[y++]);
    return out;
}

static void records() {
    std::mt19937_64 rng(77);
    // acceptance_test.cpp:213-235 shape: tagged elements, the tagged oracle
    for (auto [m, n, alphabet] : {std::tuple<std::size_t, std::size_t, unsigned>{0, 0, 3},
                                  {1, 0, 3}, {0, 5, 3}, {1000, 999, 4}, {5000, 3, 50},
                                  {200003, 150001, 100}, {1 << 20, (1 << 20) + 3, 1000}}) {
        std::vector<tagged<std::uint64_t>> ta(m), tb(n);
        std::vector<std::uint64_t> ka(m), kb(n);
        for (auto& x : ka) x = rng() % alphabet;
        for (auto& x : kb) x = rng() % alphabet;
        std::sort(ka.begin(), ka.end());
        std::sort(kb.begin(), kb.end());
        for (std::size_t i = 0; i < m; ++i) ta[i] = {ka[i], origin::from_a, std::uint32_t(i)};
        for (std::size_t i = 0; i < n; ++i) tb[i] = {kb[i], origin::from_b, std::uint32_t(i)};
        const auto expect = naive_merge_by_key(ta, tb);
        for (std::size_t workers : {1, 4, 33}) {
            std::vector<tagged<std::uint64_t>> out(m + n);
            const auto rep = cm::merge_parallel(ta, tb, out, workers, tagged_key_less{});
            CHECK(out == expect);
            CHECK(rep.block_sizes.size() == workers);
        }
        // the reference's tagged<int32_t> / tagged<uint32_t>: 12-byte records,
        // host vectors and (offset) device views
        static_assert(sizeof(tagged<std::int32_t>) == 12 && sizeof(tagged<std::uint32_t>) == 12);
        {
            std::vector<tagged<std::int32_t>> ia(m), ib(n);
            for (std::size_t i = 0; i < m; ++i)
                ia[i] = {std::int32_t(ka[i]) - 3, origin::from_a, std::uint32_t(i)};
            for (std::size_t i = 0; i < n; ++i)
                ib[i] = {std::int32_t(kb[i]) - 3, origin::from_b, std::uint32_t(i)};
            const auto iexpect = naive_merge_by_key(ia, ib);
            for (std::size_t workers : {1, 7}) {
                std::vector<tagged<std::int32_t>> out(m + n);
                cm::merge_parallel(ia, ib, out, workers, tagged_key_less{});
                CHECK(out == iexpect);
            }
            std::vector<tagged<std::uint32_t>> ua(m), ub(n);
            for (std::size_t i = 0; i < m; ++i)
                ua[i] = {std::uint32_t(ka[i]), origin::from_a, std::uint32_t(i)};
            for (std::size_t i = 0; i < n; ++i)
                ub[i] = {std::uint32_t(kb[i]), origin::from_b, std::uint32_t(i)};
            using U = tagged<std::uint32_t>;
            U *ua_d = nullptr, *ub_d = nullptr, *uo_d = nullptr;
            cudaMalloc(&ua_d, (m + 1) * sizeof(U));
            cudaMalloc(&ub_d, (n + 3) * sizeof(U));
            cudaMalloc(&uo_d, (m + n + 2) * sizeof(U));
            cudaMemcpy(ua_d + 1, ua.data(), m * sizeof(U), cudaMemcpyHostToDevice);
            cudaMemcpy(ub_d + 3, ub.data(), n * sizeof(U), cudaMemcpyHostToDevice);
            cm::device_span<const U> sa{ua_d + 1, m}, sb{ub_d + 3, n};
            cm::device_span<U> so{uo_d + 2, m + n};
            cm::stable_merge(sa, sb, so, tagged_key_less{});
            std::vector<U> back(m + n);
            cudaMemcpy(back.data(), uo_d + 2, (m + n) * sizeof(U), cudaMemcpyDeviceToHost);
            CHECK(back == naive_merge_by_key(ua, ub));
            cudaFree(ua_d);
            cudaFree(ub_d);
            cudaFree(uo_d);
        }
        // 8-byte records with 32-bit keys, on the device
        std::vector<cm::record<std::int32_t>> ra(m), rb(n);
        for (std::size_t i = 0; i < m; ++i) ra[i] = {std::int32_t(ka[i]) - 7, std::uint32_t(i)};
        for (std::size_t i = 0; i < n; ++i) rb[i] = {std::int32_t(kb[i]) - 7, std::uint32_t(i) | 1u << 31};
        const auto rexpect = naive_merge_by_key(ra, rb);
        using R = cm::record<std::int32_t>;
        R *da = nullptr, *db = nullptr, *dout = nullptr;
        cudaMalloc(&da, (m + 1) * sizeof(R));
        cudaMalloc(&db, (n + 1) * sizeof(R));
        cudaMalloc(&dout, (m + n + 1) * sizeof(R));
        cudaMemcpy(da + 1, ra.data(), m * sizeof(R), cudaMemcpyHostToDevice);  // offset views
        cudaMemcpy(db, rb.data(), n * sizeof(R), cudaMemcpyHostToDevice);
        cm::device_span<const R> sa{da + 1, m}, sb{db, n};
        cm::device_span<R> so{dout + 1, m + n};
        cm::stable_merge(sa, sb, so, cm::key_less{});
        std::vector<R> back(m + n);
        cudaMemcpy(back.data(), dout + 1, (m + n) * sizeof(R), cudaMemcpyDeviceToHost);
        CHECK(back == rexpect);
        cudaFree(da);
        cudaFree(db);
        cudaFree(dout);
    }
    // merge.hpp:62-66 contract through the record overloads
    std::vector<cm::record<std::uint32_t>> x(3), y(2), bad(4);
    CHECK(throws_with<std::invalid_argument>(
        [&] { cm::stable_merge(x, y, bad, cm::key_less{}); }, "output length must equal"));
    CHECK(throws_with<std::invalid_argument>(
        [&] { cm::merge_parallel(x, y, bad, 2, cm::key_less{}); }, "output length must equal"));
}

// co_rank / co_rank_counted / plan / merge_parallel_synced / count_comparisons
// over records with a key-only comparator: everything equals the same call on
// the records' key arrays (only keys are compared).
static void records_api() {
    // corank_test.cpp:205-214: ordering on the first component only, ties stay
    // a-before-b ({int, char} as an 8-byte record with the key first)
    struct pr {
        std::int32_t key;
        char tag;
    };
    static_assert(sizeof(pr) == 8);
    const std::vector<pr> pa{{1, 'x'}, {2, 'y'}}, pb{{1, 'z'}, {2, 'w'}};
    CHECK((cm::co_rank(1, pa, pb, cm::key_less{}) == cm::co_ranks{1, 0}));
    CHECK((cm::co_rank(2, pa, pb, cm::key_less{}) == cm::co_ranks{1, 1}));
    CHECK((cm::co_rank(3, pa, pb, cm::key_less{}) == cm::co_ranks{2, 1}));
    CHECK(throws_with<std::out_of_range>([&] { cm::co_rank(5, pa, pb, cm::key_less{}); },
                                         "rank out of range"));
    std::mt19937_64 rng(21);
    const std::size_t m = 3001, n = 1777;
    keys ka(m), kb(n);
    for (auto& x : ka) x = rng() % 40;
    for (auto& x : kb) x = rng() % 40;
    std::sort(ka.begin(), ka.end());
    std::sort(kb.begin(), kb.end());
    auto check_shape = [&](auto tag, auto keys_tag) {
        using T = decltype(tag);
        using K = decltype(keys_tag);
        std::vector<T> ta(m), tb(n);
        std::vector<K> xa(m), xb(n);
        for (std::size_t i = 0; i < m; ++i) {
            xa[i] = K(ka[i]);
            ta[i] = {K(ka[i]), origin::from_a, std::uint32_t(i)};
        }
        for (std::size_t i = 0; i < n; ++i) {
            xb[i] = K(kb[i]);
            tb[i] = {K(kb[i]), origin::from_b, std::uint32_t(i)};
        }
        for (std::size_t i : {std::size_t{0}, std::size_t{1}, m, (m + n) / 2, m + n - 1, m + n}) {
            cm::co_rank_stats sr, sk;
            CHECK((cm::co_rank(i, ta, tb, tagged_key_less{}, &sr) == cm::co_rank(i, xa, xb, {}, &sk)));
            CHECK(sr.iterations == sk.iterations && sr.comparisons == sk.comparisons);
            cm::comparison_counter cr, ck;
            cm::co_rank_counted(i, ta, tb, tagged_key_less{}, cr);
            cm::co_rank_counted(i, xa, xb, {}, ck);
            CHECK(cr.count == ck.count);
        }
        for (std::size_t w : {std::size_t{1}, std::size_t{5}, std::size_t{64}}) {
            const auto pr_ = cm::plan(ta, tb, w, tagged_key_less{});
            const auto pk = cm::plan(xa, xb, w);
            CHECK(pr_.workers == w && pr_.blocks == pk.blocks);
            cm::merge_options opts;
            opts.count_comparisons = true;
            std::vector<T> out(m + n);
            std::vector<K> kout(m + n);
            const auto expect = naive_merge_by_key(ta, tb);
            for (bool synced : {false, true}) {
                const auto rr = synced ? cm::merge_parallel_synced(ta, tb, out, w, tagged_key_less{}, opts)
                                       : cm::merge_parallel(ta, tb, out, w, tagged_key_less{}, opts);
                const auto rk = synced ? cm::merge_parallel_synced(xa, xb, kout, w, {}, opts)
                                       : cm::merge_parallel(xa, xb, kout, w, {}, opts);
                CHECK(out == expect);
                CHECK(rr.comparisons.has_value() && rr.comparisons == rk.comparisons);
                CHECK(rr.block_sizes == rk.block_sizes);
                CHECK(rr.corank_iterations == rk.corank_iterations);
                CHECK(rr.corank_iterations.size() == (synced ? w : 2 * w));
            }
            CHECK(!cm::merge_parallel(ta, tb, out, w, tagged_key_less{}).comparisons.has_value());
        }
        CHECK(throws_with<std::invalid_argument>([&] { cm::plan(ta, tb, 0, tagged_key_less{}); },
                                                 "worker count must be positive"));
    };
    check_shape(tagged<std::uint64_t>{}, std::uint64_t{});
    check_shape(tagged<std::int32_t>{}, std::int32_t{});
    check_shape(tagged<std::uint32_t>{}, std::uint32_t{});
}

// host-buffer merges of vectors in page-locked memory (pinned_allocator)
static void pinned_vectors() {
    std::mt19937_64 rng(5);
    const std::size_t m = 1500001, n = 1200003;  // >= 2^20: the chunked host pipeline
    std::vector<std::uint64_t> ka(m), kb(n);
    for (auto& x : ka) x = rng();
    for (auto& x : kb) x = rng();
    std::sort(ka.begin(), ka.end());
    std::sort(kb.begin(), kb.end());
    std::vector<std::uint64_t, cm::pinned_allocator<std::uint64_t>> pa(ka.begin(), ka.end()),
        pb(kb.begin(), kb.end()), out(m + n);
    cm::merge_parallel(pa, pb, out, 8);
    std::vector<std::uint64_t> expect(m + n);
    std::merge(ka.begin(), ka.end(), kb.begin(), kb.end(), expect.begin());
    CHECK(std::equal(out.begin(), out.end(), expect.begin()));
    std::vector<tagged<std::int32_t>, cm::pinned_allocator<tagged<std::int32_t>>> ta(m), tb(n),
        to(m + n);
    for (std::size_t i = 0; i < m; ++i) ta[i] = {std::int32_t(ka[i] >> 40), origin::from_a, std::uint32_t(i)};
    for (std::size_t i = 0; i < n; ++i) tb[i] = {std::int32_t(kb[i] >> 40), origin::from_b, std::uint32_t(i)};
    cm::merge_parallel(ta, tb, to, 8, tagged_key_less{});
    const auto texpect = naive_merge_by_key(std::vector<tagged<std::int32_t>>(ta.begin(), ta.end()),
                                            std::vector<tagged<std::int32_t>>(tb.begin(), tb.end()));
    CHECK(std::equal(to.begin(), to.end(), texpect.begin()));
}

int main() {
    kats();
    pinned_vectors();
    comparisons();
    records();
    records_api();
    sweep<std::int32_t>(1);
    sweep<std::uint32_t>(2);
    sweep<std::uint64_t>(3);
    std::printf("shim_test: %d failure(s)\n", g_fail);
    return g_fail;
}
