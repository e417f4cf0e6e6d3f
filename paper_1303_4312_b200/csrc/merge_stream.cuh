// merge_stream.cuh -- persistent, warp-specialised streaming merge (sm_100a).
//
// Algorithm 2 of arXiv 1303.4312 (reference
// parallel.hpp:201-207) with one CTA per worker:
//
//   * The grid is the persistent set of G = (#SMs x CTAs/SM) workers.  CTA c
//     owns the output tiles [floor(c*ntiles/G), floor((c+1)*ntiles/G)) -- the
//     reference's partition_output (parallel.hpp:60-67) over tiles, so block
//     sizes differ by at most one tile (Proposition 2).
//   * Each CTA co-ranks both ends of its block itself (synchronisation-free
//     form, parallel.hpp:204-205): warps 0-3 search the start diagonal and
//     warps 4-7 the end diagonal with a 129-ary cooperative search of the
//     Lemma-1 predicate (4 dependent probe rounds for 2^27-element inputs
//     instead of ~27 for a binary search).  No partition kernel, no
//     workspace.
//   * Producer warp (warp 8): streams the CTA's A window [j_c, j_{c+1}) and
//     B window [k_c, k_{c+1}) through two shared-memory rings of NS chunks
//     with cp.async.bulk (TMA 1-D bulk copies, 16-byte aligned), completion
//     on one mbarrier per slot; consumers release a slot through an "empty"
//     mbarrier once the merge front has passed it.  Every input byte is read
//     from HBM once.
//   * Consumer warps (0-7): per output tile of T = 256*VT elements, every
//     thread co-ranks its VT-slot diagonal inside the ring windows (the same
//     split, now in shared memory), runs the branch-free serial merge of
//     merge.hpp:22-31 (take b only when b < a) for VT elements in registers,
//     writes them to a double-buffered staging tile, and one thread stores the
//     tile with a TMA bulk store (cp.async.bulk.global.shared::cta).  The end
//     of a tile's merge path is the start of the next one, so tiles need no
//     global co-rank at all.
#pragma once

#include <cstdint>

#include "corank.cuh"
#include "merge_tile.cuh"

namespace comerge_b200 {

// ------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}

// Same, letting the waiting thread sleep up to `hint_ns` inside try_wait
// (returns as soon as the phase completes): fewer spin iterations for
// latency-tolerant waiters.
__device__ __forceinline__ void mbar_wait_sleepy(uint64_t* bar, uint32_t parity,
                                                 uint32_t hint_ns) {
    uint32_t ok;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity), "r"(hint_ns)
            : "memory");
    } while (!ok);
}

// 1-D TMA bulk copy global -> shared, completing `bytes` on `bar`.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// 1-D TMA bulk copy shared -> global (bulk async-group).
__device__ __forceinline__ void tma_store_1d(void* dst, const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}

// bulk store with an L2 eviction-priority hint (streamed output: evict_first
// keeps it from displacing lines that are read again soon)
__device__ __forceinline__ void tma_store_1d_hint(void* dst, const void* src, uint32_t bytes,
                                                  uint64_t policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(policy)
                 : "memory");
}

// bulk prefetch of global memory into L2 (no completion to wait for)
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void tma_store_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int N>
__device__ __forceinline__ void tma_store_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void tma_store_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// arrive on a named barrier without waiting (producer side of bar.sync)
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// ------------------------------------------------------------ configuration
//
// Each tile of T outputs needs up to T elements of EACH input resident (the
// merge path may take all of them from one side); what the rings hold beyond
// that window is prefetch.  Rings are NS chunks of CH elements (NS need not be
// a power of two: a ring index is wrapped with one conditional subtract).
// Budgets target 2 CTAs per SM (<= ~110 KB each) with >= 24 KB of prefetch
// per input per CTA.

template <typename K, bool HAS_V>
struct stream_cfg;

// 32-bit keys only: tile 3840, chunk 4 KB, ring 12 chunks (48 KB) per input.
template <>
struct stream_cfg<int32_t, false> {
    static constexpr int VT = 15, CH = 1024, NS = 12;
};
template <>
struct stream_cfg<uint32_t, false> : stream_cfg<int32_t, false> {};
// 32-bit keys + payload: tile 1792, chunk 512, ring 6144 elements (48 KB).
template <>
struct stream_cfg<int32_t, true> {
    static constexpr int VT = 7, CH = 512, NS = 12;
};
template <>
struct stream_cfg<uint32_t, true> : stream_cfg<int32_t, true> {};
// 64-bit keys only: tile 1792, ring 6144 elements (48 KB).
template <>
struct stream_cfg<uint64_t, false> {
    static constexpr int VT = 7, CH = 512, NS = 12;
};
// 64-bit keys + payload: tile 1280, chunk 256, ring 3584 elements (42 KB).
template <>
struct stream_cfg<uint64_t, true> {
    static constexpr int VT = 5, CH = 256, NS = 14;
};

template <typename K, bool HAS_V>
struct stream_layout {
    using C = stream_cfg<K, HAS_V>;
    static constexpr int kConsumers = 256;
    static constexpr int kThreads = kConsumers + 32;  // + producer warp
    static constexpr int VT = C::VT;
    static constexpr int T = kConsumers * VT;
    static constexpr int CH = C::CH;
    static constexpr int NS = C::NS;
    static constexpr int RING = CH * NS;  // elements per input ring
    static_assert(RING >= T + CH, "ring must hold a full tile window plus one chunk");
    static_assert((T * sizeof(K)) % 16 == 0 && (T * 4) % 16 == 0, "tile must be 16B multiple");
    static_assert((CH * sizeof(K)) % 16 == 0 && CH % 4 == 0, "chunks must be 16B multiples");
    static constexpr int VECE = 16 / sizeof(K);  // elements per 16 bytes
    // byte offsets in dynamic shared memory
    static constexpr size_t kRingKeys = size_t(RING) * sizeof(K);
    static constexpr size_t kRingVals = HAS_V ? size_t(RING) * 4 : 0;
    static constexpr size_t oRingA = 0;
    static constexpr size_t oRingB = oRingA + kRingKeys;
    static constexpr size_t oRingAV = oRingB + kRingKeys;
    static constexpr size_t oRingBV = oRingAV + kRingVals;
    static constexpr size_t oStage = oRingBV + kRingVals;
    static constexpr size_t kStageKeys = size_t(T) * sizeof(K);
    static constexpr size_t kStageVals = HAS_V ? size_t(T) * 4 : 0;
    static constexpr size_t oBars = oStage + kStageKeys + kStageVals;
    static constexpr size_t kBars = size_t(4 * NS) * 8;
    static constexpr size_t oMisc = oBars + kBars;
    static constexpr size_t kMisc = 128;
    static constexpr size_t kSmem = oMisc + kMisc;
};

// ------------------------------------------------------------ block search

// Cooperative P-ary search of the Lemma-1 split for diagonal i by the P
// threads of group `bar_id` (gtid in [0, P)); `cnt` is P/32 shared slots.
template <typename K, int P>
__device__ __forceinline__ uint64_t group_co_rank(uint64_t i, const K* __restrict__ a, uint64_t m,
                                                  const K* __restrict__ b, uint64_t n, int gtid,
                                                  int bar_id, volatile int* cnt) {
    uint64_t lo = i > n ? i - n : 0;
    uint64_t hi = i < m ? i : m;
    int round = 0;
    while (hi > lo) {
        const uint64_t width = hi - lo;
        const uint64_t q = lo + 1 + ((width - 1) * uint64_t(gtid)) / uint64_t(P - 1);
        // P(q): too much taken from a (guard 1, corank.hpp:93-94)
        const bool too_far = ldg_elem(b + (i - q)) < ldg_elem(a + (q - 1));
        const unsigned ballot = __ballot_sync(0xffffffffu, !too_far);
        volatile int* slot = cnt + (round & 1) * (P / 32);
        if ((gtid & 31) == 0) slot[gtid >> 5] = __popc(ballot);
        named_bar_sync(bar_id, P);
        int nfalse = 0;
#pragma unroll
        for (int w = 0; w < P / 32; ++w) nfalse += slot[w];
        const int f = nfalse - 1;  // last probe with !P
        const uint64_t nlo = f >= 0 ? lo + 1 + ((width - 1) * uint64_t(f)) / uint64_t(P - 1) : lo;
        const uint64_t nhi =
            f + 1 < P ? lo + 1 + ((width - 1) * uint64_t(f + 1)) / uint64_t(P - 1) - 1 : hi;
        lo = nlo;
        hi = nhi;
        ++round;
    }
    return lo;
}

// ------------------------------------------------------------ the kernel

struct stream_args {
    const void* a;
    const uint32_t* av;
    uint64_t m;
    const void* b;
    const uint32_t* bv;
    uint64_t n;
    void* out;
    uint32_t* outv;
    uint64_t ntiles;
    unsigned long long* trace;  // optional per-CTA phase timestamps (ns), 8 per CTA
    int search_mode;            // unused (kept for layout)
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <typename K, bool HAS_V>
__global__ void __launch_bounds__(stream_layout<K, HAS_V>::kThreads, 2)
    merge_stream_kernel(const stream_args args) {
    using L = stream_layout<K, HAS_V>;
    constexpr int NC = L::kConsumers;
    constexpr int VT = L::VT;
    constexpr int T = L::T;
    constexpr int CH = L::CH;
    constexpr int NS = L::NS;
    constexpr int RING = L::RING;
    auto wrap = [](uint32_t x) { return x >= uint32_t(RING) ? x - uint32_t(RING) : x; };
    constexpr int VECE = L::VECE;

    extern __shared__ __align__(128) unsigned char smem[];
    K* ringA = reinterpret_cast<K*>(smem + L::oRingA);
    K* ringB = reinterpret_cast<K*>(smem + L::oRingB);
    uint32_t* ringAV = reinterpret_cast<uint32_t*>(smem + L::oRingAV);
    uint32_t* ringBV = reinterpret_cast<uint32_t*>(smem + L::oRingBV);
    uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + L::oBars);
    uint64_t* fullB = fullA + NS;
    uint64_t* emptyA = fullB + NS;
    uint64_t* emptyB = emptyA + NS;
    uint64_t* misc64 = reinterpret_cast<uint64_t*>(smem + L::oMisc);   // [0] j_begin [1] j_end
    volatile int* misc32 = reinterpret_cast<volatile int*>(misc64 + 4);  // search slots, used

    const K* __restrict__ a = static_cast<const K*>(args.a);
    const K* __restrict__ b = static_cast<const K*>(args.b);
    const uint64_t m = args.m, n = args.n, total = m + n;
    const int tid = threadIdx.x;
    const int warp = tid >> 5;

    // this worker's output block (partition_output over tiles)
    const uint64_t G = gridDim.x, c = blockIdx.x;
    const uint64_t t0 = (c * args.ntiles) / G, t1 = ((c + 1) * args.ntiles) / G;
    const uint64_t o_begin = t0 * T;
    const uint64_t o_end = t1 * T < total ? t1 * T : total;

    if (args.trace && tid == 0) args.trace[8 * blockIdx.x + 0] = globaltimer_ns();
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&fullA[s], 1);
            mbar_init(&fullB[s], 1);
            mbar_init(&emptyA[s], 1);
            mbar_init(&emptyB[s], 1);
        }
        mbar_fence_init();
    }
    // co-rank both ends of the block: warps 0-3 start, warps 4-7 end
    if (warp < 8) {
        const int g = warp >> 2;
        const uint64_t i = g == 0 ? o_begin : o_end;
        const uint64_t j = group_co_rank<K, 128>(i, a, m, b, n, tid & 127, 1 + g, misc32 + 8 * g);
        if ((tid & 127) == 0) misc64[g] = j;
    }
    __syncthreads();
    if (args.trace && tid == 0) args.trace[8 * blockIdx.x + 1] = globaltimer_ns();
    const uint64_t j_begin = misc64[0], j_end = misc64[1];
    const uint64_t k_begin = o_begin - j_begin, k_end = o_end - j_end;

    // chunk q of an input covers absolute elements [q*CH, (q+1)*CH); relative
    // chunk r = q - q0 lives in slot r % NS, so element e sits at ring
    // position (e - q0*CH) % RING.
    const uint64_t qa0 = j_begin / CH, qb0 = k_begin / CH;
    const uint64_t na = j_end > j_begin ? (j_end - 1) / CH + 1 - qa0 : 0;
    const uint64_t nb = k_end > k_begin ? (k_end - 1) / CH + 1 - qb0 : 0;

    if (warp == 8) {
        // ------------------------------------------------------- producer
        if ((tid & 31) != 0) return;
        const uint64_t policy = policy_evict_first();
        uint64_t ia = 0, ib = 0;
        // issue chunk r (relative) of one input
        auto issue = [&](const K* src, const uint32_t* srcv, uint64_t len, uint64_t lo_limit,
                         uint64_t hi_limit, uint64_t q0, uint64_t r, K* ring, uint32_t* ringv,
                         uint64_t* full) {
            const uint64_t q = q0 + r;
            uint64_t lo = q * CH;
            const uint64_t lo_al = lo_limit & ~uint64_t(VECE - 1);
            if (lo < lo_al) lo = lo_al;
            uint64_t hi = (q + 1) * CH;
            if (hi > hi_limit) hi = hi_limit;
            // 16-byte aligned body for TMA; a scalar tail only at the array end
            uint64_t hi_v = (hi + VECE - 1) & ~uint64_t(VECE - 1);
            const uint64_t len_v = len & ~uint64_t(VECE - 1);
            if (hi_v > len) hi_v = len_v > lo ? len_v : lo;
            // payloads: their own 16-byte (4-element) alignment
            uint64_t lo_v = q * CH;
            if (lo_v < (lo_limit & ~uint64_t(3))) lo_v = lo_limit & ~uint64_t(3);
            uint64_t hi_vv = (hi + 3) & ~uint64_t(3);
            const uint64_t len_vv = len & ~uint64_t(3);
            if (hi_vv > len) hi_vv = len_vv > lo_v ? len_vv : lo_v;
            const int slot = int(r % NS);
            const uint64_t base = q * CH;                 // first element of chunk r
            K* const dst = ring + size_t(slot) * CH;      // chunk r's slot
            uint32_t* const dstv = ringv + size_t(slot) * CH;
            for (uint64_t e = hi_v; e < hi; ++e) dst[e - base] = src[e];
            if (HAS_V)
                for (uint64_t e = hi_vv; e < hi; ++e) dstv[e - base] = srcv[e];
            const uint32_t kb = uint32_t((hi_v - lo) * sizeof(K));
            const uint32_t vb = HAS_V ? uint32_t((hi_vv - lo_v) * 4) : 0;
            mbar_arrive_expect_tx(&full[slot], kb + vb);
            if (kb) tma_load_1d(dst + (lo - base), src + lo, kb, &full[slot], policy);
            if (HAS_V && vb)
                tma_load_1d(dstv + (lo_v - base), srcv + lo_v, vb, &full[slot], policy);
        };
        while (ia < na || ib < nb) {
            bool progressed = false;
            if (ia < na && (ia < NS || mbar_test(&emptyA[ia % NS], uint32_t((ia / NS - 1) & 1)))) {
                issue(a, args.av, m, j_begin, j_end, qa0, ia, ringA, ringAV, fullA);
                ++ia;
                progressed = true;
            }
            if (ib < nb && (ib < NS || mbar_test(&emptyB[ib % NS], uint32_t((ib / NS - 1) & 1)))) {
                issue(b, args.bv, n, k_begin, k_end, qb0, ib, ringB, ringBV, fullB);
                ++ib;
                progressed = true;
            }
            if (!progressed) __nanosleep(64);
        }
        return;
    }

    // ----------------------------------------------------------- consumers
    K* const sk = reinterpret_cast<K*>(smem + L::oStage);
    uint32_t* const sv = reinterpret_cast<uint32_t*>(smem + L::oStage + L::kStageKeys);
    K* __restrict__ out = static_cast<K*>(args.out);
    uint32_t* __restrict__ outv = args.outv;
    volatile int* used = misc32 + 16;

    uint64_t a_pos = j_begin, b_pos = k_begin, o = o_begin;
    uint64_t ready_a = 0, ready_b = 0;  // chunks known complete (relative)
    uint64_t rel_a = 0, rel_b = 0;      // chunks released (relative)
    uint32_t a_base = uint32_t((a_pos - qa0 * CH) % RING);
    uint32_t b_base = uint32_t((b_pos - qb0 * CH) % RING);
    int s = 0;
    while (o < o_end) {
        const int len = int(o_end - o < uint64_t(T) ? o_end - o : uint64_t(T));
        const int a_cnt = int(j_end - a_pos < uint64_t(len) ? j_end - a_pos : uint64_t(len));
        const int b_cnt = int(k_end - b_pos < uint64_t(len) ? k_end - b_pos : uint64_t(len));
        // wait for the chunks that cover this tile's windows
        if (a_cnt > 0) {
            const uint64_t need = (a_pos + a_cnt - 1) / CH - qa0 + 1;
            for (; ready_a < need; ++ready_a)
                mbar_wait(&fullA[ready_a % NS], uint32_t((ready_a / NS) & 1));
        }
        if (b_cnt > 0) {
            const uint64_t need = (b_pos + b_cnt - 1) / CH - qb0 + 1;
            for (; ready_b < need; ++ready_b)
                mbar_wait(&fullB[ready_b % NS], uint32_t((ready_b / NS) & 1));
        }
#define RA(x) ringA[wrap(a_base + uint32_t(x))]
#define RB(x) ringB[wrap(b_base + uint32_t(x))]
        const int diag = min(tid * VT, len);
        // co-rank of the diagonal inside the tile (Lemma-1 split)
        int lo = diag > b_cnt ? diag - b_cnt : 0;
        int hi = diag < a_cnt ? diag : a_cnt;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (RB(diag - mid) < RA(mid - 1))
                hi = mid - 1;
            else
                lo = mid;
        }
        int ia = lo, ib = diag - lo;
        K ka = RA(ia), kb = RB(ib);
        K keys[VT];
        uint32_t src[VT];
        const int cnt = len - diag < VT ? len - diag : VT;
#pragma unroll
        for (int v = 0; v < VT; ++v) {
            if (v < cnt) {
                const bool take_b = ib < b_cnt && (ia >= a_cnt || kb < ka);
                keys[v] = take_b ? kb : ka;
                if constexpr (HAS_V)
                    src[v] = take_b ? (wrap(b_base + uint32_t(ib)) | 0x80000000u)
                                    : wrap(a_base + uint32_t(ia));
                if (take_b) {
                    ++ib;
                    kb = RB(ib);
                } else {
                    ++ia;
                    ka = RA(ia);
                }
            }
        }
#undef RA
#undef RB
        if constexpr (HAS_V) {
#pragma unroll
            for (int v = 0; v < VT; ++v)
                if (v < cnt)
                    src[v] = (src[v] & 0x80000000u) ? ringBV[src[v] & 0x7fffffffu] : ringAV[src[v]];
        }
        if (tid == NC - 1) {
            used[0] = ia;
            used[1] = ib;
        }
        if (tid == 0) tma_store_wait_read<0>();  // previous tile's store has read the stage
        named_bar_sync(1, NC);                     // ring reads done, `used` visible
        const int used_a = used[0], used_b = used[1];
#pragma unroll
        for (int v = 0; v < VT; ++v)
            if (v < cnt) {
                sk[tid * VT + v] = keys[v];
                if constexpr (HAS_V) sv[tid * VT + v] = src[v];
            }
        fence_proxy_async_smem();
        named_bar_sync(1, NC);
        a_pos += used_a;
        b_pos += used_b;
        a_base = wrap(a_base + uint32_t(used_a));
        b_base = wrap(b_base + uint32_t(used_b));
        if (tid == 0) {
            // release chunks the merge front has passed
            while (rel_a < ready_a && (qa0 + rel_a + 1) * CH <= a_pos) {
                mbar_arrive(&emptyA[rel_a % NS]);
                ++rel_a;
            }
            while (rel_b < ready_b && (qb0 + rel_b + 1) * CH <= b_pos) {
                mbar_arrive(&emptyB[rel_b % NS]);
                ++rel_b;
            }
            // tile store: 16-byte body by TMA, a scalar tail at the very end
            const uint32_t kb_bytes = uint32_t(len * sizeof(K)) & ~15u;
            if (kb_bytes) tma_store_1d(out + o, sk, kb_bytes);
            for (int x = kb_bytes / sizeof(K); x < len; ++x) out[o + x] = sk[x];
            if constexpr (HAS_V) {
                const uint32_t vb_bytes = uint32_t(len * 4) & ~15u;
                if (vb_bytes) tma_store_1d(outv + o, sv, vb_bytes);
                for (int x = vb_bytes / 4; x < len; ++x) outv[o + x] = sv[x];
            }
            tma_store_commit();
        }
        if (args.trace && tid == 0 && s == 0) args.trace[8 * blockIdx.x + 2] = globaltimer_ns();
        o += len;
        ++s;
    }
    if (tid == 0) tma_store_wait_all();
    if (args.trace && tid == 0) args.trace[8 * blockIdx.x + 3] = globaltimer_ns();
}

}  // namespace comerge_b200
