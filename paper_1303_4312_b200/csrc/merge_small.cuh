// merge_small.cuh -- one-wave merge for small inputs (latency-bound sizes,
// e.g. BASELINE C1: 2^20 + 2^20 int32, 16.8 MB).
//
// Algorithm 2 of arXiv 1303.4312 (parallel.hpp:201-207)
// with one CTA per output tile and the whole merge in one wave, written for
// the shortest dependent chain instead of sustained streaming (the persistent
// pipeline's warp-specialised hand-offs, sleeps and dynamic tail are pure
// latency when every CTA owns one tile):
//
//   1. thread 0 pulls this CTA's share of A and B into L2 (bulk prefetch), so
//      the later co-rank rounds and window loads mostly hit L2;
//   2. both tile boundaries are co-ranked at once, each by 4 warps as one
//      129-ary search of the Lemma-1 predicate (guard 1 of corank.hpp:93-94)
//      whose per-round vote is a single `bar.red.popc` over the 128 threads,
//      stopped once the bracket is <= 64 wide: 2 dependent rounds for a
//      2^20-element diagonal (a one-warp 33-ary search to the end needs 4-5);
//   3. one TMA load per input of the SUPERSET windows the brackets allow; the
//      tile is a fixed output range of their merge (see the kernel), so the
//      searches' last round is the threads' own splits in shared memory, then
//      the serial merge of merge_serial.cuh (ties to A, merge.hpp:22-31) and
//      one bulk store (byte-space windows and stores: any alignment).
#pragma once

#include <cstdint>

#include "merge_pipe.cuh"

namespace comerge_b200 {

struct small_args {
    const void* a;
    const uint32_t* av;
    uint64_t m;
    const void* b;
    const uint32_t* bv;
    uint64_t n;
    void* out;
    uint32_t* outv;
    uint32_t prefetch;           // pull this CTA's share of the inputs into L2 at start
    uint32_t stop;               // co-rank brackets this wide are finished in shared memory
    unsigned long long* trace;   // optional per-CTA timestamps (8 x u64 per CTA)
};

template <typename K, bool HAS_V>
struct small_layout {
    using L = pipe_layout<K, HAS_V>;
    static constexpr int kThreads = 256;
    static constexpr int VT = L::VT;
    static constexpr int T = kThreads * VT;
    // the windows are supersets: each boundary's bracket is left up to kStop
    // wide by the global search and finished by the threads' own splits
    static constexpr int kStop = 64;
    static constexpr size_t kKeys = L::kStageKeys + (2 * kStop * sizeof(K) + 127) / 128 * 128;
    static constexpr size_t kVals = HAS_V ? L::kStageVals + (2 * kStop * 4 + 127) / 128 * 128 : 0;
    static constexpr size_t oBar = kKeys + kVals;
    static constexpr size_t kSmem = oBar + 64;
    static_assert(L::kConsumers == kThreads, "one thread per pipeline consumer slot");
};

// 129-ary search by the 128 threads of named barrier `bar` for the largest q in
// [lo, hi] with !pred(q) (pred monotone, !pred(lo)); every thread of the group
// ends with the same lo.
template <typename Pred>
__device__ __forceinline__ void group128_search(uint64_t& lo, uint64_t& hi, int r, int bar,
                                                uint64_t stop, Pred pred) {
    constexpr uint64_t G = 128;
    while (hi - lo > stop) {
        const uint64_t width = hi - lo;
        const uint64_t q = lo + ((uint64_t(r) + 1) * width + G) / (G + 1);  // in (lo, hi]
        const uint32_t notfar = pred(q) ? 0u : 1u;
        uint32_t cnt;
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.u32 p, %1, 0;\n bar.red.popc.u32 %0, %2, %3, p;\n}\n"
            : "=r"(cnt)
            : "r"(notfar), "r"(bar), "r"(128)
            : "memory");
        const int f = int(cnt) - 1;
        const uint64_t nlo = f >= 0 ? lo + ((uint64_t(f) + 1) * width + G) / (G + 1) : lo;
        const uint64_t nhi = uint64_t(f + 1) < G ? lo + ((uint64_t(f) + 2) * width + G) / (G + 1) - 1 : hi;
        lo = nlo;
        hi = nhi;
    }
}

template <typename K, bool HAS_V>
__global__ void __launch_bounds__(256, 2) merge_small_kernel(const small_args args) {
    using SL = small_layout<K, HAS_V>;
    constexpr int VT = SL::VT;
    constexpr uint64_t T = uint64_t(SL::T);
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* sk = smem;
    unsigned char* svb = smem + SL::kKeys;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + SL::oBar);
    uint64_t* sh = bar + 1;  // [0] j0, [1] j1, [2] a_first, [3] b_base | b_first << 32, [4..5] payload

    const K* __restrict__ a = static_cast<const K*>(args.a);
    const K* __restrict__ b = static_cast<const K*>(args.b);
    const uint64_t m = args.m, n = args.n, total = m + n;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t G = gridDim.x, c = blockIdx.x;
    const uint64_t i0 = uint64_t(c) * T, i1 = i0 + T < total ? i0 + T : total;

    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
        if (args.prefetch) {  // this CTA's share of each input into L2
            auto pull = [&](const void* base, uint64_t len, uint32_t esz) {
                const uint64_t x0 = len * c / G, x1 = len * (c + 1) / G;
                const uintptr_t B = reinterpret_cast<uintptr_t>(base);
                uintptr_t b0 = (B + x0 * esz) & ~uintptr_t(15), b1 = (B + x1 * esz) & ~uintptr_t(15);
                while (b1 > b0) {
                    const uintptr_t ch = b1 - b0 < (uintptr_t(1) << 20) ? b1 - b0 : (uintptr_t(1) << 20);
                    prefetch_l2(reinterpret_cast<const void*>(b0), uint32_t(ch));
                    b0 += ch;
                }
            };
            if (m) pull(args.a, m, sizeof(K));
            if (n) pull(args.b, n, sizeof(K));
            if (HAS_V && m) pull(args.av, m, 4);
            if (HAS_V && n) pull(args.bv, n, 4);
        }
    }
    if (args.trace && tid == 0) args.trace[8 * c] = globaltimer_ns();
    // both boundaries at once: warps 0-3 co-rank i0, warps 4-7 co-rank i1,
    // each down to a bracket [lo, hi] at most `stop` wide
    {
        const int grp = warp >> 2, r = tid & 127;
        const uint64_t i = grp ? i1 : i0;
        uint64_t lo = i > n ? i - n : 0, hi = i < m ? i : m;
        group128_search(lo, hi, r, 1 + grp, args.stop, [&](uint64_t q) {
            return probe_elem(b + (i - q)) < probe_elem(a + (q - 1));
        });
        if (r == 0) {
            sh[2 * grp] = lo;
            sh[2 * grp + 1] = hi;
        }
    }
    __syncthreads();
    if (args.trace && tid == 0) args.trace[8 * c + 1] = globaltimer_ns();
    // Superset windows A[lo0, hi1), B[i0 - hi0, i1 - lo1): in their stable
    // merge the elements before global rank i0 are exactly A[lo0, j0) and
    // B[i0 - hi0, k0) -- (j0 - lo0) + (hi0 - j0) = hi0 - lo0 of them whatever
    // j0 is -- so the tile is output ranks [hi0 - lo0, + (i1 - i0)) of that
    // merge (every pair's relative order is fixed by its keys and sources
    // alone), and the last round of each search becomes the threads' splits.
    const uint64_t lo0 = sh[0], hi0 = sh[1], lo1 = sh[2], hi1 = sh[3];
    const uint64_t j0 = lo0, j1 = hi1, k0 = i0 - hi0, k1 = i1 - lo1;
    const int a_len = int(j1 - j0), b_len = int(k1 - k0);
    const int base = int(hi0 - lo0), len = int(i1 - i0);
    __syncthreads();
    if (tid == 0) {
        const win_plan pa = plan_window(a, m, sizeof(K), j0, j1, sk);
        const win_plan pb = plan_window(b, n, sizeof(K), k0, k1, sk + pa.span);
        uint32_t bytes = pa.bytes + pb.bytes;
        win_plan pav{}, pbv{};
        if constexpr (HAS_V) {
            pav = plan_window(args.av, m, 4, j0, j1, svb);
            pbv = plan_window(args.bv, n, 4, k0, k1, svb + pav.span);
            bytes += pav.bytes + pbv.bytes;
        }
        const uint64_t policy = policy_evict_first();
        mbar_arrive_expect_tx(bar, bytes);
        if (pa.bytes) tma_load_1d(sk + pa.dst_off, pa.src, pa.bytes, bar, policy);
        if (pb.bytes) tma_load_1d(sk + pa.span + pb.dst_off, pb.src, pb.bytes, bar, policy);
        if constexpr (HAS_V) {
            if (pav.bytes) tma_load_1d(svb + pav.dst_off, pav.src, pav.bytes, bar, policy);
            if (pbv.bytes) tma_load_1d(svb + pav.span + pbv.dst_off, pbv.src, pbv.bytes, bar, policy);
            sh[4] = pav.first | (uint64_t(pav.span) << 16) | (uint64_t(pbv.first) << 48);
        }
        sh[2] = pa.first;
        sh[3] = pa.span | (uint64_t(pb.first) << 32);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    if (args.trace && tid == 0) args.trace[8 * c + 2] = globaltimer_ns();
    const K* sA = reinterpret_cast<const K*>(sk + sh[2]);
    const K* sB = reinterpret_cast<const K*>(sk + (sh[3] & 0xffffffffu) + (sh[3] >> 32));
    const int diag = min(tid * VT, len);
    K keys[VT];
    uint32_t src[VT];
    merge_thread_lean<K, VT, HAS_V>(sA, a_len, sB, b_len, base + diag, keys, src);
    if constexpr (HAS_V) {  // source element address -> its payload
        const uint64_t pv = sh[4];
        const uint32_t* sav = reinterpret_cast<const uint32_t*>(svb + (pv & 0xffff));
        const uint32_t* sbv = reinterpret_cast<const uint32_t*>(svb + ((pv >> 16) & 0xffffffffu) +
                                                                (pv >> 48));
        const uint32_t aA = smem_addr(sA), aB = smem_addr(sB);
        constexpr int SH = sizeof(K) == 8 ? 3 : 2;
#pragma unroll
        for (int v = 0; v < VT; ++v)
            if (diag + v < len) {
                const bool isb = src[v] >= aB;
                const int x = int((src[v] - (isb ? aB : aA)) >> SH);
                src[v] = isb ? sbv[x] : sav[x];
            }
    }
    __syncthreads();  // windows consumed: the tile goes back into the same buffers
    const uint32_t o_shift =
        uint32_t((reinterpret_cast<uintptr_t>(args.out) + i0 * sizeof(K)) & 15u);
    const uint32_t ov_shift =
        HAS_V ? uint32_t((reinterpret_cast<uintptr_t>(args.outv) + i0 * 4) & 15u) : 0u;
    const int cnt = len - diag < VT ? len - diag : VT;
    const uint32_t ko = smem_addr(sk) + o_shift + uint32_t(tid * VT) * uint32_t(sizeof(K));
    const uint32_t vo = smem_addr(svb) + ov_shift + uint32_t(tid * VT) * 4u;
#pragma unroll
    for (int v = 0; v < VT; ++v)
        if (v < cnt) {
            smem_io<K>::st(ko + uint32_t(v) * uint32_t(sizeof(K)), keys[v]);
            if constexpr (HAS_V) smem_io<uint32_t>::st(vo + uint32_t(v) * 4u, src[v]);
        }
    fence_proxy_async_smem();
    __syncthreads();
    if (tid == 0) {
        if (args.trace) args.trace[8 * c + 3] = globaltimer_ns();
        const uint64_t spolicy = policy_evict_first();
        store_window(args.out, i0, len, uint32_t(sizeof(K)), sk, false, spolicy);
        if constexpr (HAS_V) store_window(args.outv, i0, len, 4u, svb, false, spolicy);
        tma_store_commit();
        tma_store_wait_all();
        if (args.trace) args.trace[8 * c + 4] = globaltimer_ns();
    }
}

}  // namespace comerge_b200
