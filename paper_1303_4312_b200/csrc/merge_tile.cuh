// merge_tile.cuh -- tile-parallel stable merge for sm_100a (v1 path).
//
// Mapping of the reference's Algorithm 2 (parallel.hpp:180-282) onto the GPU:
//
//   reference worker r, block [i_r, i_{r+1})      ->  CTA t, tile [t*T, (t+1)*T)
//   co_rank(i_r), co_rank(i_{r+1})  (:204-205)     ->  partition_kernel: one
//        thread per tile boundary, co_rank_split against HBM, written once
//        (the synced variant's "one co-rank per worker", :209-219)
//   merge_into(a-window, b-window) (:194-199)      ->  merge_tile_kernel:
//        windows staged in shared memory with 128-bit loads, each thread
//        co-ranks its own VT-slot diagonal inside the tile (the same
//        Lemma-1 split, now over shared memory) and runs a branch-free
//        serial merge of VT elements in registers (merge.hpp:22-31: take b
//        only when b < a), then the tile is written back with 128-bit
//        coalesced stores from a shared-memory staging buffer.
//
// Tiles are all T elements except the last, so blocks differ by at most T
// (Proposition 2 up to the tile granularity) and the output is independent of
// any worker count (acceptance criterion 6).
#pragma once

#include <cstdint>

#include "corank.cuh"
#include "records.cuh"

namespace comerge_b200 {

template <typename K>
struct tile_cfg {
    static constexpr int kThreads = 256;
    // VT odd: per-thread staging rows (stride VT) hit distinct banks.
    static constexpr int kVT = sizeof(K) == 8 ? 11 : 15;
    static constexpr int kTile = kThreads * kVT;
};

enum tile_flags : int {
    kAAligned = 1,
    kBAligned = 2,
    kOutAligned = 4,
    kAVAligned = 8,
    kBVAligned = 16,
    kOutVAligned = 32,
};

__device__ __forceinline__ uint4 ld_vec_nc(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_vec_na(void* p, uint4 v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

template <typename T>
__device__ __forceinline__ T ldg_elem(const T* p) {
    if constexpr (is_rec<T>::value) {  // records compare by key: load the key only
        T r{};
        r.key = ldg_elem(&p->key);
        return r;
    } else if constexpr (sizeof(T) == 8)
        return static_cast<T>(__ldg(reinterpret_cast<const unsigned long long*>(p)));
    else
        return __ldg(p);
}

// A co-rank probe: one scattered element, cached in L2 only.  (Through the
// read-only L1 path every probe fetched a whole 128-byte line -- ncu: L2
// requests of C4 exceeded the window bytes by 3.5 sectors per probe.)
// Records (records.cuh) probe their key only.
template <typename T>
__device__ __forceinline__ typename key_of<T>::type probe_elem(const T* p) {
    if constexpr (is_rec<T>::value)
        return probe_elem(&p->key);
    else if constexpr (sizeof(T) == 8)
        return static_cast<T>(__ldcg(reinterpret_cast<const unsigned long long*>(p)));
    else
        return __ldcg(p);
}

// Stage src[lo, hi) into shared memory: element x lands at
// dst[x - (lo & ~(VEC-1))], so 16-byte vectors of src map onto 16-byte
// aligned shared-memory slots.  Vectors that straddle the array end (or any
// element when src itself is not 16-byte aligned) fall back to scalar loads.
template <typename T, int THREADS>
__device__ __forceinline__ void load_window(const T* __restrict__ src, uint64_t src_len,
                                            uint64_t lo, uint64_t hi, T* dst, bool aligned) {
    constexpr int VEC = 16 / sizeof(T);
    if (hi <= lo) return;
    const uint64_t alo = lo & ~uint64_t(VEC - 1);
    const int nvec = static_cast<int>((hi - alo + VEC - 1) / VEC);
    for (int q = threadIdx.x; q < nvec; q += THREADS) {
        const uint64_t x0 = alo + uint64_t(q) * VEC;
        if (aligned && x0 + VEC <= src_len) {
            *reinterpret_cast<uint4*>(dst + q * VEC) = ld_vec_nc(src + x0);
        } else {
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
                const uint64_t x = x0 + e;
                if (x >= lo && x < hi) dst[q * VEC + e] = ldg_elem(src + x);
            }
        }
    }
}

// out[0, len) <- staged[0, len); `out` is 16-byte aligned when `aligned`.
template <typename T, int THREADS>
__device__ __forceinline__ void store_tile(T* __restrict__ out, const T* staged, int len,
                                           bool aligned) {
    constexpr int VEC = 16 / sizeof(T);
    if (aligned) {
        const int nfull = len / VEC;
        for (int q = threadIdx.x; q < nfull; q += THREADS)
            st_vec_na(out + q * VEC, *reinterpret_cast<const uint4*>(staged + q * VEC));
        for (int x = nfull * VEC + threadIdx.x; x < len; x += THREADS) out[x] = staged[x];
    } else {
        for (int x = threadIdx.x; x < len; x += THREADS) out[x] = staged[x];
    }
}

// Per-thread merge of VT outputs starting at diagonal `diag` of the tile
// formed by sA[0, a_len) and sB[0, b_len) (shared memory).  Ties take A
// (merge.hpp:23-26).  src[v] = index into sA, or index into sB | 1<<31.
template <typename KC, int VT, bool TRACK>
__device__ __forceinline__ void merge_thread(const KC* sA, int a_len, const KC* sB, int b_len,
                                             int diag, KC (&keys)[VT], uint32_t (&src)[VT]) {
    const int ia0 = co_rank_split<KC, int>(diag, sA, a_len, sB, b_len,
                                           [](const KC* p) { return *p; });
    int ia = ia0, ib = diag - ia0;
    // one-element look-ahead on both sides: the shared-memory load for the
    // next step is already in flight, so each step waits on compare/select
    // only (reads may touch the window slack past a_len / b_len, never used)
    KC ka = sA[ia], kb = sB[ib];
    KC ka1 = sA[ia + 1], kb1 = sB[ib + 1];
#pragma unroll
    for (int v = 0; v < VT; ++v) {
        const bool take_b = ib < b_len && (ia >= a_len || kb < ka);
        keys[v] = take_b ? kb : ka;
        if constexpr (TRACK) src[v] = take_b ? (uint32_t(ib) | 0x80000000u) : uint32_t(ia);
        if (take_b) {
            ++ib;
            kb = kb1;
            kb1 = sB[ib + 1];
        } else {
            ++ia;
            ka = ka1;
            ka1 = sA[ia + 1];
        }
    }
}

// ---------------------------------------------------------------- kernels

// bj[t] = co-rank (A prefix length) of output rank min(t*tile, m+n).
template <typename K>
__global__ void partition_kernel(const K* __restrict__ a, uint64_t m, const K* __restrict__ b,
                                 uint64_t n, uint64_t tile, uint64_t nbound,
                                 uint64_t* __restrict__ bj) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nbound) return;
    const uint64_t total = m + n;
    const uint64_t i = t * tile < total ? t * tile : total;
    bj[t] = co_rank_split<K, uint64_t>(i, a, m, b, n, [](const K* p) { return ldg_elem(p); });
}

// One CTA per output tile.
template <typename K, bool HAS_V>
__global__ void __launch_bounds__(tile_cfg<K>::kThreads)
    merge_tile_kernel(const K* __restrict__ a, const uint32_t* __restrict__ av, uint64_t m,
                      const K* __restrict__ b, const uint32_t* __restrict__ bv, uint64_t n,
                      K* __restrict__ out, uint32_t* __restrict__ outv,
                      const uint64_t* __restrict__ bj, int flags) {
    constexpr int THREADS = tile_cfg<K>::kThreads;
    constexpr int VT = tile_cfg<K>::kVT;
    constexpr int T = tile_cfg<K>::kTile;
    constexpr int VEC = 16 / sizeof(K);
    constexpr int WIN = ((T + 4 * VEC + VT + 3) + VEC - 1) / VEC * VEC;
    constexpr int WINV = HAS_V ? ((T + 16 + VT + 2) + 3) / 4 * 4 : 4;
    __shared__ __align__(16) K s_keys[WIN];
    __shared__ __align__(16) uint32_t s_vals[WINV];

    const uint64_t t = blockIdx.x;
    const uint64_t total = m + n;
    const uint64_t i0 = t * T;
    const uint64_t i1 = i0 + T < total ? i0 + T : total;
    const uint64_t j0 = bj[t], j1 = bj[t + 1];
    const uint64_t k0 = i0 - j0, k1 = i1 - j1;
    const int a_len = int(j1 - j0), b_len = int(k1 - k0);
    const int len = a_len + b_len;

    const int a_off = int(j0 & (VEC - 1));
    const int b_base = (a_off + a_len + VEC - 1) / VEC * VEC;
    const int b_off = int(k0 & (VEC - 1));
    load_window<K, THREADS>(a, m, j0, j1, s_keys, flags & kAAligned);
    load_window<K, THREADS>(b, n, k0, k1, s_keys + b_base, flags & kBAligned);
    int av_off = 0, bv_base = 0, bv_off = 0;
    if constexpr (HAS_V) {
        av_off = int(j0 & 3);
        bv_base = (av_off + a_len + 3) / 4 * 4;
        bv_off = int(k0 & 3);
        load_window<uint32_t, THREADS>(av, m, j0, j1, s_vals, flags & kAVAligned);
        load_window<uint32_t, THREADS>(bv, n, k0, k1, s_vals + bv_base, flags & kBVAligned);
    }
    __syncthreads();

    const int diag = min(int(threadIdx.x) * VT, len);
    K keys[VT];
    uint32_t src[VT];
    merge_thread<K, VT, HAS_V>(s_keys + a_off, a_len, s_keys + b_base + b_off, b_len, diag, keys,
                               src);
    if constexpr (HAS_V) {
        const uint32_t* sav = s_vals + av_off;
        const uint32_t* sbv = s_vals + bv_base + bv_off;
#pragma unroll
        for (int v = 0; v < VT; ++v)
            if (diag + v < len)
                src[v] = (src[v] & 0x80000000u) ? sbv[src[v] & 0x7fffffffu] : sav[src[v]];
    }
    __syncthreads();  // windows consumed; reuse them as output staging
    const int cnt = len - diag < VT ? len - diag : VT;
#pragma unroll
    for (int v = 0; v < VT; ++v)
        if (v < cnt) s_keys[threadIdx.x * VT + v] = keys[v];
    if constexpr (HAS_V) {
#pragma unroll
        for (int v = 0; v < VT; ++v)
            if (v < cnt) s_vals[threadIdx.x * VT + v] = src[v];
    }
    __syncthreads();
    store_tile<K, THREADS>(out + i0, s_keys, len, flags & kOutAligned);
    if constexpr (HAS_V) store_tile<uint32_t, THREADS>(outv + i0, s_vals, len, flags & kOutVAligned);
}

// Batched co-rank with the reference's exact search and statistics.
template <typename K>
__global__ void co_rank_batch_kernel(const uint64_t* __restrict__ ranks, uint64_t count,
                                     const K* __restrict__ a, uint64_t m, const K* __restrict__ b,
                                     uint64_t n, uint64_t* __restrict__ out_j,
                                     uint32_t* __restrict__ out_it, uint32_t* __restrict__ out_cmp) {
    const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q >= count) return;
    const uint64_t i = ranks[q];
    if (i > m + n) {
        out_j[q] = ~uint64_t(0);
        if (out_it) out_it[q] = 0;
        if (out_cmp) out_cmp[q] = 0;
        return;
    }
    corank_stats st;
    out_j[q] = co_rank_alg1(i, a, m, b, n, [](const K* p) { return ldg_elem(p); }, &st);
    if (out_it) out_it[q] = st.iterations;
    if (out_cmp) out_cmp[q] = st.comparisons;
}

// ------------------------------------------------------------- segmented
//
// The batch of independent pairs is one merge over composite keys
// (segment, key): A and B are both sorted by that composite, and its stable
// merge places pair s exactly at a_off[s] + b_off[s] with A-before-B ties.
// Tile boundaries co-rank inside their segment; inside a tile the windows
// are widened to 64-bit composites and merged with the same code path.

template <typename K>
__device__ __forceinline__ uint32_t ordered_u32(K k) {
    if constexpr (sizeof(K) == 4 && K(-1) < K(0))
        return uint32_t(k) ^ 0x80000000u;
    else
        return uint32_t(k);
}
template <typename K>
__device__ __forceinline__ K from_ordered_u32(uint32_t u) {
    if constexpr (K(-1) < K(0))
        return K(u ^ 0x80000000u);
    else
        return K(u);
}

// Largest s in [lo, hi] with off[s] <= x (off nondecreasing, off[lo] <= x).
__device__ __forceinline__ uint64_t seg_upper(const uint64_t* __restrict__ off, uint64_t lo,
                                              uint64_t hi, uint64_t x) {
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo + 1) / 2;
        if (__ldg(reinterpret_cast<const unsigned long long*>(off + mid)) <= x)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

template <typename K>
__global__ void seg_partition_kernel(const K* __restrict__ a, const uint64_t* __restrict__ a_off,
                                     const K* __restrict__ b, const uint64_t* __restrict__ b_off,
                                     uint64_t nseg, uint64_t total, uint64_t tile, uint64_t nbound,
                                     uint64_t* __restrict__ bj, uint64_t* __restrict__ bseg) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= nbound) return;
    const uint64_t i = t * tile < total ? t * tile : total;
    // largest s in [0, nseg-1] with out_off[s] = a_off[s] + b_off[s] <= i
    uint64_t lo = 0, hi = nseg - 1;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo + 1) / 2;
        if (__ldg(reinterpret_cast<const unsigned long long*>(a_off + mid)) +
                __ldg(reinterpret_cast<const unsigned long long*>(b_off + mid)) <=
            i)
            lo = mid;
        else
            hi = mid - 1;
    }
    const uint64_t s = lo;
    const uint64_t as = a_off[s], bs = b_off[s];
    const uint64_t ma = a_off[s + 1] - as, nb = b_off[s + 1] - bs;
    const uint64_t li = i - as - bs;  // <= ma + nb by construction
    const uint64_t jl = co_rank_split<K, uint64_t>(li < ma + nb ? li : ma + nb, a + as, ma, b + bs,
                                                   nb, [](const K* p) { return ldg_elem(p); });
    bj[t] = as + jl;
    bseg[t] = s;
}

template <typename K>
struct seg_cfg {
    static constexpr int kThreads = 256;
    static constexpr int kVT = 11;
    static constexpr int kTile = kThreads * kVT;
};

template <typename K>
__global__ void __launch_bounds__(seg_cfg<K>::kThreads)
    seg_merge_tile_kernel(const K* __restrict__ a, const uint64_t* __restrict__ a_seg, uint64_t m,
                          const K* __restrict__ b, const uint64_t* __restrict__ b_seg, uint64_t n,
                          K* __restrict__ out, const uint64_t* __restrict__ bj,
                          const uint64_t* __restrict__ bseg, int flags) {
    constexpr int THREADS = seg_cfg<K>::kThreads;
    constexpr int VT = seg_cfg<K>::kVT;
    constexpr int T = seg_cfg<K>::kTile;
    constexpr int VEC = 16 / sizeof(K);
    constexpr int WIN = ((T + 4 * VEC + VT + 2) + VEC - 1) / VEC * VEC;
    __shared__ __align__(16) K s_raw[WIN];
    __shared__ __align__(16) uint64_t s_comp[T + VT + 4];

    const uint64_t t = blockIdx.x;
    const uint64_t total = m + n;
    const uint64_t i0 = t * T;
    const uint64_t i1 = i0 + T < total ? i0 + T : total;
    const uint64_t j0 = bj[t], j1 = bj[t + 1];
    const uint64_t k0 = i0 - j0, k1 = i1 - j1;
    const uint64_t s0 = bseg[t], s1 = bseg[t + 1];
    const int a_len = int(j1 - j0), b_len = int(k1 - k0);
    const int len = a_len + b_len;
    const int a_off = int(j0 & (VEC - 1));
    const int b_base = (a_off + a_len + VEC - 1) / VEC * VEC;
    const int b_off = int(k0 & (VEC - 1));
    load_window<K, THREADS>(a, m, j0, j1, s_raw, flags & kAAligned);
    load_window<K, THREADS>(b, n, k0, k1, s_raw + b_base, flags & kBAligned);
    __syncthreads();
    // widen to (segment, key) composites: A part at [0, a_len), B part after
    for (int x = threadIdx.x; x < len; x += THREADS) {
        uint64_t seg;
        uint32_t u;
        if (x < a_len) {
            seg = seg_upper(a_seg, s0, s1, j0 + x);
            u = ordered_u32(s_raw[a_off + x]);
        } else {
            seg = seg_upper(b_seg, s0, s1, k0 + (x - a_len));
            u = ordered_u32(s_raw[b_base + b_off + (x - a_len)]);
        }
        s_comp[x] = (seg << 32) | u;
    }
    __syncthreads();
    const int diag = min(int(threadIdx.x) * VT, len);
    uint64_t keys[VT];
    uint32_t src[VT];
    merge_thread<uint64_t, VT, false>(s_comp, a_len, s_comp + a_len, b_len, diag, keys, src);
    __syncthreads();
    const int cnt = len - diag < VT ? len - diag : VT;
#pragma unroll
    for (int v = 0; v < VT; ++v)
        if (v < cnt) s_raw[threadIdx.x * VT + v] = from_ordered_u32<K>(uint32_t(keys[v]));
    __syncthreads();
    store_tile<K, THREADS>(out + i0, s_raw, len, flags & kOutAligned);
}

}  // namespace comerge_b200
