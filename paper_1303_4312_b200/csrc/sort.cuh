// sort.cuh -- stable merge sort built on the merge path (SURVEY.md §8f row 1:
// "GPU merge sort built on the segmented kernel").
//
//   1. block_sort_kernel: every CTA sorts one run of R = NT*VT elements in
//      shared memory -- VT elements per thread by a sorting network in
//      registers (keys only; the key-value variant uses odd-even
//      transposition, swapping only on strictly-less, so equal keys keep
//      their order), then log2(NT) rounds of pairwise merges of the sorted lists,
//      each thread taking VT outputs at its merge-path split (the Lemma-1
//      split of corank.hpp:93-94, ties to the left list as merge.hpp:22-31).
//   2. log2(n/R) merge passes of the tile pipeline in merge-pass mode
//      (merge_pipe.cuh, pipe_args::run_len): pass p merges runs 2s and 2s+1
//      of length R*2^p as one segmented batch with implicit offsets.
//
// The result equals a stable sort (std::stable_sort) of the keys: bottom-up
// merging of adjacent runs with left-first ties preserves input order.
#pragma once

#include <cstdint>
#include <limits>

#include "corank.cuh"
#include "ptx.cuh"

namespace comerge_b200 {

template <typename K>
struct sort_cfg {
    static constexpr int NT = 512;
    static constexpr int VT = sizeof(K) == 8 ? 8 : 16;
    static constexpr int R = NT * VT;  // base run (a power of two)
};

// Batcher's odd-even merge sort network over the VT registers of a thread
// (keys only: equal keys are indistinguishable, so the network need not be
// stable): 63 compare-exchanges for 16 keys, 19 for 8, against 120 / 28 for
// odd-even transposition; min / max of 32-bit keys are one instruction each.
template <typename K, int VT>
__device__ __forceinline__ void network_sort(K (&k)[VT]) {
#pragma unroll
    for (int p = 1; p < VT; p <<= 1)
#pragma unroll
        for (int q = p; q >= 1; q >>= 1)
#pragma unroll
            for (int j = q % p; j + q < VT; j += 2 * q)
#pragma unroll
                for (int i = 0; i < q && i + j + q < VT; ++i)
                    if ((i + j) / (2 * p) == (i + j + q) / (2 * p)) {
                        const K x = k[i + j], y = k[i + j + q];
                        k[i + j] = y < x ? y : x;
                        k[i + j + q] = y < x ? x : y;
                    }
}

// Shared-memory index with one pad word per 32 elements: thread t's VT
// consecutive elements (t*VT + v) then fall in distinct banks across a warp
// (without it VT = 16 is a 16-way bank conflict on every staging access).
__device__ __forceinline__ int spad(int i) { return i + (i >> 5); }

template <typename K>
__global__ void __launch_bounds__(sort_cfg<K>::NT)
    block_sort_kernel(const K* __restrict__ in, K* __restrict__ out, uint64_t n) {
    constexpr int NT = sort_cfg<K>::NT, VT = sort_cfg<K>::VT, R = sort_cfg<K>::R;
    // + slack: a finished list may be read one past its end (never used)
    __shared__ K s[R + R / 32 + 4];
    pdl_trigger();  // the first merge pass may be scheduled (it waits for this grid)
    const uint64_t base = uint64_t(blockIdx.x) * R;
    const int cnt = n - base < uint64_t(R) ? int(n - base) : R;
    const int t = threadIdx.x;
    // padding sorts last and, being last in input order, stays behind real maxima
    const K pad = std::numeric_limits<K>::max();
    for (int x = t; x < R; x += NT) s[spad(x)] = x < cnt ? in[base + x] : pad;
    __syncthreads();
    K k[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) k[v] = s[spad(t * VT + v)];
    network_sort<K, VT>(k);
    for (int w = VT; w < R; w *= 2) {
        __syncthreads();  // previous round's reads are done
#pragma unroll
        for (int v = 0; v < VT; ++v) s[spad(t * VT + v)] = k[v];
        __syncthreads();
        const int d = t * VT;
        const int a0 = d / (2 * w) * (2 * w), b0 = a0 + w;  // list starts
        const int diag = d - a0;
        int lo = diag > w ? diag - w : 0, hi = diag < w ? diag : w;
        while (lo < hi) {  // Lemma-1 split (ties to the left list)
            const int mid = (lo + hi + 1) >> 1;
            if (s[spad(b0 + diag - mid)] < s[spad(a0 + mid - 1)])
                hi = mid - 1;
            else
                lo = mid;
        }
        int ia = lo, ib = diag - lo;
        K ka = s[spad(a0 + ia)], kb = s[spad(b0 + ib)];
#pragma unroll
        for (int v = 0; v < VT; ++v) {  // branch-free: one shared load per output
            const bool take_b = ib < w && (ia >= w || kb < ka);
            k[v] = take_b ? kb : ka;
            ia += take_b ? 0 : 1;
            ib += take_b ? 1 : 0;
            const K nx = s[spad(take_b ? b0 + ib : a0 + ia)];
            ka = take_b ? ka : nx;
            kb = take_b ? nx : kb;
        }
    }
    __syncthreads();
#pragma unroll
    for (int v = 0; v < VT; ++v) s[spad(t * VT + v)] = k[v];
    __syncthreads();
    for (int x = t; x < cnt; x += NT) out[base + x] = s[spad(x)];
}

// Key-value variant: the uint32 payload moves with its key (VT = 8, runs of
// 4096 pairs, 2048 for 64-bit keys; keys and payloads in two padded shared
// arrays within the 48 KB static limit).
template <typename K>
struct sort_pairs_cfg {
    static constexpr int NT = sizeof(K) == 8 ? 256 : 512;
    static constexpr int VT = 8;
    static constexpr int R = NT * VT;
};

template <typename K>
__global__ void __launch_bounds__(sort_pairs_cfg<K>::NT)
    block_sort_pairs_kernel(const K* __restrict__ in, const uint32_t* __restrict__ in_v,
                            K* __restrict__ out, uint32_t* __restrict__ out_v, uint64_t n) {
    constexpr int NT = sort_pairs_cfg<K>::NT, VT = sort_pairs_cfg<K>::VT,
                  R = sort_pairs_cfg<K>::R;
    __shared__ K s[R + R / 32 + 4];
    __shared__ uint32_t sv[R + R / 32 + 4];
    pdl_trigger();
    const uint64_t base = uint64_t(blockIdx.x) * R;
    const int cnt = n - base < uint64_t(R) ? int(n - base) : R;
    const int t = threadIdx.x;
    const K pad = std::numeric_limits<K>::max();
    for (int x = t; x < R; x += NT) {
        s[spad(x)] = x < cnt ? in[base + x] : pad;
        sv[spad(x)] = x < cnt ? in_v[base + x] : 0u;
    }
    __syncthreads();
    K k[VT];
    uint32_t p[VT];
#pragma unroll
    for (int v = 0; v < VT; ++v) {
        k[v] = s[spad(t * VT + v)];
        p[v] = sv[spad(t * VT + v)];
    }
#pragma unroll
    for (int pass = 0; pass < VT; ++pass) {
#pragma unroll
        for (int v = pass & 1; v + 1 < VT; v += 2) {
            if (k[v + 1] < k[v]) {  // strict: equal keys keep their order
                const K x = k[v];
                k[v] = k[v + 1];
                k[v + 1] = x;
                const uint32_t y = p[v];
                p[v] = p[v + 1];
                p[v + 1] = y;
            }
        }
    }
    for (int w = VT; w < R; w *= 2) {
        __syncthreads();
#pragma unroll
        for (int v = 0; v < VT; ++v) {
            s[spad(t * VT + v)] = k[v];
            sv[spad(t * VT + v)] = p[v];
        }
        __syncthreads();
        const int d = t * VT;
        const int a0 = d / (2 * w) * (2 * w), b0 = a0 + w;
        const int diag = d - a0;
        int lo = diag > w ? diag - w : 0, hi = diag < w ? diag : w;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (s[spad(b0 + diag - mid)] < s[spad(a0 + mid - 1)])
                hi = mid - 1;
            else
                lo = mid;
        }
        int ia = lo, ib = diag - lo;
        K ka = s[spad(a0 + ia)], kb = s[spad(b0 + ib)];
#pragma unroll
        for (int v = 0; v < VT; ++v) {
            const bool take_b = ib < w && (ia >= w || kb < ka);
            k[v] = take_b ? kb : ka;
            p[v] = sv[spad(take_b ? b0 + ib : a0 + ia)];
            ia += take_b ? 0 : 1;
            ib += take_b ? 1 : 0;
            const K nx = s[spad(take_b ? b0 + ib : a0 + ia)];
            ka = take_b ? ka : nx;
            kb = take_b ? nx : kb;
        }
    }
    __syncthreads();
#pragma unroll
    for (int v = 0; v < VT; ++v) {
        s[spad(t * VT + v)] = k[v];
        sv[spad(t * VT + v)] = p[v];
    }
    __syncthreads();
    for (int x = t; x < cnt; x += NT) {
        out[base + x] = s[spad(x)];
        out_v[base + x] = sv[spad(x)];
    }
}

}  // namespace comerge_b200
