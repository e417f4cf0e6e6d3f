// sort.cuh -- stable merge sort built on the merge path (SURVEY.md §8f row 1:
// "GPU merge sort built on the segmented kernel").
//
//   1. block_sort_kernel: every CTA sorts one run of R elements in shared
//      memory -- VT (odd) elements per thread by a sorting network in
//      registers (the key-value variant sorts (key, position) composites,
//      so equal keys keep their order, and gathers the payloads by position
//      afterwards), then rounds of pairwise merges of the sorted lists
//      (the first five inside one warp: warp barriers only), each thread
//      taking VT outputs at its merge-path split (the Lemma-1 split of
//      corank.hpp:93-94, ties to the left list as merge.hpp:22-31) with the
//      pipeline consumers' serial merge (merge_serial.cuh).
//   2. log2(n/R) merge passes of the tile pipeline in merge-pass mode
//      (merge_pipe.cuh, pipe_args::run_len): pass p merges runs 2s and 2s+1
//      of length R*2^p as one segmented batch with implicit offsets.
//
// The result equals a stable sort (std::stable_sort) of the keys: bottom-up
// merging of adjacent runs with left-first ties preserves input order.
#pragma once

#include <cstdint>
#include <limits>
#include <type_traits>

#include "corank.cuh"
#include "merge_serial.cuh"
#include "ptx.cuh"

namespace comerge_b200 {

// elements per thread of the block sorts (odd: see sort_cfg) and base runs.
// Measured on 2^26 keys (ms; R = 8192 / 4096 / 4096 unless noted): 32-bit keys
// VT 17: 1.804, 21: 1.762, 25: 1.723, 29: 1.709, 33: 1.671, 41: 1.704, 49:
// 1.723, 65: 1.755; R = 16384 with VT 33: 1.664, VT 65: 1.626 (R = 32768:
// 1.699).  64-bit keys VT 9: 3.609, 13: 3.451, 17: 3.354, 25: 3.359, 33: 3.285;
// R = 8192 with VT 33: 3.147 (VT 17: 3.333, VT 65: 3.541).  32-bit pairs VT 9:
// 3.477, 13: 3.401, 17: 3.337, 21: 3.408, 33: 3.437; R = 8192 with VT 17:
// 3.289, VT 33: 3.267 (VT 65: 3.879).  More keys per thread amortise the split
// search of every round and leave fewer block-wide rounds (5 warp-local rounds
// + log2(warps)); a power-of-two warp count keeps the last round full.
#ifndef SORT_VT32
#define SORT_VT32 65
#endif
#ifndef SORT_VT64
#define SORT_VT64 33
#endif
#ifndef SORTP_VT
#define SORTP_VT 33
#endif
#ifndef SORTP_VT64
#define SORTP_VT64 33
#endif
// base runs (powers of two): 32-bit keys, 64-bit keys, 32-bit pairs, 64-bit pairs
#ifndef SORT_R32
#define SORT_R32 16384
#endif
#ifndef SORT_R64
#define SORT_R64 8192
#endif
#ifndef SORTP_R32
#define SORTP_R32 8192
#endif
#ifndef SORTP_R64
#define SORTP_R64 4096
#endif

// CTAs per SM the shared memory allows (227 KB, 1 KB reserved per CTA), as the
// kernels' launch bound -- the register allocation must not be what lowers the
// occupancy (64-bit keys at 86 registers fell from 3 to 2 CTAs per SM) --
// but never forcing fewer than 64 registers per thread.
constexpr int block_sort_min_blocks(size_t smem, int nt) {
    const int by_smem = int(size_t(227) * 1024 / (smem + 1024));
    const int by_regs = 1024 / nt;
    const int b = by_smem < by_regs ? by_smem : by_regs;
    return b < 1 ? 1 : b;
}

// Base runs of R elements (a power of two: the merge passes' run arithmetic
// is shifts) sorted by NA = ceil(R / VT) threads of VT elements each, VT ODD:
// thread t's elements sit at s[t*VT + v], an odd word stride, so the staging
// accesses of a warp are bank-conflict free without padding and the rounds
// can run the pipeline consumers' lean serial merge on plain shared addresses
// (merge_serial.cuh, ~12 instructions per output).  The last slots (R .. NA*VT)
// hold padding keys.
// SMALL: half the run with half the keys per thread -- twice the CTAs -- for
// inputs of fewer than one full-size run per SM (the host chooses).
template <typename K, bool SMALL = false>
struct sort_cfg {
    static constexpr int VTB = sizeof(K) == 8 ? SORT_VT64 : SORT_VT32;
    static constexpr int RB = sizeof(K) == 8 ? SORT_R64 : SORT_R32;
    static constexpr int VT = SMALL ? (VTB + 1) / 2 : VTB;
    static constexpr int R = SMALL ? RB / 2 : RB;           // base run (a power of two)
    static constexpr int NA = (R + VT - 1) / VT;            // threads holding elements
    static constexpr int NT = (NA + 31) / 32 * 32;
    static constexpr int S = NA * VT;                       // slots incl. padding
    static constexpr size_t kSmem = size_t(S + 4) * sizeof(K);  // dynamic shared memory
    static constexpr int kMinBlocks = block_sort_min_blocks(kSmem, NT);
    static_assert(NA <= NT && (R & (R - 1)) == 0 && VT % 2 == 1, "block sort shape");
};

// Batcher's odd-even merge sort network over the VT registers of a thread
// (keys only: equal keys are indistinguishable, so the network need not be
// stable; any VT: the power-of-two network with the comparators beyond VT
// dropped, checked by the 0-1 principle for 8 .. 21): 85 compare-exchanges for
// 17 keys, 221 for 33; min / max of 32-bit keys are one instruction each.
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

// Stable variant for key-value pairs: the same network over (key, position in
// the thread) composites -- distinct, so any sorting network orders them the
// stable way -- carrying only the position; the caller gathers the payloads
// by it afterwards.  32-bit keys: one 64-bit word (order-preserving key bits,
// then the position), a compare-exchange is a 64-bit compare and four selects;
// 64-bit keys: key and position compared lexicographically.  (Odd-even
// transposition on {key, payload}, the previous form, takes VT^2 / 2
// compare-exchanges: 528 for 33 keys against the network's 221.)
template <typename K, int VT>
__device__ __forceinline__ void stable_network_sort(K (&k)[VT], uint32_t (&pos)[VT]) {
    if constexpr (sizeof(K) == 4) {
        constexpr uint32_t flip = std::is_signed<K>::value ? 0x80000000u : 0u;
        uint64_t c[VT];
#pragma unroll
        for (int v = 0; v < VT; ++v)
            c[v] = (uint64_t(uint32_t(k[v]) ^ flip) << 32) | uint32_t(v);
        network_sort<uint64_t, VT>(c);
#pragma unroll
        for (int v = 0; v < VT; ++v) {
            k[v] = K(uint32_t(c[v] >> 32) ^ flip);
            pos[v] = uint32_t(c[v]);
        }
    } else {
#pragma unroll
        for (int v = 0; v < VT; ++v) pos[v] = uint32_t(v);
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
                            const uint32_t px = pos[i + j], py = pos[i + j + q];
                            const bool sw = (y < x) | ((y == x) & (py < px));
                            k[i + j] = sw ? y : x;
                            k[i + j + q] = sw ? x : y;
                            pos[i + j] = sw ? py : px;
                            pos[i + j + q] = sw ? px : py;
                        }
    }
}

// The merge rounds of the block sort: round k merges sorted lists of
// W = VT << k slots in pairs (the last list of the array may be short or
// missing); thread t takes the VT outputs from its merge-path split (the
// Lemma-1 split of corank.hpp:93-94, ties to the left list as
// merge.hpp:22-31).  A list pair spans 2^(k+1) threads, so its start is a
// shift of the thread index.  Rounds whose pairs lie inside one warp's 32*VT
// slots (k < 5) synchronise the warp only.  One rolled loop over the rounds:
// unrolled per round, the 8-9 copies of the VT-step merge overflowed the
// instruction cache (ncu: 9% of the stall samples on no_instructions).
template <typename K, int VT, int S, bool HAS_V>
__device__ __forceinline__ void block_sort_rounds(K* s, uint32_t* sv, int t, bool active,
                                                  K (&k)[VT], uint32_t (&p)[VT]) {
#pragma unroll 1
    for (int r = 0; (VT << r) < S; ++r) {
        const int W = VT << r;
        const bool warp_local = r < 5;
        if (warp_local) __syncwarp(); else __syncthreads();  // previous reads are done
        if (active) {
#pragma unroll
            for (int v = 0; v < VT; ++v) {
                s[t * VT + v] = k[v];
                if constexpr (HAS_V) sv[t * VT + v] = p[v];
            }
        }
        if (warp_local) __syncwarp(); else __syncthreads();
        if (!active) continue;
        const int a0 = ((t >> (r + 1)) << (r + 1)) * VT;
        const int la = S - a0 < W ? S - a0 : W;
        const int b0 = a0 + la;
        const int lb = S - b0 < W ? S - b0 : W;
        uint32_t src[VT];
        // Lemma-1 split of the thread's diagonal (the data-dependent search of
        // merge_serial.cuh; a branch-free fixed-trip form -- 8 instead of 13
        // instructions per iteration -- measured 2^26 int32 keys 1.860 instead
        // of 1.805 ms: threads near a list pair's ends have narrow brackets)
        const int diag = t * VT - a0;
        const K* sA = s + a0;
        const K* sB = s + b0;
        const int j = smem_split<K>(sA, la, sB, lb, diag);
        const uint32_t pa0 = smem_addr(sA), pb0 = smem_addr(sB);
        constexpr uint32_t SZ = sizeof(K);
        serial_merge<K, VT, HAS_V, false>(pa0 + uint32_t(j) * SZ, pa0 + uint32_t(la) * SZ,
                                          pb0 + uint32_t(diag - j) * SZ, pb0 + uint32_t(lb) * SZ,
                                          0, 0, VT, k, src);
        if constexpr (HAS_V) {
            const uint32_t base = smem_addr(s);
            constexpr int SH = sizeof(K) == 8 ? 3 : 2;
#pragma unroll
            for (int v = 0; v < VT; ++v) p[v] = sv[(src[v] - base) >> SH];
        }
    }
}

// Shared body of the keys and key-value block sorts (CFG: NT, VT, R, NA, S).
template <typename K, typename CFG, bool HAS_V>
__device__ __forceinline__ void block_sort_body(K* s, uint32_t* sv, const K* __restrict__ in,
                                                const uint32_t* __restrict__ in_v,
                                                K* __restrict__ out, uint32_t* __restrict__ out_v,
                                                uint64_t n) {
    constexpr int NT = CFG::NT, VT = CFG::VT, R = CFG::R, NA = CFG::NA, S = CFG::S;
    pdl_trigger();  // the first merge pass may be scheduled (it waits for this grid)
    const uint64_t base = uint64_t(blockIdx.x) * R;
    const int cnt = n - base < uint64_t(R) ? int(n - base) : R;
    const int t = threadIdx.x;
    // padding sorts last and, being last in input order, stays behind real maxima
    const K pad = std::numeric_limits<K>::max();
    {  // coalesced loads, all in flight before the first shared store
        constexpr int kIters = (S + 4 + NT - 1) / NT;  // + the merge's look-ahead slack
        K lk[kIters];
        uint32_t lv[kIters];
#pragma unroll
        for (int i = 0; i < kIters; ++i) {
            const int x = t + i * NT;
            lk[i] = x < cnt ? in[base + x] : pad;
            if constexpr (HAS_V) lv[i] = x < cnt ? in_v[base + x] : 0u;
        }
#pragma unroll
        for (int i = 0; i < kIters; ++i) {
            const int x = t + i * NT;
            if (x < S + 4) {
                s[x] = lk[i];
                if constexpr (HAS_V) sv[x] = lv[i];
            }
        }
    }
    __syncthreads();
    const bool active = t < NA;
    K k[VT];
    uint32_t p[VT];
    if (active) {
#pragma unroll
        for (int v = 0; v < VT; ++v) {
            k[v] = s[t * VT + v];
        }
        if constexpr (HAS_V) {
            // the payloads are still where they were loaded: gather by position
            uint32_t pos[VT];
            stable_network_sort<K, VT>(k, pos);
#pragma unroll
            for (int v = 0; v < VT; ++v) p[v] = sv[t * VT + int(pos[v])];
        } else {
            network_sort<K, VT>(k);
        }
    }
    block_sort_rounds<K, VT, S, HAS_V>(s, sv, t, active, k, p);
    __syncthreads();
    if (active) {
#pragma unroll
        for (int v = 0; v < VT; ++v) {
            s[t * VT + v] = k[v];
            if constexpr (HAS_V) sv[t * VT + v] = p[v];
        }
    }
    __syncthreads();
    for (int x = t; x < cnt; x += NT) {
        out[base + x] = s[x];
        if constexpr (HAS_V) out_v[base + x] = sv[x];
    }
}

template <typename K, bool SMALL>
__global__ void __launch_bounds__(sort_cfg<K, SMALL>::NT, sort_cfg<K, SMALL>::kMinBlocks)
    block_sort_kernel(const K* __restrict__ in, K* __restrict__ out, uint64_t n) {
    extern __shared__ __align__(16) unsigned char bs_smem[];
    block_sort_body<K, sort_cfg<K, SMALL>, false>(reinterpret_cast<K*>(bs_smem), nullptr, in,
                                                  nullptr, out, nullptr, n);
}

// Key-value variant: the uint32 payload moves with its key (runs of 8192
// pairs, 4096 for 64-bit keys; keys and payloads in two shared arrays).
template <typename K, bool SMALL = false>
struct sort_pairs_cfg {
    static constexpr int VTB = sizeof(K) == 8 ? SORTP_VT64 : SORTP_VT;
    static constexpr int VT = SMALL ? (VTB + 1) / 2 : VTB;
    static constexpr int RB = sizeof(K) == 8 ? SORTP_R64 : SORTP_R32;
    static constexpr int R = SMALL ? RB / 2 : RB;
    static constexpr int NA = (R + VT - 1) / VT;
    static constexpr int NT = (NA + 31) / 32 * 32;
    static constexpr int S = NA * VT;
    static constexpr size_t kKeys = (size_t(S + 4) * sizeof(K) + 15) / 16 * 16;
    static constexpr size_t kSmem = kKeys + size_t(S + 4) * 4;  // keys, then payloads
    static constexpr int kMinBlocks = block_sort_min_blocks(kSmem, NT);
    static_assert(NA <= NT && (R & (R - 1)) == 0 && VT % 2 == 1, "block sort shape");
};

template <typename K, bool SMALL>
__global__ void __launch_bounds__(sort_pairs_cfg<K, SMALL>::NT, sort_pairs_cfg<K, SMALL>::kMinBlocks)
    block_sort_pairs_kernel(const K* __restrict__ in, const uint32_t* __restrict__ in_v,
                            K* __restrict__ out, uint32_t* __restrict__ out_v, uint64_t n) {
    extern __shared__ __align__(16) unsigned char bs_smem[];
    using C = sort_pairs_cfg<K, SMALL>;
    block_sort_body<K, C, true>(reinterpret_cast<K*>(bs_smem),
                                reinterpret_cast<uint32_t*>(bs_smem + C::kKeys), in, in_v, out,
                                out_v, n);
}

}  // namespace comerge_b200
