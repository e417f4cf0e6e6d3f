// merge_serial.cuh -- the consumers' per-thread serial merge of the tile
// pipeline (merge_pipe.cuh), written for instruction count: the consumer
// warps are issue-bound (ncu, C5: 35 SASS instructions per output step in the
// previous form, the tile pipeline's largest cost after HBM).
//
// One step is the reference's merge_into step (merge.hpp:22-31: take b only
// when b < a, so ties go to A), from shared-memory windows:
//
//     p      = pb < pb_end && (pa >= pa_end || *pb < *pa)
//     out[v] = p ? *pb : *pa;   advance the side taken
//
// with a one-element look-ahead per side (the load for the element after the
// next one issues in the step that consumes it, off the compare chain): one
// SEL of the load address, one LDS, two predicated pointer increments and the
// four predicated register moves of the look-ahead -- about 12 instructions.
// Payload tracking records the shared address of each output's source element
// (one more SEL); the caller turns it into the payload's address.
//
// Segmented tiles: inside a segment it is the same loop with the segment's
// window limits; a thread whose VT outputs cross one segment end switches the
// limits at a fixed step (one compare and two predicated moves per step; the
// whole warp runs that loop when any of its lanes needs it);
// threads crossing two or more segment ends (segments shorter than VT) run a
// compact rolled loop through local memory.
#pragma once

#include <cstdint>
#include <cstdio>

#include "records.cuh"

namespace comerge_b200 {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// element load from a shared-window address (records: records.cuh)
template <typename K>
__device__ __forceinline__ K lds(uint32_t addr) {
    return smem_io<K>::ld(addr);
}

#ifndef COMERGE_SERIAL_LOOKAHEAD
#define COMERGE_SERIAL_LOOKAHEAD 1
#endif

// VT outputs of the merge of A [pa, pa_end) and B [pb, pb_end) (shared
// addresses) starting at their current heads; for v >= sw the limits become
// (pa_end2, pb_end2) (a segment end: both sides of the first segment are
// exhausted after sw steps).  The windows must be readable two elements past
// every limit (stage slack).  Bitwise & / | keep the predicate three ISETPs.
template <typename K, int VT, bool TRACK, bool SWITCH>
__device__ __forceinline__ void serial_merge(uint32_t pa, uint32_t pa_end, uint32_t pb,
                                             uint32_t pb_end, uint32_t pa_end2, uint32_t pb_end2,
                                             int sw, K (&keys)[VT], uint32_t (&src)[VT]) {
    constexpr uint32_t S = sizeof(K);
    K ka = lds<K>(pa), kb = lds<K>(pb);
#if COMERGE_SERIAL_LOOKAHEAD
    K ka1 = lds<K>(pa + S), kb1 = lds<K>(pb + S);
#endif
#pragma unroll
    for (int v = 0; v < VT; ++v) {
        if constexpr (SWITCH) {
            if (v == sw) {
                pa_end = pa_end2;
                pb_end = pb_end2;
            }
        }
        const bool p = (pb < pb_end) & ((pa >= pa_end) | (kb < ka));
        keys[v] = p ? kb : ka;
        const uint32_t q = p ? pb : pa;
        if constexpr (TRACK) src[v] = q;
#if COMERGE_SERIAL_LOOKAHEAD
        const K t = lds<K>(q + 2 * S);
        if (p) {
            pb += S;
            kb = kb1;
            kb1 = t;
        } else {
            pa += S;
            ka = ka1;
            ka1 = t;
        }
#else
        const K t = lds<K>(q + S);
        if (p) {
            pb += S;
            kb = t;
        } else {
            pa += S;
            ka = t;
        }
#endif
    }
}

// Lemma-1 split of diagonal `diag` of windows sA[0, na), sB[0, nb) (the
// reference's co-rank, corank.hpp:72-121, as a one-sided binary search over
// guard 1): the number of outputs taken from A.  (A branch-free form with a
// fixed, warp-uniform trip count -- 7 instructions per iteration instead of
// 13 -- measured 3% slower on C5: the data-dependent loop ends early for the
// many threads whose bracket is narrow.)
template <typename K>
__device__ __forceinline__ int smem_split(const K* sA, int na, const K* sB, int nb, int diag) {
    int l = diag > nb ? diag - nb : 0, h = diag < na ? diag : na;
    while (l < h) {
        const int mid = (l + h + 1) >> 1;
        if (sB[diag - mid] < sA[mid - 1])
            h = mid - 1;
        else
            l = mid;
    }
    return l;
}

// Plain tile: VT outputs from window diagonal `diag`.
template <typename K, int VT, bool TRACK>
__device__ __forceinline__ void merge_thread_lean(const K* sA, int a_len, const K* sB, int b_len,
                                                  int diag, K (&keys)[VT], uint32_t (&src)[VT]) {
    const int ia = smem_split<K>(sA, a_len, sB, b_len, diag);
    const uint32_t a0 = smem_addr(sA), b0 = smem_addr(sB);
    constexpr uint32_t S = sizeof(K);
    serial_merge<K, VT, TRACK, false>(a0 + ia * S, a0 + a_len * S, b0 + (diag - ia) * S,
                                      b0 + b_len * S, 0, 0, VT, keys, src);
}

// Segmented tile from the segment-end table `se` (entry k: window-relative end
// of the tile's k-th segment, x1 | y1 << 16; the last entry is the windows'
// ends).  A segment's windows start where the previous one's end.
template <typename K, int VT, bool TRACK>
__device__ __forceinline__ void merge_thread_segends_lean(const K* sA, const K* sB, int diag,
                                                          const uint32_t* se, int nse,
                                                          K (&keys)[VT], uint32_t (&src)[VT]) {
    int lo = 0, hi = nse - 1;  // first segment whose window part ends past diag
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const uint32_t e = se[mid];
        if (int(e & 0xffffu) + int(e >> 16) > diag)
            hi = mid;
        else
            lo = mid + 1;
    }
    const int k = lo;
    const uint32_t e0 = k > 0 ? se[k - 1] : 0u;
    const int x0 = int(e0 & 0xffffu), y0 = int(e0 >> 16);
    const uint32_t e1 = se[k];
    const int x1 = int(e1 & 0xffffu), y1 = int(e1 >> 16);
    const int dl = diag - x0 - y0;
    const int ia = x0 + smem_split<K>(sA + x0, x1 - x0, sB + y0, y1 - y0, dl);
    const int ib = y0 + (dl - (ia - x0));
    const int rem = (x1 - ia) + (y1 - ib);  // outputs left in segment k
#ifdef COMERGE_DEBUG_CHECKS
    // the segment-end table is monotone and the split lies inside segment k
    if (!(x0 <= ia && ia <= x1 && y0 <= ib && ib <= y1 && x0 <= x1 && y0 <= y1 &&
          (k + 1 >= nse || (int(se[k + 1] & 0xffffu) >= x1 && int(se[k + 1] >> 16) >= y1)) &&
          (diag >= int(se[nse - 1] & 0xffffu) + int(se[nse - 1] >> 16) || rem > 0))) {
        printf("comerge: bad segmented split diag %d k %d/%d x %d..%d..%d y %d..%d..%d\n", diag,
               k, nse, x0, ia, x1, y0, ib, y1);
        __trap();
    }
#endif
    const uint32_t a0 = smem_addr(sA), b0 = smem_addr(sB);
    constexpr uint32_t S = sizeof(K);
    // path: 0 no segment end inside the thread's VT outputs (the common case),
    // 1 exactly one (switch the limits at step `rem`), 2 more (rolled loop)
    int x2 = x1, y2 = y1, path = 0;
    if (!(rem >= VT || k == nse - 1)) {
        const uint32_t e2 = se[k + 1];
        x2 = int(e2 & 0xffffu);
        y2 = int(e2 >> 16);
        path = rem + (x2 - x1) + (y2 - y1) >= VT || k + 1 == nse - 1 ? 1 : 2;
    }
    // Warp-uniform choice between 0 and 1: a lane on the switching loop while
    // its neighbours ran the plain one made the warp execute both (2.25x the
    // steps), and the tile's other warps waited for it at the consumer
    // barrier; now the whole warp switches (lanes without a segment end never
    // reach step VT), 15 instead of 12 instructions per step for that warp.
    const bool warp_switch = __any_sync(0xffffffffu, path == 1);
    // likewise the rolled loop (it handles every case): all lanes or none
    if (__any_sync(0xffffffffu, path == 2)) path = 2;
    if (path != 2) {
        if (warp_switch)
            serial_merge<K, VT, TRACK, true>(a0 + ia * S, a0 + x1 * S, b0 + ib * S, b0 + y1 * S,
                                             a0 + x2 * S, b0 + y2 * S, path ? rem : VT, keys, src);
        else
            serial_merge<K, VT, TRACK, false>(a0 + ia * S, a0 + x1 * S, b0 + ib * S, b0 + y1 * S,
                                              0, 0, VT, keys, src);
        return;
    }
    // two or more segment ends inside VT outputs (segments shorter than VT):
    // a rolled loop, outputs through local memory
    K tk[VT];
    uint32_t ts[VT];
    const K* pa = sA + ia;
    const K* pb = sB + ib;
    const K* pae = sA + x1;
    const K* pbe = sB + y1;
    int kk = k;
#pragma unroll 1
    for (int v = 0; v < VT; ++v) {
        while (pa == pae && pb == pbe && kk < nse - 1) {
            const uint32_t e = se[++kk];
            pae = sA + int(e & 0xffffu);
            pbe = sB + int(e >> 16);
        }
        const bool p = pb < pbe && (pa >= pae || *pb < *pa);
        const K* q = p ? pb : pa;
        tk[v] = *q;
        if constexpr (TRACK) ts[v] = smem_addr(q);
        if (p)
            ++pb;
        else
            ++pa;
    }
#pragma unroll
    for (int v = 0; v < VT; ++v) {
        keys[v] = tk[v];
        if constexpr (TRACK) src[v] = ts[v];
    }
}

}  // namespace comerge_b200
