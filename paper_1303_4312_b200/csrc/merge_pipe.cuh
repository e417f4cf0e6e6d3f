// merge_pipe.cuh -- persistent, self-scheduling tile pipeline for sm_100a
// (the default merge path).
//
// Algorithm 2 of arXiv 1303.4312 (reference
// parallel.hpp:180-282) mapped onto a persistent grid:
//
//   * Work unit = an output tile of T = 256*VT elements.  CTA c owns an equal
//     contiguous static range of the first 70% of the tiles (a reference
//     worker's block, parallel.hpp:201-207: co-rank its start, then every
//     later boundary); the remaining 30% form a dynamic tail claimed one tile
//     at a time from a global counter, their co-ranks computed in the
//     background by a tail warp in every CTA (from kernel start: it takes no
//     part in the start-up barriers).  The tail absorbs the start-up
//     skew between CTAs and the ~25% spread of per-SM streaming rates
//     (B200 GPCs differ).
//   * Scheduler warp: co-ranks its range start (33-ary warp search over the
//     whole diagonal, finished by the consumer warps together with the next 8
//     boundaries), then every later boundary bracketed by its predecessor
//     (lane-group searches, 1, 4, then 8 boundaries per pass, at most 8 tiles
//     ahead of the producer), and pushes tile descriptors (i0, j0, j1, i1, s0,
//     s1) into a shared-memory ring; then claims tail tiles.
//   * Producer warp: per descriptor, waits for a free stage and TMA-loads
//     exactly the tile's A window [j0, j1) and B window [i0-j0, i1-j1) (16-byte
//     aligned supersets, payloads too): every input byte crosses HBM once.
//     Segmented batches: after the loads are issued, the whole warp writes
//     the tile's segment-end table into the stage.
//   * Consumers (8 warps): tile-local co-rank per VT-slot diagonal and the
//     branch-free serial merge (merge.hpp:22-31, ties to A) of
//     merge_serial.cuh (12 instructions per output step);
//     the merged tile is written back into the stage and handed to the store
//     warp, which stores it with one TMA bulk store and releases the stage
//     once the store has read it (consumers never wait on a store).
//   * SEG selects the input model: 0 plain, 1 segmented batch, 2 merge pass
//     of the sort (runs of run_len), 3 pieced inputs (multi-GPU split); any
//     launch merges the output range [out_base, out_end).
#pragma once

#include <cstdint>
#include <cstdio>

#include "corank.cuh"
#include "ptx.cuh"
#include "merge_tile.cuh"
#include "merge_serial.cuh"
#include "records.cuh"

namespace comerge_b200 {

#ifndef PIPE_K32_NC
#define PIPE_K32_NC 256
#define PIPE_K32_VT 31
#define PIPE_K32_NST 3
#endif
#ifndef PIPE_KV32_NC
#define PIPE_KV32_NC 256
#endif
template <typename K, bool HAS_V>
struct pipe_cfg;
// 32-bit keys only: tile 7936, 3 stages of ~31 KB (VT=31 halves the per-output
// cost of the tile-local split search, which dominates keys-only merges).
template <>
struct pipe_cfg<int32_t, false> {
    static constexpr int NC = PIPE_K32_NC, VT = PIPE_K32_VT, NST = PIPE_K32_NST;
};
template <>
struct pipe_cfg<uint32_t, false> : pipe_cfg<int32_t, false> {};
// 32-bit keys + payload: tile 3840, 3 stages of ~31 KB.
#ifndef PIPE_KV32_VT
#define PIPE_KV32_VT 15
#define PIPE_KV32_NST 3
#define PIPE_KV32_MINB 2
#endif
template <>
struct pipe_cfg<int32_t, true> {
    static constexpr int NC = PIPE_KV32_NC, VT = PIPE_KV32_VT, NST = PIPE_KV32_NST;
};
template <>
struct pipe_cfg<uint32_t, true> : pipe_cfg<int32_t, true> {};
// 64-bit keys only (the reference's key_t): tile 3840, 3 stages of ~31 KB
// (2^26 + 2^26 uniform keys: VT 11 x 4 stages 365 us, 13 x 4 346, 15 x 3 341,
// 17 x 3 343 -- fewer, larger tiles amortise the per-tile barriers and probes).
#ifndef PIPE_K64_VT
#define PIPE_K64_VT 15
#define PIPE_K64_NST 3
#endif
template <>
struct pipe_cfg<uint64_t, false> {
    static constexpr int NC = 256, VT = PIPE_K64_VT, NST = PIPE_K64_NST;
};
// 64-bit keys + payload: tile 2816, 3 stages of ~34 KB.
template <>
struct pipe_cfg<uint64_t, true> {
    static constexpr int NC = 256, VT = 11, NST = 3;
};

// key-value records (records.cuh): 8-byte records as the 32-bit key-value
// tile (3840 outputs), 12-byte records 2816 outputs (odd VT: 33-word thread
// stride, conflict-free staging), 16-byte records 1792 outputs; 3 stages of
// 29-34 KB
template <typename KT, int S, int A>
struct pipe_cfg<rec<KT, S, A>, false> {
    static constexpr int NC = 256, VT = S == 8 ? 15 : (S == 12 ? 11 : 7), NST = 3;
};

// SEG: 0 plain merge, 1 segmented batch (explicit offsets), 2 merge pass
// (runs of run_len, implicit offsets; sort.cuh), 3 plain merge of inputs
// held as pieces in several device arrays (a multi-GPU split, peer memory)
template <typename K, bool HAS_V, int SEG = 0>
struct pipe_layout {
    using C = pipe_cfg<K, HAS_V>;
    static constexpr int kConsumers = C::NC;
    static constexpr int kThreads = kConsumers + 128;  // + producer, scheduler, tail, store warps
    static constexpr int kCW = kConsumers / 32;       // consumer warps (roles follow them)
    static constexpr int VT = C::VT;
    static constexpr int T = kConsumers * VT;
    static constexpr int NST = C::NST;
    static constexpr int VECE = 16 / sizeof(K);
    static constexpr int NB = 64;  // tile-descriptor ring entries
    static_assert((T * sizeof(K)) % 16 == 0 && T % 4 == 0, "tile must be 16B multiple");
    static constexpr int KW = ((T + 4 * VECE + VT + 3) + VECE - 1) / VECE * VECE;
    static constexpr int VW = HAS_V ? ((T + 16 + VT + 2) + 3) / 4 * 4 : 0;
    static constexpr size_t kStageKeys = (size_t(KW) * sizeof(K) + 127) / 128 * 128;
    static constexpr size_t kStageVals = (size_t(VW) * 4 + 127) / 128 * 128;
    // segmented batches: the tile's segment-end table (window-relative
    // x1 | y1 << 16 of segments s0 .. s0+SEGCAP-1), written by the producer warp
    static constexpr int SEGCAP = 512;
    // more segments than this in a tile (average under ~8 VT outputs each, so
    // many warps hold a thread crossing two segment ends):
    // consumers use the general per-step segment test instead of the lean loop
#ifndef PIPE_LEAN_SEGS_DIV
#define PIPE_LEAN_SEGS_DIV 8
#endif
    static constexpr int kLeanSegs = PIPE_LEAN_SEGS_DIV ? T / (PIPE_LEAN_SEGS_DIV * VT) : SEGCAP;
    static constexpr bool kSeg = SEG == 1 || SEG == 2;  // segmented modes
    static constexpr size_t kStageOffs = kSeg ? size_t(SEGCAP) * 4 : 0;
    static constexpr size_t kStage = kStageKeys + kStageVals + kStageOffs;
    static constexpr size_t oStages = 0;
    static constexpr size_t oBars = oStages + NST * kStage;
    static constexpr size_t oMeta = oBars + size_t(3 * NST) * 8;  // NST x 8 x u64
    static constexpr size_t oDesc = oMeta + size_t(NST) * 64;      // NB x {i0,j0,j1,i1,s0,s1,-,-}
    static constexpr size_t oScratch = oDesc + size_t(NB) * 64;    // 40 x u64
    static constexpr size_t oMisc = oScratch + 40 * 8;
    static constexpr size_t kMisc = 64;
    static_assert(!kSeg || KW < 65536, "segment ends are packed as 16-bit window offsets");
    static constexpr size_t kSmem = oMisc + kMisc;
};

constexpr int kMaxPipeGrid = 512;
constexpr int kMaxPieces = 8;  // SEG == 3: pieces per input (one per GPU of a node)

struct pipe_args {
    const void* a;
    const uint32_t* av;
    uint64_t m;
    const void* b;
    const uint32_t* bv;
    uint64_t n;
    void* out;
    uint32_t* outv;
    uint64_t ntiles;
    const uint64_t* aoff;        // segmented batches: nseg+1 offsets into a (else NULL)
    const uint64_t* boff;        // segmented batches: nseg+1 offsets into b
    uint64_t nseg;
    unsigned long long* trace;   // optional per-CTA timestamps (8 x u64 per CTA)
    uint64_t static_tiles;       // tiles [0, static_tiles) are split statically (equal shares)
    uint32_t lookahead;          // claim a tail tile when fewer than this are queued
    // dynamic-tail anchors: the tail warps co-rank every tail_unit-th tail
    // boundary (and each of the last tail_single) over the whole diagonal --
    // every probe of such a search misses L2 and pulls a 128-byte line -- and
    // the boundaries between two anchors bracketed by the first (a few
    // lines); tail_unit = 1: every boundary over the whole diagonal
    uint32_t tail_unit;
    uint64_t tail_single;
    uint64_t* tail;              // dynamic tail workspace (16B aligned): {tag, count} + slots
    uint64_t epoch;              // per-launch tag validating tail state (no memset needed)
    uint32_t eager_start;        // co-rank the first tiles' boundaries concurrently (small inputs)
    uint32_t flags;              // benchmarking knobs (bit 0: no split start-up search)
    uint32_t sched_cap;          // most boundaries co-ranked per scheduler pass (<= 32)
    uint32_t sched_ahead;        // most descriptors queued beyond the producer (<= NB, >= sched_cap)
    uint32_t store_evict_first;  // output stores with an L2 evict_first hint
    // merge-pass mode (SEG only; sort passes): a == b == one array of sorted
    // runs of run_len elements, segment s pairs run 2s (its A part) with run
    // 2s+1 (its B part); offsets are implicit: aoff(s) = min(s*L, m),
    // boff(s) = min(s*L, n), A index x at element x + (x/L)*L, B index y at
    // y + (y/L + 1)*L; aoff / boff are NULL.  0 = explicit offsets.
    uint64_t run_len;
    // output range: this launch merges output ranks [out_base, out_end) of the
    // whole merge into out[0, out_end - out_base) (whole merges: 0, m + n)
    uint64_t out_base, out_end;
    // SEG == 3: input A (B) is npa (npb) pieces, piece q = global indices
    // [pa_start[q], pa_start[q+1]) at pa[q] (any device pointer, e.g. a peer
    // GPU's buffer mapped over NVLink); starts are multiples of 16 bytes
    uint32_t npa, npb;
    const void* pa[kMaxPieces];
    const void* pb[kMaxPieces];
    const uint32_t* pav[kMaxPieces];  // payload pieces (HAS_V), same cuts as the keys
    const uint32_t* pbv[kMaxPieces];
    uint64_t pa_start[kMaxPieces + 1];
    uint64_t pb_start[kMaxPieces + 1];
};

// Lane-group (P+1)-ary search for the largest q in [lo, hi] with !pred(q),
// given !pred(lo) and pred monotone (false ... false true ... true).  The
// warp is split into 32/P groups of P lanes (P a power of two); every group
// has its own bracket and predicate arguments.  All 32 lanes must call it.
// With stop > 0 it returns early, once every bracket is at most stop wide:
// the answer is then in [lo, hi] (both updated; the return value is lo).
template <typename Pred>
__device__ __forceinline__ uint64_t group_search_pred(uint64_t& lo, uint64_t& hi, int P,
                                                      Pred pred, uint32_t* rounds,
                                                      uint64_t stop = 0) {
    const int lane = threadIdx.x & 31;
    const int g = lane / P, r = lane % P;
    const unsigned gmask = P == 32 ? 0xffffffffu : ((1u << P) - 1u) << (g * P);
    const uint64_t P1 = uint64_t(P) + 1;
    while (__any_sync(0xffffffffu, hi - lo > stop)) {
        const bool active = hi - lo > stop;
        const uint64_t width = hi - lo;
        const uint64_t q = lo + ((uint64_t(r) + 1) * width + P) / P1;  // in (lo, hi]
        bool not_far = true;
        if (active) not_far = !pred(q);
        const int nfalse = __popc(__ballot_sync(0xffffffffu, not_far) & gmask);
        if (active) {
            const int f = nfalse - 1;
            const uint64_t nlo = f >= 0 ? lo + ((uint64_t(f) + 1) * width + P) / P1 : lo;
            const uint64_t nhi = f + 1 < P ? lo + ((uint64_t(f) + 2) * width + P) / P1 - 1 : hi;
            lo = nlo;
            hi = nhi;
        }
        if (rounds) ++*rounds;
    }
    return lo;
}

// Lemma-1 split of diagonal i of (a, b) inside [lo, hi] (guard 1 of
// corank.hpp:93-94 is the monotone predicate).
template <typename K>
__device__ __forceinline__ uint64_t group_search(uint64_t i, uint64_t lo, uint64_t hi, int P,
                                                 const K* __restrict__ a,
                                                 const K* __restrict__ b,
                                                 uint32_t* rounds = nullptr) {
    return group_search_pred(
        lo, hi, P, [=](uint64_t q) { return probe_elem(b + (i - q)) < probe_elem(a + (q - 1)); },
        rounds);
}
// group_search narrowed only until the bracket [lo, hi] is at most stop wide
template <typename K>
__device__ __forceinline__ void group_narrow(uint64_t i, uint64_t& lo, uint64_t& hi, int P,
                                             const K* __restrict__ a, const K* __restrict__ b,
                                             uint64_t stop) {
    group_search_pred(
        lo, hi, P, [=](uint64_t q) { return probe_elem(b + (i - q)) < probe_elem(a + (q - 1)); },
        nullptr, stop);
}

// Stage src[lo, hi) for a TMA copy whose destination `dst` corresponds to
// element lo - lo % vece: returns the 16-byte-multiple body in bytes; the
// elements past the array's last full 16 bytes are copied here (scalar).
template <typename E>
__device__ __forceinline__ uint32_t stage_copy_plan(const E* __restrict__ src, uint64_t len,
                                                    uint64_t lo, uint64_t hi, E* dst, int vece) {
    if (hi <= lo) return 0;
    const uint64_t lo_al = lo - lo % vece;
    uint64_t hi_al = (hi + vece - 1) / vece * vece;
    const uint64_t len_al = len - len % vece;
    if (hi_al > len) hi_al = len_al > lo_al ? len_al : lo_al;
    for (uint64_t e = hi_al; e < hi; ++e) dst[e - lo_al] = src[e];
    return uint32_t((hi_al - lo_al) * sizeof(E));
}

// Byte-space staging of window [lo, hi) of an array of S-byte elements at
// `base` (any 4-byte aligned address; S a multiple of 4) into the 16-byte
// aligned stage slot `dst`, whose byte 0 stands for the 16-byte boundary at or
// below the window's first byte -- so a window keeps its address offset
// modulo 16 in shared memory, and misaligned arrays (any element offset into
// an allocation) stream through the same TMA copies as aligned ones.  The
// 16-byte blocks wholly inside the array form the bulk copy (planned here,
// issued by the caller); the words of the partial blocks at the array's two
// ends are copied here (at most 3 per end).
struct win_plan {
    const unsigned char* src;  // bulk source (16-byte aligned)
    uint32_t dst_off;          // its offset in dst
    uint32_t bytes;            // bulk bytes (a multiple of 16, may be 0)
    uint32_t first;            // offset of element lo in dst (0..15)
    uint32_t span;             // bytes of dst the window occupies, rounded up to 16
};

__device__ __forceinline__ win_plan plan_window(const void* base, uint64_t len, uint32_t S,
                                                uint64_t lo, uint64_t hi, unsigned char* dst) {
    const uintptr_t B = reinterpret_cast<uintptr_t>(base);
    const uintptr_t W0 = B + lo * S, W1 = B + (hi > lo ? hi : lo) * S;
    const uintptr_t A0 = W0 & ~uintptr_t(15);
    const uintptr_t in0 = (B + 15) & ~uintptr_t(15), in1 = (B + len * S) & ~uintptr_t(15);
    uintptr_t b0 = A0 > in0 ? A0 : in0;
    uintptr_t b1 = (W1 + 15) & ~uintptr_t(15);
    if (b1 > in1) b1 = in1;
    if (b1 < b0) b1 = b0;
    const uintptr_t h1 = b0 > W0 ? (b0 < W1 ? b0 : W1) : W0;  // head words [W0, h1)
    for (uintptr_t x = W0; x < h1; x += 4)
        *reinterpret_cast<uint32_t*>(dst + (x - A0)) = *reinterpret_cast<const uint32_t*>(x);
    for (uintptr_t x = b1 > h1 ? b1 : h1; x < W1; x += 4)  // tail words
        *reinterpret_cast<uint32_t*>(dst + (x - A0)) = *reinterpret_cast<const uint32_t*>(x);
    win_plan p;
    p.src = reinterpret_cast<const unsigned char*>(b0);
    p.dst_off = uint32_t(b0 - A0);
    p.bytes = uint32_t(b1 - b0);
    p.first = uint32_t(W0 - A0);
    p.span = uint32_t(((W1 + 15) & ~uintptr_t(15)) - A0);
    return p;
}

// Byte-space store of `len` S-byte elements to out + pos*S (any 4-byte aligned
// address) from the stage, where the consumers wrote element 0 at
// src_al + (destination address mod 16) (src_al 16-byte aligned): the 16-byte
// blocks wholly inside the range are one TMA bulk store, the words of the
// partial blocks at its ends plain stores (tiles of neighbouring CTAs write
// the other words of those blocks).
__device__ __forceinline__ void store_window(void* out, uint64_t pos, int len, uint32_t S,
                                             const unsigned char* src_al, bool hint,
                                             uint64_t policy) {
    if (len <= 0) return;
    const uintptr_t W0 = reinterpret_cast<uintptr_t>(out) + pos * S, W1 = W0 + uint64_t(len) * S;
    const uintptr_t A0 = W0 & ~uintptr_t(15);
    uintptr_t b0 = (W0 + 15) & ~uintptr_t(15), b1 = W1 & ~uintptr_t(15);
    if (b1 < b0) b1 = b0;
    if (b1 > b0) {
        void* d = reinterpret_cast<void*>(b0);
        const unsigned char* sp = src_al + (b0 - A0);
        if (hint)
            tma_store_1d_hint(d, sp, uint32_t(b1 - b0), policy);
        else
            tma_store_1d(d, sp, uint32_t(b1 - b0));
    }
    const uintptr_t h1 = b0 < W1 ? b0 : W1;
    for (uintptr_t x = W0; x < h1; x += 4)
        *reinterpret_cast<uint32_t*>(x) = *reinterpret_cast<const uint32_t*>(src_al + (x - A0));
    for (uintptr_t x = b1 > h1 ? b1 : h1; x < W1; x += 4)
        *reinterpret_cast<uint32_t*>(x) = *reinterpret_cast<const uint32_t*>(src_al + (x - A0));
}

// merge-pass runs: L is a power of two (sort.cuh's base runs, doubled every
// pass; checked at launch), so run arithmetic is shifts, not 64-bit divisions
// (the producer lane stages every window through stage_runs)
__device__ __forceinline__ int run_lg(uint64_t L) { return __ffsll((long long)L) - 1; }

// Merge pass: stage the window [x0, x1) of one side's index space, element x
// at src[x + (x/L + shift) * L] (shift 0 for A, 1 for B), as one TMA copy per
// run it touches (runs are physically contiguous; L is a multiple of vece, so
// every piece after the first starts 16-byte aligned at its place in `dst`,
// which corresponds to index x0 - x0 % vece).  issue == false: plan only
// (scalar tails copied, bytes returned); issue == true: the copies.
template <typename E>
__device__ __forceinline__ uint32_t stage_runs(const E* __restrict__ src, uint64_t phys_len,
                                               uint64_t x0, uint64_t x1, uint64_t L,
                                               uint64_t shift, E* dst, int vece, bool issue,
                                               uint64_t* bar, uint64_t policy) {
    uint32_t total = 0;
    const uint64_t base = x0 - x0 % vece;
    const int lg = run_lg(L);
    for (uint64_t x = x0; x < x1;) {
        const uint64_t run = x >> lg;
        const uint64_t y = x1 < ((run + 1) << lg) ? x1 : ((run + 1) << lg);
        const uint64_t sh = (run + shift) << lg;  // physical = index + sh
        E* d = dst + ((x - x % vece) - base);
        if (!issue) {
            total += stage_copy_plan(src, phys_len, x + sh, y + sh, d, vece);
        } else {
            const uint64_t lo = x + sh, lo_al = lo - lo % vece;
            uint64_t hi_al = (y + sh + vece - 1) / vece * vece;
            const uint64_t len_al = phys_len - phys_len % vece;
            if (hi_al > phys_len) hi_al = len_al > lo_al ? len_al : lo_al;
            const uint32_t bytes = uint32_t((hi_al - lo_al) * sizeof(E));
            if (bytes) tma_load_1d(d, src + lo_al, bytes, bar, policy);
            total += bytes;
        }
        x = y;
    }
    return total;
}

__device__ __forceinline__ uint64_t ldg_u64(const uint64_t* p) {  // L2-only, like probe_elem
    return static_cast<uint64_t>(__ldcg(reinterpret_cast<const unsigned long long*>(p)));
}

// merge-pass mode: implicit offsets and element positions (see pipe_args)
__device__ __forceinline__ uint64_t run_off(uint64_t s, uint64_t L, uint64_t len) {
    const uint64_t o = s * L;
    return o < len ? o : len;
}
__device__ __forceinline__ uint64_t run_pos_a(uint64_t x, uint64_t L) { return x + (x & ~(L - 1)); }
__device__ __forceinline__ uint64_t run_pos_b(uint64_t y, uint64_t L) {
    return y + (y & ~(L - 1)) + L;
}

// SEG == 3: element x of a pieced input (linear scan: at most kMaxPieces)
template <typename K>
__device__ __forceinline__ typename key_of<K>::type piece_probe(const void* const* p,
                                                                const uint64_t* st, uint32_t np,
                                                                uint64_t x) {
    uint32_t q = 0;
    while (q + 1 < np && st[q + 1] <= x) ++q;
    return probe_elem(static_cast<const K*>(p[q]) + (x - st[q]));
}

// SEG == 3: stage the window [x0, x1) of a pieced input (dst <-> index
// x0 - x0 % vece) as one TMA copy per piece it touches; issue == false: plan
// only (scalar tails copied, bytes returned) -- as stage_runs.
template <typename E>
__device__ __forceinline__ uint32_t stage_pieces(const void* const* p, const uint64_t* st,
                                                 uint32_t np, uint64_t x0, uint64_t x1, E* dst,
                                                 int vece, bool issue, uint64_t* bar,
                                                 uint64_t policy) {
    uint32_t total = 0;
    const uint64_t base = x0 - x0 % vece;
    for (uint32_t q = 0; q < np; ++q) {
        const uint64_t lo = x0 > st[q] ? x0 : st[q];
        const uint64_t hi = x1 < st[q + 1] ? x1 : st[q + 1];
        if (lo >= hi) continue;
        const E* src = static_cast<const E*>(p[q]);
        const uint64_t plen = st[q + 1] - st[q];
        E* d = dst + ((lo - lo % vece) - base);
        if (!issue) {
            total += stage_copy_plan(src, plen, lo - st[q], hi - st[q], d, vece);
        } else {
            const uint64_t l = lo - st[q], l_al = l - l % vece;
            uint64_t h_al = (hi - st[q] + vece - 1) / vece * vece;
            const uint64_t len_al = plen - plen % vece;
            if (h_al > plen) h_al = len_al > l_al ? len_al : l_al;
            const uint32_t bytes = uint32_t((h_al - l_al) * sizeof(E));
            if (bytes) tma_load_1d(d, src + l_al, bytes, bar, policy);
            total += bytes;
        }
    }
    return total;
}

// A tile boundary: co-rank j of output rank i and, for segmented batches, the
// segment s that holds it (largest s with aoff[s] + boff[s] <= i).
struct boundary {
    uint64_t j;
    uint64_t s;
};

// Boundary search for the lane's group: i with j in [jlo, jhi] and, when SEG,
// s >= slo.  Segmented: the segment by a lane-group search over the
// (L2-resident) offsets, then the co-rank inside that segment (the batch is
// one merge over (segment, key) composites, so the split of a rank inside
// segment s is s's own co-rank).
template <typename K, int SEG>
__device__ __forceinline__ boundary find_boundary(const pipe_args& args, uint64_t i, uint64_t jlo,
                                                  uint64_t jhi, uint64_t slo, int P,
                                                  uint32_t* rounds) {
    const K* __restrict__ a = static_cast<const K*>(args.a);
    const K* __restrict__ b = static_cast<const K*>(args.b);
    if constexpr (SEG == 0) {
        return {group_search<K>(i, jlo, jhi, P, a, b, rounds), 0};
    } else if constexpr (SEG == 3) {
        uint64_t lo = jlo, hi = jhi;
        const uint64_t j = group_search_pred(
            lo, hi, P,
            [&](uint64_t q) {
                return piece_probe<K>(args.pb, args.pb_start, args.npb, i - q) <
                       piece_probe<K>(args.pa, args.pa_start, args.npa, q - 1);
            },
            rounds);
        return {j, 0};
    } else {
        if constexpr (SEG == 2) {  // merge pass: pair s holds output ranks [2sL, 2sL + 2L)
            const uint64_t L = args.run_len;
            uint64_t s = i >> (run_lg(L) + 1);
            if (s > args.nseg - 1) s = args.nseg - 1;
            const uint64_t as = run_off(s, L, args.m), bs = run_off(s, L, args.n);
            const uint64_t ma = run_off(s + 1, L, args.m) - as, nb = run_off(s + 1, L, args.n) - bs;
            const uint64_t li = i - as - bs;
            uint64_t lo = li > nb ? li - nb : 0, hi = li < ma ? li : ma;
            if (jlo > as && jlo - as > lo) lo = jlo - as;
            if (jhi < as + hi) hi = jhi > as ? jhi - as : 0;
            if (hi < lo) hi = lo;
            return {as + group_search<K>(li, lo, hi, P, a + run_pos_a(as, L), b + run_pos_b(bs, L),
                                         rounds),
                    s};
        }
        const uint64_t* __restrict__ ao = args.aoff;
        const uint64_t* __restrict__ bo = args.boff;
        uint64_t shi = args.nseg - 1;
        const uint64_t s = group_search_pred(
            slo, shi, P, [=](uint64_t q) { return ldg_u64(ao + q) + ldg_u64(bo + q) > i; },
            rounds);
        const uint64_t as = ldg_u64(ao + s), bs = ldg_u64(bo + s);
        const uint64_t ma = ldg_u64(ao + s + 1) - as, nb = ldg_u64(bo + s + 1) - bs;
        const uint64_t li = i - as - bs;  // <= ma + nb
        uint64_t lo = li > nb ? li - nb : 0, hi = li < ma ? li : ma;
        if (jlo > as && jlo - as > lo) lo = jlo - as;
        if (jhi < as + hi) hi = jhi > as ? jhi - as : 0;
        if (hi < lo) hi = lo;
        return {as + group_search<K>(li, lo, hi, P, a + as, b + bs, rounds), s};
    }
}

// ---- dynamic tail state.  The workspace is not cleared between launches;
// every word is validated against this launch's 64-bit epoch instead:
//   tail[0..1]     = {tag, count}: reset once per launch by a 128-bit CAS
//   tail[4]        = launch counter (any initial value): every CTA claims until
//                    it draws an index past the tail, so the launch's last claim
//                    is number (tail tiles + CTAs - 1); that claimer bumps it
//   slot q (32 B)  = {j, s, hash(epoch, q, j, s), 0} at tail + kTailSlots + 4q
// The epoch is the host's per-call salt mixed with the launch counter, so it
// changes on every launch even when a CUDA graph replays identical arguments.
constexpr int kTailSlots = 8;  // u64 words before the first slot
__device__ __forceinline__ uint64_t tail_hash(uint64_t epoch, uint64_t q, uint64_t j,
                                              uint64_t s) {
    uint64_t x = epoch ^ (q * 0x9e3779b97f4a7c15ULL) ^ (j + 0x632be59bd9b4e019ULL) ^
                 (s * 0xd1b54a32d192ed03ULL);
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__device__ __forceinline__ void cas128(uint64_t* addr, uint64_t clo, uint64_t chi, uint64_t vlo,
                                       uint64_t vhi, uint64_t& dlo, uint64_t& dhi) {
    asm volatile(
        "{\n .reg .b128 c, v, d;\n mov.b128 c, {%2, %3};\n mov.b128 v, {%4, %5};\n"
        " atom.global.cas.b128 d, [%6], c, v;\n mov.b128 {%0, %1}, d;\n}\n"
        : "=l"(dlo), "=l"(dhi)
        : "l"(clo), "l"(chi), "l"(vlo), "l"(vhi), "l"(addr)
        : "memory");
}

__device__ __forceinline__ void st_pair(uint64_t* p, uint64_t x, uint64_t y) {
    asm volatile("st.global.relaxed.gpu.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(x), "l"(y)
                 : "memory");
}

__device__ __forceinline__ void ld_pair(const uint64_t* p, uint64_t& x, uint64_t& y) {
    asm volatile("ld.global.relaxed.gpu.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(p)
                 : "memory");
}

// Claim the next tail tile index (0-based) of this launch.  `checked`: this
// caller has already seen the counter carry this launch's tag (it cannot
// change again within the launch), so the claim is one atomic round trip
// instead of a tag read followed by the atomic.
__device__ __forceinline__ uint64_t tail_claim(uint64_t* tail, uint64_t epoch, bool& checked) {
    if (!checked) {
        uint64_t tag, cnt;
        ld_pair(tail, tag, cnt);
        if (tag != epoch) {
            uint64_t dt, dc;
            cas128(tail, tag, cnt, epoch, 0, dt, dc);  // first claimer of this launch resets
        }
        checked = true;
    }
    return atomicAdd(reinterpret_cast<unsigned long long*>(tail + 1), 1ull);
}

__device__ __forceinline__ int pow2_group(int k) {  // lanes per group for k searches
    int p = 32;
    while (p > 1 && (32 / p) < k) p >>= 1;
    return p;
}

template <typename K, bool HAS_V>
struct pipe_min_blocks {
    static constexpr int value = 2;
};
template <>
struct pipe_min_blocks<int32_t, true> {
    static constexpr int value = PIPE_KV32_MINB;
};

// Segmented consumer merge: VT outputs from window diagonal `diag` of a tile
// whose windows hold A[j0, j0+a_len) and B[k0, k0+b_len) of a batch of
// independent pairs; s_lo..s_hi bound the segments the tile touches.
// Segment offsets in global memory (the fallback for tiles touching more
// than SEGCAP segments, where no segment-end table is built).
struct seg_offsets {
    const uint64_t* ao;
    const uint64_t* bo;
    __device__ __forceinline__ uint64_t a(uint64_t s) const { return ldg_u64(ao + s); }
    __device__ __forceinline__ uint64_t b(uint64_t s) const { return ldg_u64(bo + s); }
};

// Segmented consumer merge: VT outputs from window diagonal `diag` of a tile
// whose windows hold A[j0, j0+a_len) and B[k0, k0+b_len) of a batch of
// independent pairs; s_lo..s_hi bound the segments the tile touches.
template <typename K, int VT>
__device__ __forceinline__ void merge_thread_seg(const K* sA, int a_len, const K* sB, int b_len,
                                                 int diag, uint64_t i0, uint64_t j0, uint64_t k0,
                                                 uint64_t s_lo, uint64_t s_hi,
                                                 const seg_offsets& off, K (&keys)[VT]) {
    // segment holding output rank i0 + diag
    const uint64_t gi = i0 + uint64_t(diag);
    uint64_t lo = s_lo, hi = s_hi;
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo + 1) / 2;
        if (off.a(mid) + off.b(mid) <= gi)
            lo = mid;
        else
            hi = mid - 1;
    }
    uint64_t s = lo;
    // the segment's part of the windows (window-relative [x0, x1) / [y0, y1))
    auto seg_span = [&](uint64_t sg, int& x0, int& x1, int& y0, int& y1) {
        const uint64_t as = off.a(sg), ae = off.a(sg + 1);
        const uint64_t bs = off.b(sg), be = off.b(sg + 1);
        x0 = as > j0 ? int(as - j0) : 0;
        x1 = ae > j0 ? int(ae - j0 < uint64_t(a_len) ? ae - j0 : uint64_t(a_len)) : 0;
        y0 = bs > k0 ? int(bs - k0) : 0;
        y1 = be > k0 ? int(be - k0 < uint64_t(b_len) ? be - k0 : uint64_t(b_len)) : 0;
    };
    int x0, x1, y0, y1;
    seg_span(s, x0, x1, y0, y1);
    // split of the diagonal inside the segment (plain key order there)
    const int dl = diag - x0 - y0;
    const int na = x1 - x0, nb = y1 - y0;
    int l = dl > nb ? dl - nb : 0, h = dl < na ? dl : na;
    while (l < h) {
        const int mid = (l + h + 1) >> 1;
        if (sB[y0 + dl - mid] < sA[x0 + mid - 1])
            h = mid - 1;
        else
            l = mid;
    }
    int ia = x0 + l, ib = y0 + dl - l;
    K ka = sA[ia], kb = sB[ib];
    K ka1 = sA[ia + 1], kb1 = sB[ib + 1];  // look-ahead (see merge_thread)
#pragma unroll
    for (int v = 0; v < VT; ++v) {
        if (ia >= x1 && ib >= y1) {  // segment done: next non-empty one (rare)
            while (ia >= x1 && ib >= y1 && s < s_hi) {
                ++s;
                seg_span(s, x0, x1, y0, y1);
            }
        }
        const bool take_b = ib < y1 && (ia >= x1 || kb < ka);
        keys[v] = take_b ? kb : ka;
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

// Segmented consumer merge from the tile's segment-end table `se` (entry k:
// window-relative end of segment s_lo + k, x1 | y1 << 16; the last entry is
// (a_len, b_len)).  A segment's windows start where the previous one's end,
// so a segment change only moves the limits x1 / y1: the per-step cost over
// merge_thread is one test, and the rare change is two shared loads.
template <typename K, int VT, bool TRACK = false>
__device__ __forceinline__ void merge_thread_segends(const K* sA, const K* sB, int diag,
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
    int k = lo;
    const uint32_t e0 = k > 0 ? se[k - 1] : 0u;
    const int x0 = int(e0 & 0xffffu), y0 = int(e0 >> 16);
    uint32_t e1 = se[k];
    int x1 = int(e1 & 0xffffu), y1 = int(e1 >> 16);
    const int dl = diag - x0 - y0;
    const int na = x1 - x0, nb = y1 - y0;
    int l = dl > nb ? dl - nb : 0, h = dl < na ? dl : na;
    while (l < h) {
        const int mid = (l + h + 1) >> 1;
        if (sB[y0 + dl - mid] < sA[x0 + mid - 1])
            h = mid - 1;
        else
            l = mid;
    }
    int ia = x0 + l, ib = y0 + dl - l;
    K ka = sA[ia], kb = sB[ib];
    K ka1 = sA[ia + 1], kb1 = sB[ib + 1];
    int rem = (x1 - ia) + (y1 - ib);  // outputs left in the current segment
#pragma unroll
    for (int v = 0; v < VT; ++v) {
        if (rem == 0 && k < nse - 1) {  // next non-empty segment (rare)
            do {
                e1 = se[++k];
                x1 = int(e1 & 0xffffu);
                y1 = int(e1 >> 16);
                rem = (x1 - ia) + (y1 - ib);
            } while (rem == 0 && k < nse - 1);
        }
        --rem;
        const bool take_b = ib < y1 && (ia >= x1 || kb < ka);
        keys[v] = take_b ? kb : ka;
        if constexpr (TRACK) src[v] = smem_addr(take_b ? sB + ib : sA + ia);
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

template <typename K, bool HAS_V, int SEG>
__global__ void __launch_bounds__(pipe_layout<K, HAS_V>::kThreads, pipe_min_blocks<K, HAS_V>::value)
    merge_pipe_kernel(const pipe_args args) {
    using L = pipe_layout<K, HAS_V, SEG>;
    constexpr int NC = L::kConsumers;
    constexpr int VT = L::VT;
    constexpr int T = L::T;
    constexpr int NST = L::NST;
    constexpr int VECE = L::VECE;
    constexpr int NB = L::NB;
    static_assert(!(SEG == 1 && HAS_V), "explicit-offset segmented batches are keys-only");
    constexpr bool SEGM = L::kSeg;

    extern __shared__ __align__(128) unsigned char smem[];
    pdl_wait();     // inputs written by a preceding grid (sort passes) are visible
    pdl_trigger();  // the next pass may be scheduled as SMs free up
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::oBars);
    uint64_t* empty = full + NST;
    uint64_t* staged = empty + NST;  // consumers -> store warp: tile written to the stage
    uint64_t* meta = reinterpret_cast<uint64_t*>(smem + L::oMeta);
    uint64_t* desc = reinterpret_cast<uint64_t*>(smem + L::oDesc);
    uint64_t* scratch = reinterpret_cast<uint64_t*>(smem + L::oScratch);
    volatile uint32_t* pushed = reinterpret_cast<volatile uint32_t*>(smem + L::oMisc);
    volatile uint32_t* issued = pushed + 1;

    const K* __restrict__ a = static_cast<const K*>(args.a);
    const K* __restrict__ b = static_cast<const K*>(args.b);
    const uint64_t m = args.m, n = args.n, total = m + n;
    const uint64_t NT = args.ntiles;
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const uint32_t G = gridDim.x, c = blockIdx.x;
    const uint64_t NS = args.static_tiles;

    const uint64_t out_base = args.out_base, out_end = args.out_end;
    auto diag_of = [=](uint64_t t) {  // output rank of tile boundary t
        const uint64_t d = out_base + t * uint64_t(T);
        return d < out_end ? d : out_end;
    };
    auto full_bracket = [=](uint64_t i, uint64_t& lo, uint64_t& hi) {
        lo = i > n ? i - n : 0;
        hi = i < m ? i : m;
    };
    // bracket of boundary i from a known boundary (ic, jc) below it: at least
    // jc and at most jc + (i - ic) elements come from A
    auto step_bracket = [=](uint64_t i, uint64_t ic, uint64_t jc, uint64_t& lo, uint64_t& hi) {
        lo = jc;
        if (i > n && i - n > lo) lo = i - n;
        hi = jc + (i - ic);
        if (i < hi) hi = i;
        if (m < hi) hi = m;
    };

    const unsigned long long t_start = globaltimer_ns();
    if (args.trace && tid == 0) {
        args.trace[8 * c + 0] = t_start;
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        args.trace[8 * c + 4] = smid;
    }
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(&full[s], SEGM ? 2 : 1);  // segmented: + the producer warp's table
            mbar_init(&empty[s], 1);
            mbar_init(&staged[s], 1);
        }
        *pushed = 0;
        *issued = 0;
        // this launch's tail epoch (see kTailSlots): read before the last claim
        uint64_t e = args.epoch;
        if (args.tail) {
            uint64_t lc, pad;
            ld_pair(args.tail + 4, lc, pad);
            e ^= tail_hash(lc, 0x5eedull, 0, 0);
        }
        scratch[38] = e;
        // pull this CTA's share of an array into L2 (cp.async.bulk.prefetch)
        auto pull = [&](const void* base, uint64_t len, uint32_t esz) {
            const uint64_t x0 = len * c / G, x1 = len * (c + 1) / G;
            const uintptr_t B = reinterpret_cast<uintptr_t>(base);
            uintptr_t b0 = (B + x0 * esz) & ~uintptr_t(15), b1 = (B + x1 * esz) & ~uintptr_t(15);
            while (b1 > b0) {
                const uintptr_t chunk = b1 - b0 < (uintptr_t(1) << 20) ? b1 - b0 : (uintptr_t(1) << 20);
                prefetch_l2(reinterpret_cast<const void*>(b0), uint32_t(chunk));
                b0 += chunk;
            }
        };
        if (SEG == 1 && !(args.flags & 8192u)) {
            // segmented batches: the segment offsets (16 B per pair, a few
            // hundred bytes per CTA) go to L2 at once; every start-up boundary
            // search probes them first, so its later segment rounds hit L2
            pull(args.aoff, args.nseg + 1, 8);
            pull(args.boff, args.nseg + 1, 8);
        }
        if (SEG == 0 && args.eager_start && !(args.flags & 4096u)) {
            // small inputs: pull this CTA's share of A and B (and payloads) into
            // L2 at once, so the start-up co-rank rounds and the first window
            // loads run at L2 instead of HBM latency
            if (m) pull(args.a, m, sizeof(K));
            if (n) pull(args.b, n, sizeof(K));
            if (HAS_V && m) pull(args.av, m, 4);
            if (HAS_V && n) pull(args.bv, n, 4);
        }
        mbar_fence_init();
        __threadfence_block();
    }
    // ---- start-up: this worker's static range [ts0, te0), an equal share of
    // the first NS tiles, then co-rank its start with one warp (33-ary; few
    // concurrent probes keep rounds short) and the next 8 boundaries
    // bracketed by it.
    // scratch: [0..8] j of boundaries ts0..ts0+8, [10..18] their segments,
    // [36..37] the start's bracket after the first rounds
    uint64_t ts0 = 0, te0 = 0;
    constexpr int W_PROD = L::kCW, W_SCHED = L::kCW + 1, W_TAIL = L::kCW + 2,
                  W_STORE = L::kCW + 3;
    ts0 = NS * c / G;  // static range
    te0 = NS * (c + 1) / G;
    // boundaries ts0+1 .. ts0+known are co-ranked at start-up by the consumer warps
    const int known = te0 > ts0 ? (te0 - ts0 < 8 ? int(te0 - ts0) : 8) : 0;
    // large plain merges: the scheduler narrows the start's bracket to one tile,
    // hands it to the consumer warps (named barrier 2), and both finish their
    // searches concurrently (boundary w is in [lo, hi + (i_w - i_0)])
    const bool split_start = SEG == 0 && !args.eager_start && known > 0 && !(args.flags & 1u);
    constexpr int kSplitBar = 32 * (L::kCW + 1);
    if (warp == 0) {  // thread 0's initialisation (the tail epoch) is done
        __syncwarp();
        named_bar_arrive(5, 64);
    }
    if (warp == W_TAIL) {
        // ------------------------------------------------------ tail warp
        // (takes no part in the start-up: it starts at once, with the epoch
        // handed over by warp 0 on named barrier 5, so its full-diagonal
        // searches finish ~the start-up's length earlier -- on C2 the first
        // tail claims otherwise found their slots unpublished)
        named_bar_sync(5, 64);
        const uint64_t epoch = scratch[38];
        // co-rank the tail boundaries q = c, c+G, ... (in passes of up to 32,
        // lane groups, full-diagonal brackets) and publish them
        // slot x = boundary NS + x.  Anchors: x = 0, U, 2U, .. below nbig,
        // then every x in [nbig, ntail) (the last tail_single tiles); boundary
        // NT (x = ntail) is trivial for a whole merge, else an anchor too.
        const uint64_t U = args.tail_unit ? args.tail_unit : 1;
        const uint64_t ntail = NT > NS ? NT - NS : 0;
        const uint64_t nsingle = args.tail_single < ntail ? args.tail_single : ntail;
        const uint64_t nbig = ntail - nsingle;
        const uint64_t nbu = (nbig + U - 1) / U;
        auto anchor_x = [=](uint64_t q) {
            return q <= nbu ? (q * U < nbig ? q * U : nbig) : nbig + (q - nbu);
        };
        const uint64_t nanch = ntail ? nbu + nsingle + (out_end < total ? 1 : 0) : 0;
        auto publish = [&](uint64_t x, boundary bd) {
            uint64_t* slot = args.tail + kTailSlots + 4 * x;
            st_pair(slot, bd.j, bd.s);
            st_pair(slot + 2, tail_hash(epoch, x, bd.j, bd.s), 0);
        };
        for (uint64_t q0 = c; q0 < nanch; q0 += 32 * uint64_t(G)) {
            uint64_t left = (nanch - q0 + G - 1) / G;
            const int k = int(left < 32 ? left : 32);
            const int P = pow2_group(k);
            const int g = lane / P;
            const uint64_t q = q0 + uint64_t(g < k ? g : k - 1) * G;
            const uint64_t xa = anchor_x(q);
            const uint64_t i = diag_of(NS + xa);
            uint64_t lo, hi;
            full_bracket(i, lo, hi);
            const boundary bd = find_boundary<K, SEG>(args, i, lo, hi, 0, P, nullptr);
            if (lane % P == 0 && g < k) publish(xa, bd);
            if (U == 1 || q0 >= nbu) continue;  // no inner boundaries in this pass
            // inner boundaries x in (anchor_x(q), anchor_x(q+1)) of the pass's
            // anchors, 32 per round (one lane each, binary search), bracketed
            // by their anchor: j(x) in [j(xa), j(xa) + (i(x) - i(xa))]
            const int per = int(U - 1);
            for (int base = 0; base < k * per; base += 32) {
                const int idx = base + lane;
                const int ga = idx / per < k ? idx / per : k - 1;
                const uint64_t qa = q0 + uint64_t(ga) * G;
                const boundary ba{__shfl_sync(0xffffffffu, bd.j, ga * P),
                                  __shfl_sync(0xffffffffu, bd.s, ga * P)};
                const uint64_t x0 = anchor_x(qa), x1 = qa < nbu ? anchor_x(qa + 1) : x0;
                const uint64_t x = x0 + 1 + uint64_t(idx % per);
                const bool valid = idx < k * per && x < x1;
                const uint64_t ix = diag_of(NS + (valid ? x : x0));
                uint64_t ilo = ba.j, ihi = ba.j;
                if (valid) step_bracket(ix, diag_of(NS + x0), ba.j, ilo, ihi);
                const boundary bi = find_boundary<K, SEG>(args, ix, ilo, ihi, ba.s, 1, nullptr);
                if (valid) publish(x, bi);
            }
        }
        if (args.trace && lane == 0) args.trace[16 * 4096 + 4 * c + 1] = globaltimer_ns();
        return;
    }

    if (warp == W_SCHED) {
        if (te0 > ts0) {
            const uint64_t i = diag_of(ts0);
            uint64_t lo, hi;
            full_bracket(i, lo, hi);
            boundary bd{0, 0};
            if constexpr (SEG == 0) {
                if (split_start) {
                    group_narrow<K>(i, lo, hi, 32, a, b, uint64_t(T));
                    if (lane == 0) {
                        scratch[36] = lo;
                        scratch[37] = hi;
                    }
                    __syncwarp();
                    named_bar_sync(2, kSplitBar);
                }
            }
            bd = find_boundary<K, SEG>(args, i, lo, hi, 0, 32, nullptr);
            if (lane == 0) {
                scratch[0] = bd.j;
                scratch[10] = bd.s;
            }
        }
    } else if (warp < L::kCW && (split_start || (args.eager_start && known > 0))) {
        uint64_t lo0 = 0, hi0 = 0;
        if (split_start) {
            named_bar_sync(2, kSplitBar);
            lo0 = scratch[36];
            hi0 = scratch[37];
        }
        if (warp < known) {
            const uint64_t i = diag_of(ts0 + 1 + uint64_t(warp));
            uint64_t lo, hi;
            full_bracket(i, lo, hi);
            if (split_start) {  // j(i) >= j(i_0) >= lo0, j(i) <= j(i_0) + (i - i_0)
                const uint64_t up = hi0 + (i - diag_of(ts0));
                if (lo0 > lo) lo = lo0;
                if (up < hi) hi = up;
            }
            const boundary bd = find_boundary<K, SEG>(args, i, lo, hi, 0, 32, nullptr);
            if (lane == 0) {
                scratch[1 + warp] = bd.j;
                scratch[11 + warp] = bd.s;
            }
        }
    }
    constexpr int kStartBar = L::kThreads - 32;  // every warp but the tail warp
    named_bar_sync(4, kStartBar);
    if (!split_start && !args.eager_start && known > 0) {
        // segmented batches: boundaries ts0+1 .. ts0+known bracketed by the start
        if (warp < known) {
            const uint64_t t = ts0 + 1 + warp;
            uint64_t lo, hi;
            step_bracket(diag_of(t), diag_of(ts0), scratch[0], lo, hi);
            const boundary bd = find_boundary<K, SEG>(args, diag_of(t), lo, hi, scratch[10], 32,
                                                      nullptr);
            if (lane == 0) {
                scratch[1 + warp] = bd.j;
                scratch[11 + warp] = bd.s;
            }
        }
        named_bar_sync(4, kStartBar);
    }
    if (args.trace && tid == 0) args.trace[8 * c + 5] = globaltimer_ns();
    const uint64_t epoch = scratch[38];  // written by thread 0 before the start-up barriers
    if (warp == W_SCHED) {
        // ------------------------------------------------------ scheduler
        uint32_t n_rounds = 0, n_claims = 0, n_fallback = 0;
        unsigned long long t_search = 0;
        // at most `ahead` tiles co-ranked beyond the producer, in passes of at
        // most 8: the probes' sectors are then still in L2 when the tile's
        // windows are loaded (measured: 0.15 GB less DRAM reads on C4 with
        // the store hint below)
        const int maxcap = int(args.sched_cap);
        const uint32_t ahead = args.sched_ahead;
        // push descriptors {i0, j0, j1, i1, s0, s1} for tiles [t, t+k): lane g
        // supplies tile t+g's boundaries; waits for ring space.
        auto push = [&](uint64_t t, int k, boundary b0, boundary b1) {
            const uint32_t p = *pushed;
            while (p + uint32_t(k) > *issued + ahead) __nanosleep(1000);  // far ahead: no hurry
            if (lane < k) {
                uint64_t* d = desc + 8 * ((p + lane) % NB);
                d[0] = diag_of(t + lane);
                d[1] = b0.j;
                d[2] = b1.j;
                d[3] = diag_of(t + lane + 1);
                d[4] = b0.s;
                d[5] = b1.s;
            }
            __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                *pushed = p + uint32_t(k);
            }
            __syncwarp();
        };
        auto shfl_b = [](boundary x, int src) {
            return boundary{__shfl_sync(0xffffffffu, x.j, src), __shfl_sync(0xffffffffu, x.s, src)};
        };
        auto shfl_up_b = [](boundary x) {
            return boundary{__shfl_up_sync(0xffffffffu, x.j, 1),
                            __shfl_up_sync(0xffffffffu, x.s, 1)};
        };
        // co-rank and push every tile of chunk [ts, te) given its start
        // boundary bs.  Each pass co-ranks the next k boundaries (k = 1, 4, 8,
        // then 32: the first tiles are ready fast, later passes amortise
        // latency) in 32/k lane groups, each bracketed by the last known one.
        auto run_chunk = [&](uint64_t ts, uint64_t te, boundary bs, int known_inner) {
            uint64_t cur = ts;
            boundary bc = bs;
            if (known_inner > 0) {  // boundaries ts+1 .. ts+known_inner are in scratch
                const int k = known_inner;
                const int x = lane < k ? lane : k - 1;
                const boundary bb{scratch[1 + x], scratch[11 + x]};
                const boundary bp = shfl_up_b(bb);
                push(cur, k, lane == 0 ? bc : bp, bb);
                bc = shfl_b(bb, k - 1);
                cur += uint64_t(k);
            }
            int cap = known_inner > 0 ? maxcap : 1;
            while (cur < te) {
                int k = int(te - cur < uint64_t(cap) ? te - cur : uint64_t(cap));
                cap = cap == 1 ? 4 : (cap == 4 ? 8 : maxcap);
                const int P = pow2_group(k);
                const int g = lane / P;
                const uint64_t tb = cur + 1 + uint64_t(g < k ? g : k - 1);
                const uint64_t i = diag_of(tb);
                uint64_t lo, hi;
                step_bracket(i, diag_of(cur), bc.j, lo, hi);
                const unsigned long long t_s = args.trace ? globaltimer_ns() : 0;
                const boundary bd = find_boundary<K, SEG>(args, i, lo, hi, bc.s, P, &n_rounds);
                if (args.trace) t_search += globaltimer_ns() - t_s;
                // lane g <- boundary cur + 1 + g (the result of group g)
                const boundary bb = shfl_b(bd, (lane < k ? lane : k - 1) * P);
                const boundary bp = shfl_up_b(bb);
                push(cur, k, lane == 0 ? bc : bp, bb);
                bc = shfl_b(bb, k - 1);
                cur += uint64_t(k);
            }
        };

        if (te0 > ts0) run_chunk(ts0, te0, boundary{scratch[0], scratch[10]}, known);
        // dynamic tail [NS, NT): one tile per claim; its boundaries were
        // co-ranked in the background by the tail warps (slot q = boundary
        // NS + q), a slot not yet valid is co-ranked here instead.
        if (NS < NT) {
            bool tag_seen = false;  // lane 0: the tail counter carries this launch's tag
            for (;;) {
                while (*pushed - *issued >= args.lookahead) __nanosleep(500);
                uint64_t q = 0;
                if (lane == 0) {
                    q = tail_claim(args.tail, epoch, tag_seen);
                    if (q == NT - NS + G - 1)  // the launch's last claim: next launch, new epoch
                        atomicAdd(reinterpret_cast<unsigned long long*>(args.tail + 4), 1ull);
                }
                q = __shfl_sync(0xffffffffu, q, 0);
                if (NS + q >= NT) break;
                if (args.trace && lane == 0 && n_claims == 0)
                    args.trace[16 * 4096 + 4 * c + 2] = globaltimer_ns();  // first tail claim
                ++n_claims;
                // both boundaries' slots in one round trip: lane e (< 2) loads
                // slot q + e (the tile's start and end), the warp validates
                const uint64_t qq = q + uint64_t(lane & 1);
                boundary bd{m, SEGM ? args.nseg - 1 : 0};  // the last boundary is (m, n)
                bool ok = NS + qq == NT && out_end == total;
                if (!ok && lane < 2) {
                    const uint64_t* slot = args.tail + kTailSlots + 4 * qq;
                    uint64_t tag, pad;
                    ld_pair(slot, bd.j, bd.s);
                    ld_pair(slot + 2, tag, pad);
                    ok = tag == tail_hash(epoch, qq, bd.j, bd.s);
                }
                boundary bb[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    bb[e] = shfl_b(bd, e);
                    if (!__shfl_sync(0xffffffffu, ok, e)) {  // not published yet: co-rank here
                        if (args.trace && lane == 0) {
                            ++n_fallback;
                            args.trace[16 * 4096 + 4 * c + 3] = NS + q + e;  // the last one
                        }
                        const uint64_t i = diag_of(NS + q + e);
                        uint64_t lo, hi;
                        full_bracket(i, lo, hi);
                        bb[e] = shfl_b(find_boundary<K, SEG>(args, i, lo, hi, 0, 32, &n_rounds), 0);
                    }
                }
                push(NS + q, 1, bb[0], bb[1]);
            }
        }
        if (args.trace && lane == 0) {
            args.trace[8 * c + 1] = (uint64_t(n_claims) << 48) | (uint64_t(n_rounds) << 32) |
                                    (t_search / 1000);  // claims | rounds | search us
            args.trace[16 * 4096 + 4 * c] = n_fallback;  // tail slots co-ranked here
        }
        // end marker
        {
            const uint32_t p = *pushed;
            while (p + 1 > *issued + NB) __nanosleep(128);
            if (lane == 0) {
                desc[8 * (p % NB)] = ~uint64_t(0);
                __threadfence_block();
                *pushed = p + 1;
            }
        }
        return;
    }

    if (warp == W_STORE) {
        // ------------------------------------------------------ store warp
        // Stores each merged tile from its stage (one TMA bulk store of its
        // whole 16-byte blocks, plain word stores at misaligned ends:
        // store_window) and releases the stage to the producer once the store
        // has read it, so the consumer warps never wait on a store.
        if (lane != 0) return;
        uint32_t* __restrict__ outv = args.outv;
        const bool store_hint = args.store_evict_first != 0;
        const uint64_t spolicy = policy_evict_first();
        for (uint32_t s = 0;; ++s) {
            const int st = int(s % NST);
            mbar_wait_sleepy(&staged[st], uint32_t((s / NST) & 1), 2000);
            const uint64_t* mt = meta + 8 * st;
            if (mt[3] >> 63) break;  // end of work
            const uint64_t i0 = mt[0] - out_base;  // position in out
            const uint64_t lens = mt[2];
            const int len = int(lens >> 32) + int(lens & 0xffffffffu);
            unsigned char* stage = smem + L::oStages + size_t(st) * L::kStage;
            store_window(args.out, i0, len, uint32_t(sizeof(K)), stage, store_hint, spolicy);
            if constexpr (HAS_V)
                store_window(outv, i0, len, 4u, stage + L::kStageKeys, store_hint, spolicy);
            tma_store_commit();
            tma_store_wait_read<0>();  // the stage has been read by the store
            mbar_arrive(&empty[st]);
        }
        tma_store_wait_all();
        if (args.trace) args.trace[8 * 4096 + 4 * c + 3] = globaltimer_ns();  // stores drained
        return;
    }

    if (warp == W_PROD) {
        // ------------------------------------------------------ producer
        // lane 0 stages the windows; for segmented batches the whole warp also
        // writes the tile's segment-end table (the full barrier's 2nd arrival)
        if (!SEGM && lane != 0) return;
        const uint64_t policy = policy_evict_first();
        unsigned long long starve = 0;  // ns spent waiting for descriptors
        for (uint32_t s = 0;; ++s) {
            const int st = int(s % NST);
            if (s >= uint32_t(NST)) mbar_wait_sleepy(&empty[st], uint32_t((s / NST - 1) & 1), 1000);
            if (*pushed <= s) {
                const unsigned long long w0 = args.trace ? globaltimer_ns() : 0;
                while (*pushed <= s) __nanosleep(200);
                if (args.trace) {
                    const unsigned long long w = globaltimer_ns() - w0;
                    starve += w;
                    // trace region 3 (4 u64 per CTA): starved ns in the static
                    // range, in the dynamic tail, and the count of waits of each
                    unsigned long long* r3 = args.trace + 12 * 4096 + 4 * c;
                    const bool in_tail = uint64_t(s) >= te0 - ts0;
                    r3[in_tail ? 1 : 0] += w;
                    r3[in_tail ? 3 : 2] += 1;
                }
            }
            __threadfence_block();
            const uint64_t* d = desc + 8 * (s % NB);
            const uint64_t i0 = d[0];
            uint64_t* mt = meta + 8 * st;
            if (i0 == ~uint64_t(0)) {
                if (lane == 0) {
                    mt[3] = uint64_t(1) << 63;  // done
                    mbar_arrive(&full[st]);
                    if (SEGM) mbar_arrive(&full[st]);
                    if (args.trace) args.trace[8 * c + 6] = starve;
                }
                break;
            }
            // copy the whole descriptor out before its ring slot is released
            const uint64_t j0 = d[1], j1 = d[2], i1 = d[3], seg0 = d[4], seg1 = d[5];
            if constexpr (SEGM) __syncwarp();
            if (lane == 0) {
                __threadfence_block();
                *issued = s + 1;
            }
            if (lane == 0) {
#ifdef COMERGE_DEBUG_CHECKS
                if (!(j0 <= j1 && i0 <= i1 && i1 - i0 <= uint64_t(T) && i0 >= j0 && i1 >= j1 &&
                      i1 - j1 >= i0 - j0 && j1 <= m && i1 - j1 <= n && seg0 <= seg1 &&
                      (!SEGM || seg1 < args.nseg))) {
                    printf("comerge: bad tile descriptor cta %u s %u: i0 %llu i1 %llu j0 %llu j1 %llu "
                           "s0 %llu s1 %llu\n", c, s, (unsigned long long)i0, (unsigned long long)i1,
                           (unsigned long long)j0, (unsigned long long)j1,
                           (unsigned long long)seg0, (unsigned long long)seg1);
                    __trap();
                }
#endif
                mt[4] = seg0;
                mt[5] = seg1;
                const uint64_t k0 = i0 - j0, k1 = i1 - j1;
                const uint32_t a_len = uint32_t(j1 - j0), b_len = uint32_t(k1 - k0);
                unsigned char* stage = smem + L::oStages + size_t(st) * L::kStage;
                K* sk = reinterpret_cast<K*>(stage);
                uint32_t* sv = reinterpret_cast<uint32_t*>(stage + L::kStageKeys);
                unsigned char* svb = stage + L::kStageKeys;
                // window byte offsets in the stage: A's first element, B's
                // slot, B's first element (and the same for the payloads)
                uint32_t a_first, b_base, b_first, av_first = 0, bv_base = 0, bv_first = 0;
                uint32_t ab, bb, avb = 0, bvb = 0;
                win_plan pa{}, pb{}, pav{}, pbv{};
                if constexpr (SEG == 0 || SEG == 1) {
                    // one array per side, any 4-byte alignment: byte-space windows
                    pa = plan_window(a, m, sizeof(K), j0, j1, stage);
                    pb = plan_window(b, n, sizeof(K), k0, k1, stage + pa.span);
                    a_first = pa.first;
                    b_base = pa.span;
                    b_first = pb.first;
                    ab = pa.bytes;
                    bb = pb.bytes;
                    if constexpr (HAS_V) {
                        pav = plan_window(args.av, m, 4, j0, j1, svb);
                        pbv = plan_window(args.bv, n, 4, k0, k1, svb + pav.span);
                        av_first = pav.first;
                        bv_base = pav.span;
                        bv_first = pbv.first;
                        avb = pav.bytes;
                        bvb = pbv.bytes;
                    }
                } else {
                    // merge passes / pieced inputs: 16-byte aligned pieces, index space
                    const uint32_t ao = uint32_t(j0 % VECE);
                    const uint32_t bbe = (ao + a_len + VECE - 1) / VECE * VECE;
                    const uint32_t bo = uint32_t(k0 % VECE);
                    a_first = ao * uint32_t(sizeof(K));
                    b_base = bbe * uint32_t(sizeof(K));
                    b_first = bo * uint32_t(sizeof(K));
                    const uint64_t RL = SEG == 2 ? args.run_len : 0;  // merge pass (see pipe_args)
                    if constexpr (SEG == 3) {
                        ab = stage_pieces(args.pa, args.pa_start, args.npa, j0, j1, sk, VECE, false,
                                          nullptr, 0);
                        bb = stage_pieces(args.pb, args.pb_start, args.npb, k0, k1, sk + bbe, VECE,
                                          false, nullptr, 0);
                    } else {
                        ab = stage_runs(a, m + n, j0, j1, RL, 0, sk, VECE, false, nullptr, 0);
                        bb = stage_runs(b, m + n, k0, k1, RL, 1, sk + bbe, VECE, false, nullptr, 0);
                    }
                    if constexpr (HAS_V) {
                        const uint32_t avo = uint32_t(j0 % 4);
                        const uint32_t bvbe = (avo + a_len + 3) / 4 * 4;
                        av_first = avo * 4;
                        bv_base = bvbe * 4;
                        bv_first = uint32_t(k0 % 4) * 4;
                        if constexpr (SEG == 3) {
                            avb = stage_pieces(reinterpret_cast<const void* const*>(args.pav),
                                               args.pa_start, args.npa, j0, j1, sv, 4, false,
                                               nullptr, 0);
                            bvb = stage_pieces(reinterpret_cast<const void* const*>(args.pbv),
                                               args.pb_start, args.npb, k0, k1, sv + bvbe, 4, false,
                                               nullptr, 0);
                        } else {
                            avb = stage_runs(args.av, m + n, j0, j1, RL, 0, sv, 4, false, nullptr, 0);
                            bvb = stage_runs(args.bv, m + n, k0, k1, RL, 1, sv + bvbe, 4, false,
                                             nullptr, 0);
                        }
                    }
                }
                // the merged tile's placement: element 0 at the output
                // position's address offset modulo 16 (byte-space stores)
                const uint64_t opos = i0 - out_base;
                const uint32_t o_shift =
                    uint32_t((reinterpret_cast<uintptr_t>(args.out) + opos * sizeof(K)) & 15u);
                const uint32_t ov_shift =
                    HAS_V ? uint32_t((reinterpret_cast<uintptr_t>(args.outv) + opos * 4) & 15u) : 0u;
                mt[0] = i0;
                mt[1] = k0;
                mt[2] = (uint64_t(a_len) << 32) | b_len;
                mt[3] = uint64_t(a_first) | (uint64_t(b_first) << 8) | (uint64_t(b_base) << 16) |
                        (uint64_t(o_shift) << 40);
                mt[7] = uint64_t(av_first) | (uint64_t(bv_first) << 8) | (uint64_t(bv_base) << 16) |
                        (uint64_t(ov_shift) << 40);
                if constexpr (SEGM) mt[6] = seg1 - seg0 + 1 <= uint64_t(L::SEGCAP) ? 1 : 0;  // table?
                mbar_arrive_expect_tx(&full[st], ab + bb + avb + bvb);
                if constexpr (SEG == 0 || SEG == 1) {
                    if (ab) tma_load_1d(stage + pa.dst_off, pa.src, ab, &full[st], policy);
                    if (bb) tma_load_1d(stage + b_base + pb.dst_off, pb.src, bb, &full[st], policy);
                    if constexpr (HAS_V) {
                        if (avb) tma_load_1d(svb + pav.dst_off, pav.src, avb, &full[st], policy);
                        if (bvb)
                            tma_load_1d(svb + bv_base + pbv.dst_off, pbv.src, bvb, &full[st], policy);
                    }
                } else {
                    const uint32_t bbe = b_base / uint32_t(sizeof(K));
                    const uint64_t RL = SEG == 2 ? args.run_len : 0;
                    if constexpr (SEG == 3) {
                        stage_pieces(args.pa, args.pa_start, args.npa, j0, j1, sk, VECE, true,
                                     &full[st], policy);
                        stage_pieces(args.pb, args.pb_start, args.npb, k0, k1, sk + bbe, VECE, true,
                                     &full[st], policy);
                    } else {
                        stage_runs(a, m + n, j0, j1, RL, 0, sk, VECE, true, &full[st], policy);
                        stage_runs(b, m + n, k0, k1, RL, 1, sk + bbe, VECE, true, &full[st], policy);
                    }
                    if constexpr (HAS_V) {
                        const uint32_t bvbe = bv_base / 4;
                        if constexpr (SEG == 3) {
                            stage_pieces(reinterpret_cast<const void* const*>(args.pav),
                                         args.pa_start, args.npa, j0, j1, sv, 4, true, &full[st],
                                         policy);
                            stage_pieces(reinterpret_cast<const void* const*>(args.pbv),
                                         args.pb_start, args.npb, k0, k1, sv + bvbe, 4, true,
                                         &full[st], policy);
                        } else {
                            stage_runs(args.av, m + n, j0, j1, RL, 0, sv, 4, true, &full[st], policy);
                            stage_runs(args.bv, m + n, k0, k1, RL, 1, sv + bvbe, 4, true, &full[st],
                                       policy);
                        }
                    }
                }
            }
            // segmented: the segment-end table (merge_thread_segends), written by
            // the whole warp after lane 0 has issued the window loads (its
            // offset reads then overlap the loads; the stage's full barrier
            // waits for both)
            if constexpr (SEGM) {
                const uint64_t nse = seg1 - seg0 + 1;
                uint32_t* se = reinterpret_cast<uint32_t*>(smem + L::oStages + size_t(st) * L::kStage +
                                                           L::kStageKeys + L::kStageVals);
                if (nse <= uint64_t(L::SEGCAP)) {
                    const uint64_t k0 = i0 - j0, alen = j1 - j0, blen = (i1 - j1) - k0;
                    for (uint64_t q = lane; q < nse; q += 32) {
                        uint64_t ae, be;
                        if constexpr (SEG == 2) {
                            ae = run_off(seg0 + q + 1, args.run_len, m);
                            be = run_off(seg0 + q + 1, args.run_len, n);
                        } else {
                            ae = ldg_u64(args.aoff + seg0 + q + 1);
                            be = ldg_u64(args.boff + seg0 + q + 1);
                        }
                        const uint32_t x1 = ae > j0 ? uint32_t(ae - j0 < alen ? ae - j0 : alen) : 0u;
                        const uint32_t y1 = be > k0 ? uint32_t(be - k0 < blen ? be - k0 : blen) : 0u;
                        se[q] = x1 | (y1 << 16);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[st]);  // table written (release)
            }
        }
        return;
    }

    // ---------------------------------------------------------- consumers
    unsigned long long data_wait = 0;  // ns consumers waited for stage data
    unsigned long long ph[4] = {0, 0, 0, 0};  // trace: merge, barrier 1, staging+barrier 2, store
    for (uint32_t s = 0;; ++s) {
        const int st = int(s % NST);
        if (args.trace && tid == 0) {
            const unsigned long long w0 = globaltimer_ns();
            mbar_wait_sleepy(&full[st], uint32_t((s / NST) & 1), 500);
            data_wait += globaltimer_ns() - w0;
        }
        mbar_wait_sleepy(&full[st], uint32_t((s / NST) & 1), 500);
        const uint64_t* mt = meta + 8 * st;
        const uint64_t packed = mt[3];
        if (packed >> 63) {
            if (tid == 0) mbar_arrive(&staged[st]);  // the store warp sees the end marker
            break;
        }
        const uint64_t i0 = mt[0];
        const uint64_t lens = mt[2];
        const int a_len = int(lens >> 32), b_len = int(lens & 0xffffffffu);
        const int len = a_len + b_len;
        // byte offsets in the stage (producer): windows, output placement
        const uint32_t a_first = uint32_t(packed & 0xff), b_first = uint32_t((packed >> 8) & 0xff);
        const uint32_t b_base = uint32_t((packed >> 16) & 0xffffff);
        const uint32_t o_shift = uint32_t((packed >> 40) & 0xff);
        unsigned char* stage = smem + L::oStages + size_t(st) * L::kStage;
        unsigned char* svb = stage + L::kStageKeys;

        const int diag = min(tid * VT, len);
        K keys[VT];
        uint32_t src[VT];
        const unsigned long long p0 = args.trace && tid == 0 ? globaltimer_ns() : 0;
        const K* sA = reinterpret_cast<const K*>(stage + a_first);
        const K* sB = reinterpret_cast<const K*>(stage + b_base + b_first);
        if constexpr (SEGM) {
            const uint64_t k0 = mt[1];
            const uint64_t s_lo = mt[4], s_hi = mt[5];
            if (SEG == 2 && s_lo == s_hi) {  // merge pass, one segment: a plain merge
                merge_thread_lean<K, VT, HAS_V>(sA, a_len, sB, b_len, diag, keys, src);
            } else if (mt[6]) {  // the producer's segment-end table
                const uint32_t* se = reinterpret_cast<const uint32_t*>(stage + L::kStageKeys +
                                                                       L::kStageVals);
                const int nse = int(s_hi - s_lo) + 1;
                // tiles of many short segments (threads cross several segment
                // ends): the per-step segment test of merge_thread_segends;
                // otherwise the lean loop (a tile-uniform choice: no divergence)
                if (nse > L::kLeanSegs)
                    merge_thread_segends<K, VT, HAS_V>(sA, sB, diag, se, nse, keys, src);
                else
                    merge_thread_segends_lean<K, VT, HAS_V>(sA, sB, diag, se, nse, keys, src);
            } else if constexpr (!HAS_V) {
                const seg_offsets off{args.aoff, args.boff};
                merge_thread_seg<K, VT>(sA, a_len, sB, b_len, diag, i0, i0 - k0, k0, s_lo, s_hi,
                                        off, keys);
            } else {
                __trap();  // merge passes have at most a few segments per tile
            }
        } else {
            merge_thread_lean<K, VT, HAS_V>(sA, a_len, sB, b_len, diag, keys, src);
        }
        uint32_t ov_shift = 0;
        if constexpr (HAS_V) {  // source element address -> its payload
            const uint64_t pv = mt[7];
            ov_shift = uint32_t((pv >> 40) & 0xff);
            const uint32_t* sav = reinterpret_cast<const uint32_t*>(svb + (pv & 0xff));
            const uint32_t* sbv = reinterpret_cast<const uint32_t*>(
                svb + ((pv >> 16) & 0xffffff) + ((pv >> 8) & 0xff));
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
        const unsigned long long p1 = args.trace && tid == 0 ? globaltimer_ns() : 0;
        named_bar_sync(1, NC);  // every thread is done reading the windows
        const unsigned long long p2 = args.trace && tid == 0 ? globaltimer_ns() : 0;
        const int cnt = len - diag < VT ? len - diag : VT;
        // element x of the tile at stage + o_shift + x * sizeof(K) (store_window)
        const uint32_t ko = smem_addr(stage) + o_shift + uint32_t(tid * VT) * uint32_t(sizeof(K));
        const uint32_t vo = smem_addr(svb) + ov_shift + uint32_t(tid * VT) * 4u;
        if (cnt == VT) {  // every thread but a partial tile's last: no per-store test
#pragma unroll
            for (int v = 0; v < VT; ++v) {
                smem_io<K>::st(ko + uint32_t(v) * uint32_t(sizeof(K)), keys[v]);
                if constexpr (HAS_V) smem_io<uint32_t>::st(vo + uint32_t(v) * 4u, src[v]);
            }
        } else {
#pragma unroll
            for (int v = 0; v < VT; ++v)
                if (v < cnt) {
                    smem_io<K>::st(ko + uint32_t(v) * uint32_t(sizeof(K)), keys[v]);
                    if constexpr (HAS_V) smem_io<uint32_t>::st(vo + uint32_t(v) * 4u, src[v]);
                }
        }
        fence_proxy_async_smem();
        named_bar_sync(1, NC);
        const unsigned long long p3 = args.trace && tid == 0 ? globaltimer_ns() : 0;
        if (tid == 0) {
            mbar_arrive(&staged[st]);  // hand the tile to the store warp
            if (args.trace) {
                ph[0] += p1 - p0;
                ph[1] += p2 - p1;
                ph[2] += p3 - p2;
            }
        }
        if (args.trace && tid == 0 && s == 0) args.trace[8 * c + 2] = globaltimer_ns();
    }
    if (args.trace && tid == 0) {
        args.trace[8 * c + 3] = globaltimer_ns();
        args.trace[8 * c + 7] = data_wait;
        unsigned long long* ext = args.trace + 8 * 4096;  // phase sums, 4 per CTA
        for (int q = 0; q < 3; ++q) ext[4 * c + q] = ph[q];
    }
}

}  // namespace comerge_b200
