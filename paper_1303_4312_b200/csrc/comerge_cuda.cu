// comerge_cuda.cu -- C ABI (include/comerge_cuda.h) over the sm_100a merge
// kernels.  Host-side contract checks mirror the reference's exceptions
// (corank.hpp:67-79, merge.hpp:61-66, parallel.hpp:61-64, :185-186,
// :284-295) as status codes with the same message substrings.
#include <cuda_runtime.h>

#if defined(__x86_64__)
#include <immintrin.h>
#endif

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/comerge_cuda.h"
#include "merge_pipe.cuh"
#include "merge_small.cuh"
#include "merge_tile.cuh"
#include "sort.cuh"

using namespace comerge_b200;

namespace {

thread_local std::string g_error;
thread_local cudaEvent_t g_ev_before = nullptr, g_ev_after = nullptr;
thread_local int g_path = 0;  // 0 auto, 1 tile (v1), 3 tile pipeline, 4 small (one wave)
thread_local int g_last_path = 0;  // kernel of the last merge: 1 tile, 3 pipe, 4 segmented tile, 5-7 pipe modes
thread_local unsigned long long* g_trace = nullptr;  // debug: per-CTA timestamps
// tuning knobs of the tile pipeline (0 = default)
thread_local int g_tune_lookahead = 0, g_tune_static_pct = 0, g_tune_flags = 0;
thread_local int g_host_mode = 0;  // host buffers: 0 chunked pipeline, 1 zero-copy, 2 plain staging

// Per-device state: kernel attributes (the dynamic shared-memory opt-in is
// per device context), grid limits and the library's streams are cached per
// device, indexed by the caller's current device.
constexpr int kMaxDevices = 64;

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < kMaxDevices ? dev : 0;
}

int sm_count() {
    static std::once_flag once[kMaxDevices];
    static int n[kMaxDevices];
    const int dev = current_device();
    std::call_once(once[dev], [dev] {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n[dev] = v > 0 ? v : 148;
    });
    return n[dev];
}

// Persistent grid size for the tile-pipeline kernel (resident CTAs), with the
// kernel's shared-memory opt-in set once per device.
template <typename K, bool HAS_V, int SEG>
int pipe_grid_limit() {
    static std::once_flag once[kMaxDevices];
    static int limit[kMaxDevices];
    const int dev = current_device();
    std::call_once(once[dev], [dev] {
        using L = pipe_layout<K, HAS_V, SEG>;
        auto kern = merge_pipe_kernel<K, HAS_V, SEG>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(L::kSmem));
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::kThreads,
                                                          L::kSmem) != cudaSuccess ||
            per_sm < 1) {
            cudaGetLastError();
            per_sm = 1;
        }
        limit[dev] = per_sm * sm_count();
    });
    return limit[dev];
}

void mark_before(cudaStream_t s) {
    if (g_ev_before) cudaEventRecord(g_ev_before, s);
}
void mark_after(cudaStream_t s) {
    if (g_ev_after) cudaEventRecord(g_ev_after, s);
}

int fail(int code, const std::string& msg) {
    g_error = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    g_error = std::string(where) + ": " + cudaGetErrorString(e);
    return COMERGE_E_CUDA;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// merge.hpp:35-45 on byte ranges
bool overlaps(const void* x, size_t xbytes, const void* y, size_t ybytes) {
    if (xbytes == 0 || ybytes == 0) return false;
    const auto xb = reinterpret_cast<uintptr_t>(x), yb = reinterpret_cast<uintptr_t>(y);
    return xb < yb + ybytes && yb < xb + xbytes;
}

constexpr uint64_t kMaxTotal = uint64_t(1) << 40;  // tile ids fit a 1-D grid

uint64_t div_up(uint64_t x, uint64_t y) { return (x + y - 1) / y; }
size_t round256(size_t x) { return (x + 255) / 256 * 256; }

// Library-private stream-ordered pool (one per device) that keeps its memory
// across synchronisations, so per-call scratch costs no OS mapping.
cudaMemPool_t private_pool() {
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return nullptr;
    static std::once_flag once[64];
    std::call_once(once[dev], [dev] {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        cudaMemPool_t p = nullptr;
        if (cudaMemPoolCreate(&p, &props) == cudaSuccess) {
            uint64_t keep = UINT64_MAX;
            cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
            pools[dev] = p;
        } else {
            cudaGetLastError();
        }
    });
    return pools[dev];
}

cudaError_t pool_alloc(void** ptr, size_t bytes, cudaStream_t s) {
    cudaMemPool_t p = private_pool();
    return p ? cudaMallocFromPoolAsync(ptr, bytes, p, s) : cudaMallocAsync(ptr, bytes, s);
}

// 64-bit launch tag of the pipeline's tail state: unique per launch across
// every kernel instantiation of the process (never 0).
std::atomic<uint64_t> g_launches{0x5eed};
uint64_t next_tail_epoch() {
    uint64_t x = g_launches.fetch_add(1) + 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x ? x : 1;
}

// alignment slack of a caller workspace (see scratch::acquire)
constexpr size_t kWsSlack = 256;
size_t with_slack(size_t need) { return need ? need + kWsSlack : 0; }

// Stream-ordered scratch: caller workspace, or the private pool when ws == NULL.
struct scratch {
    void* ptr = nullptr;
    bool owned = false;
    cudaStream_t stream = nullptr;
    // A caller workspace may have any alignment: the scratch starts at its
    // first 256-byte boundary (the tail state is read with 128-bit atomics),
    // and the *_workspace_bytes queries include that slack (kWsSlack).
    int acquire(void* ws, size_t ws_bytes, size_t need, cudaStream_t s) {
        stream = s;
        if (need == 0) return COMERGE_OK;
        if (ws) {
            const uintptr_t p = reinterpret_cast<uintptr_t>(ws);
            const size_t pad = size_t((256 - (p & 255)) & 255);
            if (ws_bytes < pad || ws_bytes - pad < need)
                return fail(COMERGE_E_INVALID, "comerge: workspace too small (need " +
                                                   std::to_string(need + kWsSlack) + " bytes)");
            ptr = reinterpret_cast<void*>(p + pad);
            return COMERGE_OK;
        }
        const cudaError_t e = pool_alloc(&ptr, need, s);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: workspace allocation");
        owned = true;
        return COMERGE_OK;
    }
    ~scratch() {
        if (owned) cudaFreeAsync(ptr, stream);
    }
};

int check_launch(const char* where) {
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? COMERGE_OK : cuda_fail(e, where);
}

template <typename K>
size_t merge_ws_bytes(size_t m, size_t n) {
    if (m > SIZE_MAX - n) return 0;
    const uint64_t total = m + n;
    if (total == 0) return 0;
    // tile kernel: one co-rank per tile boundary; pipeline: tail counter + slots
    const size_t tile_ws = round256((div_up(total, tile_cfg<K>::kTile) + 1) * sizeof(uint64_t));
    // one 32-byte slot per pipeline tile covers any tail fraction
    constexpr uint64_t pt = pipe_layout<K, false>::T < pipe_layout<K, true>::T
                                ? pipe_layout<K, false>::T
                                : pipe_layout<K, true>::T;
    const size_t pipe_ws = round256(32 * (div_up(total, pt) + 4));
    return tile_ws > pipe_ws ? tile_ws : pipe_ws;
}

template <typename K>
size_t seg_ws_bytes(size_t total) {
    if (total == 0) return 0;
    const size_t tile_ws = 2 * round256((div_up(total, seg_cfg<K>::kTile) + 1) * sizeof(uint64_t));
    const size_t pipe_ws = round256(32 * (div_up(total, pipe_layout<K, false, 1>::T) + 4));
    return tile_ws > pipe_ws ? tile_ws : pipe_ws;
}

// Common contract of every merge entry (corank.hpp:67-70, merge.hpp:61-66).
template <typename K>
int check_merge_args(const char* who, const K* a, size_t m, const K* b, size_t n, const K* out,
                     const uint32_t* av, const uint32_t* bv, const uint32_t* outv, bool has_v) {
    if (m > SIZE_MAX - n)
        return fail(COMERGE_E_LENGTH, "comerge: combined input length exceeds index range");
    const uint64_t total = m + n;
    if (total > kMaxTotal)
        return fail(COMERGE_E_LENGTH, std::string(who) +
                                          ": combined input length exceeds the device index range");
    if ((m && !a) || (n && !b) || (total && !out))
        return fail(COMERGE_E_INVALID, std::string(who) + ": null data pointer");
    // any element offset into an allocation, but elements naturally aligned
    constexpr uintptr_t al = alignof(K) - 1;
    if ((m && (reinterpret_cast<uintptr_t>(a) & al)) || (n && (reinterpret_cast<uintptr_t>(b) & al)) ||
        (total && (reinterpret_cast<uintptr_t>(out) & al)) ||
        (has_v && ((m && (reinterpret_cast<uintptr_t>(av) & 3)) ||
                   (n && (reinterpret_cast<uintptr_t>(bv) & 3)) ||
                   (total && (reinterpret_cast<uintptr_t>(outv) & 3)))))
        return fail(COMERGE_E_INVALID, std::string(who) + ": arrays must be aligned to their element type");
    if (has_v && ((m && !av) || (n && !bv) || (total && !outv)))
        return fail(COMERGE_E_INVALID, std::string(who) + ": null payload pointer");
    const size_t ob = total * sizeof(K);
    if (overlaps(a, m * sizeof(K), out, ob) || overlaps(b, n * sizeof(K), out, ob))
        return fail(COMERGE_E_INVALID, std::string(who) + ": output must not alias an input");
    if (has_v) {
        const size_t vb = total * sizeof(uint32_t);
        if (overlaps(av, m * 4, outv, vb) || overlaps(bv, n * 4, outv, vb) ||
            overlaps(a, m * sizeof(K), outv, vb) || overlaps(b, n * sizeof(K), outv, vb) ||
            overlaps(av, m * 4, out, ob) || overlaps(bv, n * 4, out, ob) ||
            overlaps(out, ob, outv, vb))
            return fail(COMERGE_E_INVALID, std::string(who) + ": output must not alias an input");
    }
    return COMERGE_OK;
}

// Pieced inputs (SEG == 3) and output ranges for launch_pipe.
struct pipe_pieces {
    uint32_t na = 0, nb = 0;
    const void* pa[kMaxPieces] = {};
    const void* pb[kMaxPieces] = {};
    const uint32_t* pav[kMaxPieces] = {};
    const uint32_t* pbv[kMaxPieces] = {};
    uint64_t a_start[kMaxPieces + 1] = {};
    uint64_t b_start[kMaxPieces + 1] = {};
    uint64_t out_base = 0, out_end = 0;
};

// Launch the persistent tile pipeline (merge_pipe.cuh): a plain merge
// (SEG 0), a segmented batch (1: aoff/boff/nseg), a merge pass of the sort (2:
// run_len) or pieced inputs (3), over the whole output or pieces->[out_base,
// out_end).  Scratch: the dynamic-tail state.
template <typename K, bool HAS_V, int SEG>
int launch_pipe(const K* a, const uint32_t* av, uint64_t m, const K* b, const uint32_t* bv,
                uint64_t n, K* out, uint32_t* outv, const uint64_t* aoff, const uint64_t* boff,
                uint64_t nseg, void* ws, size_t ws_bytes, cudaStream_t s, uint64_t run_len = 0,
                const pipe_pieces* pieces = nullptr, bool pdl = false) {
    using PL = pipe_layout<K, HAS_V, SEG>;
    const uint64_t total = m + n;
    const uint64_t out_base = pieces ? pieces->out_base : 0;
    const uint64_t out_end = pieces ? pieces->out_end : total;
    const uint64_t ptiles = div_up(out_end - out_base, PL::T);
    if (ptiles == 0) return COMERGE_OK;
    if (SEG == 2 && (run_len == 0 || (run_len & (run_len - 1))))
        return fail(COMERGE_E_INVALID, "comerge: merge-pass run length must be a power of two");
    int limit = pipe_grid_limit<K, HAS_V, SEG>();
    if (limit > kMaxPipeGrid) limit = kMaxPipeGrid;
    const uint32_t grid = uint32_t(ptiles < uint64_t(limit) ? ptiles : uint64_t(limit));
    pipe_args args{};
    args.a = a;
    args.av = av;
    args.m = m;
    args.b = b;
    args.bv = bv;
    args.n = n;
    args.out = out;
    args.outv = outv;
    args.ntiles = ptiles;
    args.aoff = aoff;
    args.boff = boff;
    args.nseg = nseg;
    args.run_len = run_len;
    args.out_base = out_base;
    args.out_end = out_end;
    if (pieces) {
        args.npa = pieces->na;
        args.npb = pieces->nb;
        for (uint32_t q = 0; q < kMaxPieces; ++q) {
            args.pa[q] = pieces->pa[q];
            args.pb[q] = pieces->pb[q];
            args.pav[q] = pieces->pav[q];
            args.pbv[q] = pieces->pbv[q];
        }
        for (uint32_t q = 0; q <= kMaxPieces; ++q) {
            args.pa_start[q] = pieces->a_start[q];
            args.pb_start[q] = pieces->b_start[q];
        }
    }
    args.trace = g_trace;
    // equal static split of 70% of the tiles + a dynamic tail of 30%: the tail
    // absorbs the start-up skew (~10 us between the first and last CTA to
    // start streaming) and the ~25% spread of per-SM streaming rates (B200
    // GPCs differ).  (An earlier per-SM speed table learned from host-mapped
    // per-CTA reports cost 4 us of kernel completion on C2 for the mapped
    // writes, and bought nothing once the tail was 25-30%.)
    // (merge passes of the sort: 60% static measured 1.560 ms against 1.567 at
    // 70%, 1.582 at 50%, 1.576 at 80% for 2^26 int32 keys)
    const uint64_t static_pct =
        g_tune_static_pct > 0 ? uint64_t(g_tune_static_pct > 100 ? 100 : g_tune_static_pct)
                              : (SEG == 2 ? 60 : 70);
    // (a few tiles per CTA: nothing to balance, all static)
    const uint64_t tail_tiles =
        ptiles < 4ull * grid && g_tune_static_pct == 0 ? 0 : ptiles * (100 - static_pct) / 100;
    args.static_tiles = ptiles - tail_tiles;
    scratch sc;
    if (tail_tiles > 0) {
        if (int rc = sc.acquire(ws, ws_bytes, 32 * (tail_tiles + 4), s)) return rc;
        args.tail = static_cast<uint64_t*>(sc.ptr);
        args.epoch = next_tail_epoch();
    }
    args.lookahead = g_tune_lookahead > 0 ? uint32_t(g_tune_lookahead) : 2u;
    // tail units of 4 tiles but for the last 2 x grid tail tiles (single:
    // the end balance); flags bits 15-17 override the unit (1 = round 1's
    // one-tile claims)
    args.tail_unit = 4u;
    if (const uint32_t u = (uint32_t(g_tune_flags) >> 15) & 7u) args.tail_unit = u;
    args.tail_single = 2ull * grid;
    // small inputs: co-rank the first boundaries of every CTA concurrently
    // (their random probes hit L2; on large inputs they would contend in HBM)
    args.eager_start = total * sizeof(K) <= (size_t(32) << 20) ? 1u : 0u;
    // segmented batches: a boundary's segment search probes the (L2-resident)
    // offsets, so concurrent start-up searches are cheap there too
    if (SEG == 1 && !(g_tune_flags & 1024)) args.eager_start = 1u;
    args.flags = uint32_t(g_tune_flags);
    // scheduler look-ahead (see merge_pipe.cuh); experiment flags override:
    // bits 2-3 pass cap (1: 8, 2: 16, 3: 32), bits 4-7 look-ahead / 4,
    // bit 8 / bit 9 force the store hint on / off
    args.sched_cap = 8;
    args.sched_ahead = 8;
    // 64-bit keys: probes are a larger share of the traffic, and keeping the
    // streamed output out of L2's way keeps them resident until the load
    // (C4 1051 -> 1028 us); for 32-bit keys the hint costs more than it saves
    // (the output left dirty in L2 at kernel end is written back after it)
    args.store_evict_first = sizeof(typename key_of<K>::type) == 8 ? 1u : 0u;
    // merge passes of the sort: the next pass reads every output anyway, and
    // lines left dirty in L2 are written back during its start-up searches
    // (2^26 int32 keys 1.959 -> 1.923 ms, pairs 3.601 -> 3.550 ms)
    if (SEG == 2) args.store_evict_first = 1u;
    if (const uint32_t c = (uint32_t(g_tune_flags) >> 2) & 3u) args.sched_cap = 4u << c;
    if (const uint32_t a = (uint32_t(g_tune_flags) >> 4) & 15u) args.sched_ahead = 4u * a;
    if (args.sched_ahead < args.sched_cap) args.sched_ahead = args.sched_cap;
    if (g_tune_flags & 256) args.store_evict_first = 1;
    if (g_tune_flags & 512) args.store_evict_first = 0;
    g_last_path = SEG == 3 ? 7 : (SEG == 2 ? 6 : (SEG ? 5 : 3));
    mark_before(s);
    if (pdl) {
        // programmatic dependent launch: the grid may be scheduled while the
        // previous kernel on the stream drains; the kernel's first act is
        // griddepcontrol.wait (merge_pipe.cuh), so it reads nothing early
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(PL::kThreads);
        cfg.dynamicSmemBytes = PL::kSmem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, merge_pipe_kernel<K, HAS_V, SEG>, args);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: pipeline merge launch");
    } else {
        merge_pipe_kernel<K, HAS_V, SEG><<<grid, PL::kThreads, PL::kSmem, s>>>(args);
    }
    mark_after(s);
    return check_launch("comerge: pipeline merge launch");
}

// One-wave merge of small inputs (merge_small.cuh): one CTA per tile.
template <typename K, bool HAS_V>
int launch_small(const K* a, const uint32_t* av, uint64_t m, const K* b, const uint32_t* bv,
                 uint64_t n, K* out, uint32_t* outv, cudaStream_t s) {
    using SL = small_layout<K, HAS_V>;
    static std::once_flag once[kMaxDevices];
    const int dev = current_device();
    std::call_once(once[dev], [] {
        cudaFuncSetAttribute(merge_small_kernel<K, HAS_V>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(SL::kSmem));
    });
    const uint64_t ntiles = div_up(m + n, SL::T);
    small_args args{a, av, m, b, bv, n, out, outv, g_tune_flags & 4096 ? 0u : 1u,
                    g_tune_flags & 16384 ? 0u : uint32_t(SL::kStop), g_trace};
    g_last_path = 8;
    mark_before(s);
    merge_small_kernel<K, HAS_V><<<unsigned(ntiles), SL::kThreads, SL::kSmem, s>>>(args);
    mark_after(s);
    return check_launch("comerge: small merge launch");
}

// tiles up to which the one-wave small-merge kernel is used (auto path)
template <typename K, bool HAS_V>
uint64_t small_tiles_limit() {
    return 2ull * uint64_t(sm_count());
}

template <typename K, bool HAS_V>
int merge_device(const K* a, const uint32_t* av, size_t m, const K* b, const uint32_t* bv,
                 size_t n, K* out, uint32_t* outv, void* ws, size_t ws_bytes, cudaStream_t s) {
    const char* who = HAS_V ? "merge_pairs" : "merge_keys";
    if (int rc = check_merge_args<K>(who, a, m, b, n, out, av, bv, outv, HAS_V)) return rc;
    const uint64_t total = uint64_t(m) + n;
    if (total == 0) return COMERGE_OK;
    // the tile pipeline (any element offsets: byte-space windows) when there
    // are enough tiles to fill it; records always take it
    using PL = pipe_layout<K, HAS_V>;
    const uint64_t ptiles = div_up(total, PL::T);
    if (g_path == 4 || (g_path == 0 && ptiles <= small_tiles_limit<K, HAS_V>()))
        return launch_small<K, HAS_V>(a, av, m, b, bv, n, out, outv, s);
    if (is_rec<K>::value || g_path == 3 || g_path == 0)
        return launch_pipe<K, HAS_V, 0>(a, av, m, b, bv, n, out, outv, nullptr, nullptr, 0, ws,
                                            ws_bytes, s);
    if constexpr (is_rec<K>::value) {
        return COMERGE_OK;  // (unreachable: records always take the pipeline)
    } else {
        constexpr int T = tile_cfg<K>::kTile;
        const uint64_t ntiles = div_up(total, T);
        const uint64_t nbound = ntiles + 1;
        scratch sc;
        if (int rc = sc.acquire(ws, ws_bytes, merge_ws_bytes<K>(m, n), s)) return rc;
        uint64_t* bj = static_cast<uint64_t*>(sc.ptr);
        partition_kernel<K><<<unsigned(div_up(nbound, 256)), 256, 0, s>>>(a, m, b, n, T, nbound, bj);
        if (int rc = check_launch("comerge: partition launch")) return rc;
        int flags = 0;
        flags |= aligned16(a) ? kAAligned : 0;
        flags |= aligned16(b) ? kBAligned : 0;
        flags |= aligned16(out) ? kOutAligned : 0;
        flags |= aligned16(av) ? kAVAligned : 0;
        flags |= aligned16(bv) ? kBVAligned : 0;
        flags |= aligned16(outv) ? kOutVAligned : 0;
        g_last_path = 1;
        mark_before(s);
        merge_tile_kernel<K, HAS_V><<<unsigned(ntiles), tile_cfg<K>::kThreads, 0, s>>>(
            a, av, m, b, bv, n, out, outv, bj, flags);
        mark_after(s);
        return check_launch("comerge: merge launch");
    }
}

// Key-value records (records.cuh): the arrays' common alignment picks the
// instantiation (vector shared-memory accesses need it), then the pipeline.
template <typename KT, int S>
int records_align_class(const void* a, size_t m, const void* b, size_t n, const void* out) {
    uintptr_t x = 0;
    if (m) x |= reinterpret_cast<uintptr_t>(a);
    if (n) x |= reinterpret_cast<uintptr_t>(b);
    if (m + n) x |= reinterpret_cast<uintptr_t>(out);
    constexpr uintptr_t nat = S == 16 ? 8 : 4;  // the record struct's own alignment
    if (x & (nat - 1)) return 0;
    return (x & 15) == 0 ? 16 : ((x & 7) == 0 ? 8 : 4);
}

template <typename KT, int S>
int merge_records_device(const void* a, size_t m, const void* b, size_t n, void* out, void* ws,
                         size_t ws_bytes, cudaStream_t s) {
    const int A = records_align_class<KT, S>(a, m, b, n, out);
    if (A == 0)
        return fail(COMERGE_E_INVALID, "merge_records: arrays must be aligned to their record type");
    auto run = [&](auto tag) {
        using R = decltype(tag);
        return merge_device<R, false>(static_cast<const R*>(a), nullptr, m,
                                      static_cast<const R*>(b), nullptr, n, static_cast<R*>(out),
                                      nullptr, ws, ws_bytes, s);
    };
    if constexpr (S == 16) {
        return A >= 16 ? run(rec<KT, 16, 16>{}) : run(rec<KT, 16, 8>{});
    } else if constexpr (S == 12) {
        return run(rec<KT, 12, 4>{});
    } else {
        return A >= 8 ? run(rec<KT, 8, 8>{}) : run(rec<KT, 8, 4>{});
    }
}

template <typename KT, int S>
size_t records_ws_bytes(size_t m, size_t n) {
    if (m > SIZE_MAX - n || m + n == 0) return 0;
    return round256(32 * (div_up(m + n, pipe_layout<rec<KT, S, S == 12 ? 4 : 8>, false>::T) + 4));
}

// Output ranks [out_begin, out_end) of the stable merge of A and B, each
// given as up to kMaxPieces device arrays (a multi-GPU split: rank r passes
// every GPU's piece -- peer pointers over NVLink -- and its own output range;
// Algorithm 2 with one worker per GPU).
template <typename K, bool HAS_V>
int merge_pieces_device(const K* const* ap, const uint32_t* const* apv, const uint64_t* alen,
                        int na, const K* const* bp, const uint32_t* const* bpv,
                        const uint64_t* blen, int nb, uint64_t out_begin, uint64_t out_end,
                        K* out, uint32_t* outv, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (na < 1 || nb < 1 || na > kMaxPieces || nb > kMaxPieces || !ap || !bp || !alen || !blen ||
        (HAS_V && (!apv || !bpv)))
        return fail(COMERGE_E_INVALID, "merge_pieces: 1 to 8 pieces per input");
    // piece cuts keep every TMA copy 16-byte aligned (keys and payloads)
    constexpr uint64_t vece = HAS_V ? (16 / sizeof(K) > 4 ? 16 / sizeof(K) : 4) : 16 / sizeof(K);
    pipe_pieces pc;
    pc.na = uint32_t(na);
    pc.nb = uint32_t(nb);
    uint64_t len[2] = {0, 0};
    for (int side = 0; side < 2; ++side) {
        const int np = side ? nb : na;
        const K* const* kp = side ? bp : ap;
        const uint32_t* const* vp = side ? bpv : apv;
        const uint64_t* pl = side ? blen : alen;
        for (int q = 0; q < np; ++q) {
            if (pl[q] && (!kp[q] || !aligned16(kp[q]) || (HAS_V && (!vp[q] || !aligned16(vp[q])))))
                return fail(COMERGE_E_INVALID,
                            "merge_pieces: pieces must be 16-byte aligned device arrays");
            if (q + 1 < np && pl[q] % vece)
                return fail(COMERGE_E_INVALID, "merge_pieces: every piece but the last must be a "
                                               "multiple of 16 bytes (keys and payloads)");
            (side ? pc.pb : pc.pa)[q] = kp[q];
            if (HAS_V) (side ? pc.pbv : pc.pav)[q] = vp[q];
            (side ? pc.b_start : pc.a_start)[q] = len[side];
            len[side] += pl[q];
        }
        for (int q = np; q <= kMaxPieces; ++q) (side ? pc.b_start : pc.a_start)[q] = len[side];
    }
    const uint64_t m = len[0], n = len[1];
    if (out_begin > out_end || out_end > m + n)
        return fail(COMERGE_E_RANGE, "merge_pieces: output range exceeds m+n");
    if (out_end > out_begin &&
        (!out || !aligned16(out) || (HAS_V && (!outv || !aligned16(outv)))))
        return fail(COMERGE_E_INVALID, "merge_pieces: output must be a 16-byte aligned device array");
    pc.out_base = out_begin;
    pc.out_end = out_end;
    if (na == 1 && nb == 1)  // one array per side: the plain pipeline's range mode
        return launch_pipe<K, HAS_V, 0>(ap[0], HAS_V ? apv[0] : nullptr, m, bp[0],
                                        HAS_V ? bpv[0] : nullptr, n, out, outv, nullptr, nullptr, 0,
                                        ws, ws_bytes, s, 0, &pc);
    if constexpr (16 % sizeof(K) != 0) {  // pieced windows are index-space 16-byte copies
        return fail(COMERGE_E_INVALID, "merge_pieces: records of this size take one piece per input");
    } else {
        return launch_pipe<K, HAS_V, 3>(nullptr, nullptr, m, nullptr, nullptr, n, out, outv,
                                        nullptr, nullptr, 0, ws, ws_bytes, s, 0, &pc);
    }
}

template <typename K>
int merge_segmented_device(const K* a, const uint64_t* a_off, size_t m, const K* b,
                           const uint64_t* b_off, size_t n, size_t nseg, K* out, void* ws,
                           size_t ws_bytes, cudaStream_t s) {
    if (nseg == 0) {
        if (m || n) return fail(COMERGE_E_INVALID, "merge_segmented: no segments for nonempty input");
        return COMERGE_OK;
    }
    if (!a_off || !b_off) return fail(COMERGE_E_INVALID, "merge_segmented: null offsets");
    if (int rc = check_merge_args<K>("merge_segmented", a, m, b, n, out, nullptr, nullptr,
                                     nullptr, false))
        return rc;
    const uint64_t total = m + n;
    if (total == 0) return COMERGE_OK;
    using PL = pipe_layout<K, false>;
    if (g_path != 1 && (g_path == 3 || div_up(total, PL::T) >= 16))
        return launch_pipe<K, false, 1>(a, nullptr, m, b, nullptr, n, out, nullptr, a_off, b_off,
                                           nseg, ws, ws_bytes, s);
    constexpr int T = seg_cfg<K>::kTile;
    const uint64_t ntiles = div_up(total, T);
    const uint64_t nbound = ntiles + 1;
    scratch sc;
    if (int rc = sc.acquire(ws, ws_bytes, seg_ws_bytes<K>(total), s)) return rc;
    uint64_t* bj = static_cast<uint64_t*>(sc.ptr);
    uint64_t* bseg = bj + round256(nbound * sizeof(uint64_t)) / sizeof(uint64_t);
    seg_partition_kernel<K><<<unsigned(div_up(nbound, 256)), 256, 0, s>>>(
        a, a_off, b, b_off, nseg, total, T, nbound, bj, bseg);
    if (int rc = check_launch("comerge: segmented partition launch")) return rc;
    int flags = 0;
    flags |= aligned16(a) ? kAAligned : 0;
    flags |= aligned16(b) ? kBAligned : 0;
    flags |= aligned16(out) ? kOutAligned : 0;
    g_last_path = 4;
    mark_before(s);
    seg_merge_tile_kernel<K><<<unsigned(ntiles), seg_cfg<K>::kThreads, 0, s>>>(
        a, a_off, m, b, b_off, n, out, bj, bseg, flags);
    mark_after(s);
    return check_launch("comerge: segmented merge launch");
}

// merge_comparisons of every worker block (report bookkeeping, one thread each)
template <typename K>
__global__ void block_comparisons_kernel(const K* __restrict__ a, const K* __restrict__ b,
                                         const uint64_t* __restrict__ ranks,
                                         const uint64_t* __restrict__ js, uint64_t workers,
                                         uint64_t* __restrict__ out) {
    const uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= workers) return;
    out[r] = merge_comparisons(a, js[r], js[r + 1], b, ranks[r] - js[r], ranks[r + 1] - js[r + 1],
                               [](const K* p) { return ldg_elem(p); });
}

template <typename K>
int co_rank_batch_device(const uint64_t* ranks, size_t count, const K* a, size_t m, const K* b,
                         size_t n, uint64_t* out_j, uint32_t* out_it, uint32_t* out_cmp,
                         cudaStream_t s) {
    if (m > SIZE_MAX - n)
        return fail(COMERGE_E_LENGTH, "comerge: combined input length exceeds index range");
    if (count == 0) return COMERGE_OK;
    if (!ranks || !out_j || (m && !a) || (n && !b))
        return fail(COMERGE_E_INVALID, "co_rank: null pointer");
    co_rank_batch_kernel<K><<<unsigned(div_up(count, 128)), 128, 0, s>>>(ranks, count, a, m, b, n,
                                                                       out_j, out_it, out_cmp);
    return check_launch("comerge: co_rank launch");
}

// ------------------------------------------------ synchronous mirrors

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged;
}

// Pinned (page-locked) host memory: device-addressable under UVA, so kernels
// can read and write it directly over PCIe.
bool is_pinned_host(const void* p) {
    if (!p) return false;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return attr.type == cudaMemoryTypeHost && attr.devicePointer == p;
}

// the synchronous entry points' stream (per host thread and device)
cudaStream_t sync_stream() {
    thread_local cudaStream_t s[kMaxDevices] = {};
    const int dev = current_device();
    if (!s[dev]) cudaStreamCreateWithFlags(&s[dev], cudaStreamNonBlocking);
    return s[dev];
}

// Device view of a possibly-host array (copied in on `s` when host).
struct staged {
    void* dev = nullptr;
    bool owned = false;
    cudaStream_t s = nullptr;
    int in(const void* src, size_t bytes, cudaStream_t st, uint64_t* h2d) {
        s = st;
        if (bytes == 0 || src == nullptr) return COMERGE_OK;
        if (is_device_ptr(src)) {
            dev = const_cast<void*>(src);
            return COMERGE_OK;
        }
        cudaError_t e = pool_alloc(&dev, bytes, st);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: device staging allocation");
        owned = true;
        e = cudaMemcpyAsync(dev, src, bytes, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: host->device copy");
        if (h2d) *h2d += bytes;
        return COMERGE_OK;
    }
    int out_alloc(void* dst, size_t bytes, cudaStream_t st) {
        s = st;
        if (bytes == 0 || dst == nullptr) return COMERGE_OK;
        if (is_device_ptr(dst)) {
            dev = dst;
            return COMERGE_OK;
        }
        const cudaError_t e = pool_alloc(&dev, bytes, st);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: device staging allocation");
        owned = true;
        return COMERGE_OK;
    }
    int back(void* dst, size_t bytes, uint64_t* d2h) {
        if (!owned || bytes == 0) return COMERGE_OK;
        const cudaError_t e = cudaMemcpyAsync(dst, dev, bytes, cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: device->host copy");
        if (d2h) *d2h += bytes;
        return COMERGE_OK;
    }
    ~staged() {
        if (owned) cudaFreeAsync(dev, s);
    }
};

// parallel.hpp:60-67
int partition_output_impl(uint64_t total, uint64_t workers, uint64_t r, uint64_t* out) {
    if (workers == 0)
        return fail(COMERGE_E_INVALID, "partition_output: worker count must be positive");
    if (r > workers) return fail(COMERGE_E_INVALID, "partition_output: worker id out of range");
    *out = uint64_t((unsigned __int128)r * total / workers);
    return COMERGE_OK;
}

struct event_pair {
    cudaEvent_t a = nullptr, b = nullptr;
    event_pair() {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
    }
    ~event_pair() {
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    }
    uint64_t ns() const {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        return uint64_t(double(ms) * 1e6);
    }
};

// ---------------------------------------------------------------- host pipeline
//
// Host buffers: the output is cut into chunks whose input windows are found by
// co-ranking the chunk boundaries on the host (Algorithm 2 at the host level,
// each chunk is an independent stable merge of its two
// windows), and each chunk goes H2D -> merge on the device -> D2H on three
// streams, so host->device and device->host traffic overlap (PCIe is full
// duplex) while the device merges.  Nothing is merged on the host.
struct host_streams {
    cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
    cudaEvent_t in_done[3], merged[3], out_done[3];
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    host_streams() {
        cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking);
        for (int i = 0; i < 3; ++i) {
            cudaEventCreateWithFlags(&in_done[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&merged[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&out_done[i], cudaEventDisableTiming);
        }
        cudaEventCreate(&t0);
        cudaEventCreate(&t1);
    }
};

// ---- pageable host buffers.  The driver stages a copy from or to pageable
// memory synchronously (C4 e2e 467 ms against 69 ms from page-locked
// buffers), so the host pipeline copies pageable windows through page-locked
// staging slots itself: a pool of host threads copies a chunk's input windows
// into its slot (after the slot's previous H2D) and the chunk's merged
// output out of its slot (after its D2H), while the copy engines and the
// device work on the neighbouring chunks.

// Host copy between pageable memory and the page-locked staging slots with
// non-temporal stores (x86 AVX2, detected at run time; std::memcpy otherwise):
// the destination is read next by the DMA engine (H2D) or much later by the
// caller (D2H), so lines need not be read for ownership nor kept in cache --
// 8 threads copy 39 instead of 28 GB/s on the build host
// (tools/micro/memcpy_bw.cpp).
#if defined(__x86_64__) && defined(__GNUC__)
__attribute__((target("avx2"))) void stream_copy_avx2(char* d, const char* s, size_t n) {
    size_t i = 0;
    for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = s[i];
    for (; i + 128 <= n; i += 128) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 32));
        const __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 64));
        const __m256i e = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 96));
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 32), b);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 64), c);
        _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 96), e);
    }
    for (; i < n; ++i) d[i] = s[i];
    _mm_sfence();
}
inline void host_copy(void* dst, const void* src, size_t bytes) {
    static const bool avx2 = __builtin_cpu_supports("avx2") && !std::getenv("COMERGE_HOST_MEMCPY");
    if (avx2 && bytes >= (size_t(256) << 10))
        stream_copy_avx2(static_cast<char*>(dst), static_cast<const char*>(src), bytes);
    else
        std::memcpy(dst, src, bytes);
}
#else
inline void host_copy(void* dst, const void* src, size_t bytes) { std::memcpy(dst, src, bytes); }
#endif

// Chunks between a chunk's enqueue and its drain out of the staging slot
// (pageable outputs; 1 or 2 with three slots): 2 -- the drained chunk's D2H
// finished during the previous iteration, so the host never waits for it, and
// its slot is the next chunk's (lag 1 / lag 2 from pageable arrays: C2 13.3 /
// 12.7 ms, C3 39.9 / 33.2, C4 127.6 / 114.1, C5 11.3 / 9.8).
// COMERGE_HOST_LAG=1 restores the shorter lag (benchmarking).
inline uint64_t host_drain_lag(uint64_t) {
    static const char* e = std::getenv("COMERGE_HOST_LAG");
    return e && e[0] == '1' ? 1 : 2;
}

// The calling thread plus up to hardware_concurrency - 1 workers copy 2 MB
// pieces of one job at a time.
class copy_pool {
  public:
    static copy_pool& get() {
        static copy_pool pool;
        return pool;
    }
    void copy(void* dst, const void* src, size_t bytes) {
        constexpr size_t kPiece = size_t(2) << 20;
        if (bytes <= 2 * kPiece || workers_.empty()) {
            host_copy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> one(call_mu_);
        {
            std::lock_guard<std::mutex> lk(mu_);
            dst_ = static_cast<char*>(dst);
            src_ = static_cast<const char*>(src);
            bytes_ = bytes;
            next_.store(0);
            done_.store(0);
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return done_.load() == bytes_ && busy_ == 0; });
    }

  private:
    copy_pool() {
        const unsigned hc = std::thread::hardware_concurrency();
        const unsigned n = hc > 1 ? (hc < 16 ? hc : 16) - 1 : 0;
        for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this] { loop(); });
    }
    ~copy_pool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }
    void work() {
        constexpr size_t kPiece = size_t(2) << 20;
        for (;;) {
            const size_t o = next_.fetch_add(kPiece);
            if (o >= bytes_) break;
            const size_t len = bytes_ - o < kPiece ? bytes_ - o : kPiece;
            host_copy(dst_ + o, src_ + o, len);
            if (done_.fetch_add(len) + len == bytes_) {
                std::lock_guard<std::mutex> lk(mu_);
                done_cv_.notify_all();
            }
        }
    }
    void loop() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
                seen = gen_;
                ++busy_;
            }
            work();
            {
                std::lock_guard<std::mutex> lk(mu_);
                --busy_;
            }
            done_cv_.notify_all();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex mu_, call_mu_;
    std::condition_variable cv_, done_cv_;
    char* dst_ = nullptr;
    const char* src_ = nullptr;
    size_t bytes_ = 0;
    std::atomic<size_t> next_{0}, done_{0};
    uint64_t gen_ = 0;
    int busy_ = 0;
    bool stop_ = false;
};

// Page-locked staging for pageable host buffers (per host thread and device,
// grow-only: pinning costs ~80 ms per GB, once; at most 4 GB -- beyond it,
// or when pinning fails, the caller falls back to the driver's staging).
void* pinned_stage(size_t bytes) {
    if (bytes > (size_t(4) << 30)) return nullptr;
    struct cache {
        void* p = nullptr;
        size_t bytes = 0;
        ~cache() {
            if (p) cudaFreeHost(p);
        }
    };
    thread_local cache c[kMaxDevices];
    cache& x = c[current_device()];
    if (x.bytes < bytes) {
        if (x.p) cudaFreeHost(x.p);
        x.p = nullptr;
        x.bytes = 0;
        if (cudaHostAlloc(&x.p, bytes, cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            x.p = nullptr;
            return nullptr;
        }
        x.bytes = bytes;
    }
    return x.p;
}

host_streams& hstreams() {  // per host thread and device
    thread_local std::unique_ptr<host_streams> hs[kMaxDevices];
    const int dev = current_device();
    if (!hs[dev]) hs[dev].reset(new host_streams());
    return *hs[dev];
}

// Chunks of a host-buffer merge moving `bytes` each way: ~32 MB per chunk,
// 2 to 32 of them.  The first H2D and the last D2H run with the other
// direction idle (a chunk each), every chunk costs ~8 copy commands and a
// launch.  Measured e2e (tools/e2e_chunks.py): C1 (8.4 MB each way) 2 / 4 / 8
// chunks 0.33 / 0.35 / 0.38 ms; C2 (268 MB) 4 / 8 / 16 / 32 chunks 6.76 /
// 6.39 / 6.61 / 7.39 ms; C3 (1.07 GB) 8 / 32 / 64: 24.0 / 23.6 / 23.8 ms; C4
// (3.2 GB) 8 / 16 / 32 / 64 / 128: 71.8 / 69.4 / 68.8 / 70.0 / 72.9 ms
// (6.44 GB in 68.8 ms = 94 GB/s two-way, the link's measured ceiling).
uint64_t host_chunk_count(uint64_t bytes) {
    static const long knob = [] {
        const char* e = std::getenv("COMERGE_HOST_CHUNKS");  // tuning knob (benchmarking)
        return e ? std::atol(e) : 0L;
    }();
    if (knob > 0) return uint64_t(knob);
    return std::min<uint64_t>(32, std::max<uint64_t>(2, (bytes + (uint64_t(16) << 20)) >> 25));
}

template <typename K, bool HAS_V>
int merge_host_pipeline(const K* a, const uint32_t* av, uint64_t m, const K* b,
                        const uint32_t* bv, uint64_t n, K* out, uint32_t* outv, uint64_t* h2d,
                        uint64_t* d2h, uint64_t* merge_ns) {
    host_streams& hs = hstreams();
    const uint64_t total = m + n;
    // Copy granularity: every copy starts (and, but for an array's end, ends)
    // on a multiple of G elements = 256 bytes of 32-bit data.  Measured on C2's
    // shape (tools/micro/e2e_model2.cu): the same chunked copies take 6.1 ms
    // with 256-byte aligned windows and 7.2 ms with windows a few elements off.
    constexpr uint64_t G = 64;
    const uint64_t parts = host_chunk_count(total * (sizeof(K) + (HAS_V ? 4 : 0)));
    // `parts` equal chunks (weights); tried and not better: smaller first /
    // last chunks (a chunk's H2D overlaps the previous chunk's D2H, so the
    // bytes moved with one direction idle stay ~2x the largest chunk however
    // the sizes ramp), see DESIGN.md section 5
    std::vector<double> w(parts, 1.0);
    if (const char* ew = std::getenv("COMERGE_HOST_WEIGHTS")) {  // tuning knob (benchmarking)
        w.clear();
        for (const char* q = ew; *q;) {
            char* end = nullptr;
            const double x = std::strtod(q, &end);
            if (end == q) break;
            if (x > 0) w.push_back(x);
            q = *end ? end + 1 : end;
        }
        if (w.empty()) w.push_back(1.0);
    }
    double wsum = 0;
    for (double x : w) wsum += x;
    // chunks of at least 2^18 elements (small merges: fewer, equal chunks)
    const uint64_t min_chunk = uint64_t(1) << 18;
    if (double(total) * w.front() / wsum < double(min_chunk)) {
        const uint64_t k = std::max<uint64_t>(1, std::min<uint64_t>(parts, total / min_chunk));
        w.assign(k, 1.0);
        wsum = double(k);
    }
    std::vector<uint64_t> cuts(1, 0);
    double acc = 0;
    for (size_t q = 0; q < w.size(); ++q) {
        acc += w[q];
        const uint64_t c = q + 1 == w.size() ? total
                                            : std::min(total, uint64_t(double(total) * acc / wsum) / G * G);
        if (c > cuts.back()) cuts.push_back(c);
    }
    const uint64_t nchunks = cuts.size() - 1;
    uint64_t chunk = 0;
    for (uint64_t c = 0; c < nchunks; ++c) chunk = std::max(chunk, cuts[c + 1] - cuts[c]);
    // chunk boundaries: the Lemma-1 split of every chunk start, on host data,
    // each computed just before its chunk is enqueued (the host's cache-missing
    // probes then overlap the copies already running)
    std::vector<uint64_t> js(nchunks + 1);
    auto split = [&](uint64_t i) {
        return co_rank_split<K, uint64_t>(i, a, m, b, n, [](const K* p) { return *p; });
    };
    js[0] = 0;
    js[nchunks] = m;
    // three slots of device windows (A, B, out [+ payloads]) from the pool;
    // an input window is copied from its G-aligned start, so it holds up to
    // G - 1 leading elements of the previous chunk (+ G of end round-up)
    const uint64_t wcap = chunk + 2 * G;
    const size_t kb = round256(wcap * sizeof(K)), vb = HAS_V ? round256(wcap * 4) : 0;
    const size_t slot_bytes = 3 * (kb + vb);
    void* buf = nullptr;
    cudaError_t e = pool_alloc(&buf, 3 * slot_bytes, hs.comp);
    if (e != cudaSuccess) return cuda_fail(e, "comerge: host pipeline staging");
    cudaEventRecord(hs.in_done[0], hs.comp);  // allocation visible to the copy streams
    cudaStreamWaitEvent(hs.h2d, hs.in_done[0], 0);
    int rc = COMERGE_OK;
    // pageable arrays go through three page-locked slots (copy_pool): per
    // slot the input windows [A | B | A vals | B vals], then the chunk's
    // output [keys | vals]
    bool pg_a = m && !is_pinned_host(a), pg_b = n && !is_pinned_host(b);
    bool pg_av = HAS_V && m && !is_pinned_host(av), pg_bv = HAS_V && n && !is_pinned_host(bv);
    bool pg_o = !is_pinned_host(out), pg_ov = HAS_V && !is_pinned_host(outv);
    const size_t sin = (chunk + 4 * G) * (sizeof(K) + (HAS_V ? 4 : 0)) + 4 * 256;
    const size_t sok = round256(chunk * sizeof(K));
    const size_t sout = sok + (HAS_V ? round256(chunk * 4) : 0);
    unsigned char* pst = nullptr;
    if (pg_a || pg_b || pg_av || pg_bv || pg_o || pg_ov) {
        pst = static_cast<unsigned char*>(pinned_stage(3 * round256(sin + sout)));
        // no page-locked memory to spare: the driver's own (synchronous)
        // staging of pageable copies instead
        if (!pst) pg_a = pg_b = pg_av = pg_bv = pg_o = pg_ov = false;
    }
    const bool pg_out = pg_o || pg_ov;
    auto slot_in = [&](int sl) { return pst + size_t(sl) * round256(sin + sout); };
    auto copy_out = [&](uint64_t cc) {  // chunk cc's staged output -> the caller's arrays
        if (!pg_out) return;
        const cudaError_t ce = cudaEventSynchronize(hs.out_done[cc % 3]);
        if (ce != cudaSuccess) {
            if (!rc) rc = cuda_fail(ce, "comerge: host pipeline device->host copy");
            return;
        }
        const unsigned char* ob = slot_in(int(cc % 3)) + sin;
        const uint64_t len = cuts[cc + 1] - cuts[cc];
        if (pg_o) copy_pool::get().copy(out + cuts[cc], ob, len * sizeof(K));
        if (pg_ov) copy_pool::get().copy(outv + cuts[cc], ob + sok, len * 4);
    };
    bool first = true;
    // COMERGE_HOST_TRACE=1: per-chunk timeline on stderr (h2d start/end, merge
    // end, d2h end, us from the first copy) -- a benchmarking aid
    static const bool trace = std::getenv("COMERGE_HOST_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev(trace ? 4 * nchunks : 0);
    for (auto& ev : tev) cudaEventCreate(&ev);
    // One copy command per host array window.  The copy engines pair the two
    // directions' commands one for one, so the device->host side is cut into
    // about the same sizes in the same order as the host->device side (the
    // first |A window| outputs of a chunk, then the rest): 4 H2D + 4 matched
    // D2H commands per chunk measured 6.1 ms of copies on C2, 4 + 2 7.0 ms.
    auto h2d_copy = [&](void* dst, const void* src, size_t bytes) {
        if (!bytes || rc) return;
        const cudaError_t ce = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, hs.h2d);
        if (ce != cudaSuccess) rc = cuda_fail(ce, "comerge: host pipeline host->device copy");
    };
    auto d2h_copy = [&](void* dst, const void* src, size_t bytes) {
        if (!bytes || rc) return;
        const cudaError_t ce = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, hs.d2h);
        if (ce != cudaSuccess) rc = cuda_fail(ce, "comerge: host pipeline device->host copy");
    };
    const uint64_t lag = host_drain_lag(nchunks);
    for (uint64_t c = 0; c < nchunks && rc == COMERGE_OK; ++c) {
        const int sl = int(c % 3);
        unsigned char* base = static_cast<unsigned char*>(buf) + sl * slot_bytes;
        K* dA = reinterpret_cast<K*>(base);
        K* dB = reinterpret_cast<K*>(base + kb);
        K* dO = reinterpret_cast<K*>(base + 2 * kb);
        uint32_t* dAv = reinterpret_cast<uint32_t*>(base + 3 * kb);
        uint32_t* dBv = reinterpret_cast<uint32_t*>(base + 3 * kb + vb);
        uint32_t* dOv = reinterpret_cast<uint32_t*>(base + 3 * kb + 2 * vb);
        const uint64_t i0 = cuts[c], i1 = cuts[c + 1];
        if (c + 1 < nchunks) js[c + 1] = split(i1);
        const uint64_t j0 = js[c], j1 = js[c + 1], k0 = i0 - j0, k1 = i1 - j1;
        // aligned input windows A[sa, ea) ⊇ A[j0, j1), B[sb, eb) ⊇ B[k0, k1)
        const uint64_t sa = j0 / G * G, ea = std::min(m, div_up(j1, G) * G);
        const uint64_t sb = k0 / G * G, eb = std::min(n, div_up(k1, G) * G);
        if (c >= 3) cudaStreamWaitEvent(hs.h2d, hs.out_done[sl], 0);  // slot free again
        const void* srcA = a + sa;
        const void* srcB = b + sb;
        const void* srcAv = HAS_V ? static_cast<const void*>(av + sa) : nullptr;
        const void* srcBv = HAS_V ? static_cast<const void*>(bv + sb) : nullptr;
        if (pg_a || pg_b || pg_av || pg_bv) {
            // the slot's previous chunk has been copied to the device
            if (c >= 3) {
                const cudaError_t ce = cudaEventSynchronize(hs.in_done[sl]);
                if (ce != cudaSuccess) {
                    rc = cuda_fail(ce, "comerge: host pipeline host->device copy");
                    break;
                }
            }
            unsigned char* in = slot_in(sl);
            size_t off = 0;
            auto stage = [&](bool pg, const void*& src, size_t bytes) {
                if (!pg || !bytes) return;
                copy_pool::get().copy(in + off, src, bytes);
                src = in + off;
                off += round256(bytes);
            };
            stage(pg_a, srcA, (ea - sa) * sizeof(K));
            stage(pg_b, srcB, (eb - sb) * sizeof(K));
            if (HAS_V) {
                stage(pg_av, srcAv, (ea - sa) * 4);
                stage(pg_bv, srcBv, (eb - sb) * 4);
            }
        }
        if (trace) cudaEventRecord(tev[4 * c], hs.h2d);
        h2d_copy(dA, srcA, (ea - sa) * sizeof(K));
        if (HAS_V) h2d_copy(dAv, srcAv, (ea - sa) * 4);
        h2d_copy(dB, srcB, (eb - sb) * sizeof(K));
        if (HAS_V) h2d_copy(dBv, srcBv, (eb - sb) * 4);
        *h2d += (i1 - i0) * (sizeof(K) + (HAS_V ? 4 : 0));
        cudaEventRecord(hs.in_done[sl], hs.h2d);
        if (trace) cudaEventRecord(tev[4 * c + 1], hs.h2d);
        if (rc) break;
        cudaStreamWaitEvent(hs.comp, hs.in_done[sl], 0);
        if (first) {
            cudaEventRecord(hs.t0, hs.comp);
            first = false;
        }
        // the chunk is output ranks [(j0-sa)+(k0-sb), +(i1-i0)) of the merge
        // of A[sa, j1) and B[sb, k1): the leading elements precede every chunk
        // element in the stable order, so the range is exactly out[i0, i1)
        const K* pa[1] = {dA};
        const K* pb[1] = {dB};
        const uint32_t* pav[1] = {dAv};
        const uint32_t* pbv[1] = {dBv};
        const uint64_t la[1] = {j1 - sa}, lb[1] = {k1 - sb};
        const uint64_t r0 = (j0 - sa) + (k0 - sb);
        rc = merge_pieces_device<K, HAS_V>(pa, HAS_V ? pav : nullptr, la, 1, pb,
                                           HAS_V ? pbv : nullptr, lb, 1, r0, r0 + (i1 - i0), dO,
                                           HAS_V ? dOv : nullptr, nullptr, 0, hs.comp);
        cudaEventRecord(hs.merged[sl], hs.comp);
        if (trace) cudaEventRecord(tev[4 * c + 2], hs.comp);
        cudaStreamWaitEvent(hs.d2h, hs.merged[sl], 0);
        // out[i0, h) and out[h, i1): h on the G grid near the A window's share
        const uint64_t h = std::min(i1, i0 + (j1 - j0 + G / 2) / G * G) - i0;
        K* dstO = pg_o ? reinterpret_cast<K*>(slot_in(sl) + sin) : out + i0;
        uint32_t* dstOv = pg_ov ? reinterpret_cast<uint32_t*>(slot_in(sl) + sin + sok)
                                : (HAS_V ? outv + i0 : nullptr);
        d2h_copy(dstO, dO, h * sizeof(K));
        if (HAS_V) d2h_copy(dstOv, dOv, h * 4);
        d2h_copy(dstO + h, dO + h, (i1 - i0 - h) * sizeof(K));
        if (HAS_V) d2h_copy(dstOv + h, dOv + h, (i1 - i0 - h) * 4);
        *d2h += (i1 - i0) * (sizeof(K) + (HAS_V ? 4 : 0));
        cudaEventRecord(hs.out_done[sl], hs.d2h);
        if (trace) cudaEventRecord(tev[4 * c + 3], hs.d2h);
        // drain an earlier chunk while this chunk's copies and merge run
        // (host_drain_lag)
        if (c >= lag && !rc) copy_out(c - lag);
    }
    for (uint64_t q = std::min<uint64_t>(lag, nchunks); q >= 1 && !rc; --q) copy_out(nchunks - q);
    cudaEventRecord(hs.t1, hs.comp);
    cudaEventRecord(hs.in_done[0], hs.d2h);  // free the staging after the last copy-out
    cudaStreamWaitEvent(hs.comp, hs.in_done[0], 0);
    cudaFreeAsync(buf, hs.comp);
    e = cudaStreamSynchronize(hs.d2h);
    if (e == cudaSuccess) e = cudaStreamSynchronize(hs.comp);
    if (e != cudaSuccess) return cuda_fail(e, "comerge: host pipeline");
    if (trace) {
        for (uint64_t c = 0; c < nchunks; ++c) {
            float t[4];
            for (int q = 0; q < 4; ++q) cudaEventElapsedTime(&t[q], tev[0], tev[4 * c + q]);
            std::fprintf(stderr, "chunk %2llu  h2d %8.1f -> %8.1f  merged %8.1f  d2h done %8.1f us\n",
                         (unsigned long long)c, 1e3 * t[0], 1e3 * t[1], 1e3 * t[2], 1e3 * t[3]);
        }
        for (auto& ev : tev) cudaEventDestroy(ev);
    }
    if (rc) return rc;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, hs.t0, hs.t1);
    *merge_ns = uint64_t(double(ms) * 1e6);
    return COMERGE_OK;
}

// Chunk offsets of a segmented batch, rebased onto the chunk's windows:
// out_a[q] = clamp(a_off[s0 + q] - sa, 0, la) for q in [0, ns] (and b).
__global__ void rebase_offsets_kernel(const uint64_t* __restrict__ a_off,
                                      const uint64_t* __restrict__ b_off, uint64_t s0, uint64_t ns,
                                      uint64_t sa, uint64_t la, uint64_t sb, uint64_t lb,
                                      uint64_t* __restrict__ out_a, uint64_t* __restrict__ out_b) {
    const uint64_t q = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (q > ns) return;
    const uint64_t x = a_off[s0 + q], y = b_off[s0 + q];
    out_a[q] = x <= sa ? 0 : (x - sa < la ? x - sa : la);
    out_b[q] = y <= sb ? 0 : (y - sb < lb ? y - sb : lb);
}

// Host buffers, segmented batch (no reference counterpart: the reference's C5
// baseline is a loop of stable_merge, merge.hpp:52-68): the batch is one
// stable merge over (segment, key) composites, so it is cut into output
// chunks on the 256-byte grid exactly like merge_host_pipeline -- each cut
// co-ranked on the host (its segment by a binary search over the offsets, then
// the co-rank inside that segment) -- and each chunk is the output range
// [r0, r0 + len) of the segmented merge of its aligned windows, the segments
// it touches rebased onto them on the device.  H2D / merge / D2H overlap on
// three streams.  Requires offsets nondecreasing with a_off[nseg] <= m,
// b_off[nseg] <= n (checked).
template <typename K>
int merge_segmented_host_pipeline(const K* a, const uint64_t* a_off, uint64_t m, const K* b,
                                  const uint64_t* b_off, uint64_t n, uint64_t nseg, K* out,
                                  uint64_t* h2d, uint64_t* d2h, uint64_t* merge_ns) {
    host_streams& hs = hstreams();
    const uint64_t total = m + n;
    constexpr uint64_t G = 64;
    const uint64_t parts =
        std::max<uint64_t>(1, std::min<uint64_t>(host_chunk_count(total * sizeof(K)), total >> 18));
    std::vector<uint64_t> cuts(1, 0);
    for (uint64_t q = 1; q <= parts; ++q) {
        const uint64_t c = q == parts ? total : total * q / parts / G * G;
        if (c > cuts.back()) cuts.push_back(c);
    }
    const uint64_t nchunks = cuts.size() - 1;
    uint64_t chunk = 0;
    for (uint64_t c = 0; c < nchunks; ++c) chunk = std::max(chunk, cuts[c + 1] - cuts[c]);
    // composite co-rank of output rank i: (j, segment)
    auto seg_of = [&](uint64_t i) {  // largest s < nseg with a_off[s] + b_off[s] <= i
        uint64_t lo = 0, hi = nseg - 1;
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo + 1) / 2;
            if (a_off[mid] + b_off[mid] <= i)
                lo = mid;
            else
                hi = mid - 1;
        }
        return lo;
    };
    auto split = [&](uint64_t i, uint64_t& j, uint64_t& sg) {
        sg = seg_of(i);
        const uint64_t as = a_off[sg], bs = b_off[sg];
        const uint64_t li = i - as - bs;
        j = as + co_rank_split<K, uint64_t>(li, a + as, a_off[sg + 1] - as, b + bs,
                                            b_off[sg + 1] - bs, [](const K* p) { return *p; });
    };
    auto first_seg = [&](const uint64_t* off, uint64_t x) {  // a segment holding index x (or before)
        const uint64_t* p = std::upper_bound(off, off + nseg + 1, x);
        const uint64_t s = uint64_t(p - off);
        return s == 0 ? 0 : std::min<uint64_t>(s - 1, nseg - 1);
    };
    // device: the offsets once, then three slots of windows + rebased offsets
    const uint64_t wcap = chunk + 2 * G;
    const size_t kb = round256(wcap * sizeof(K)), ob = round256((nseg + 1) * 8);
    const size_t slot_bytes = 3 * kb + 2 * ob;
    void* buf = nullptr;
    cudaError_t e = pool_alloc(&buf, 2 * ob + 3 * slot_bytes, hs.comp);
    if (e != cudaSuccess) return cuda_fail(e, "comerge: segmented host pipeline staging");
    uint64_t* dAoff = static_cast<uint64_t*>(buf);
    uint64_t* dBoff = reinterpret_cast<uint64_t*>(static_cast<unsigned char*>(buf) + ob);
    unsigned char* slots = static_cast<unsigned char*>(buf) + 2 * ob;
    cudaEventRecord(hs.in_done[0], hs.comp);
    cudaStreamWaitEvent(hs.h2d, hs.in_done[0], 0);
    int rc = COMERGE_OK;
    auto h2d_copy = [&](void* dst, const void* src, size_t bytes) {
        if (!bytes || rc) return;
        const cudaError_t ce = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, hs.h2d);
        if (ce != cudaSuccess) rc = cuda_fail(ce, "comerge: host pipeline host->device copy");
    };
    auto d2h_copy = [&](void* dst, const void* src, size_t bytes) {
        if (!bytes || rc) return;
        const cudaError_t ce = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, hs.d2h);
        if (ce != cudaSuccess) rc = cuda_fail(ce, "comerge: host pipeline device->host copy");
    };
    h2d_copy(dAoff, a_off, (nseg + 1) * 8);
    h2d_copy(dBoff, b_off, (nseg + 1) * 8);
    // pageable key arrays through page-locked slots, as merge_host_pipeline
    bool pg_a = m && !is_pinned_host(a), pg_b = n && !is_pinned_host(b);
    bool pg_o = !is_pinned_host(out);
    const size_t sin = (chunk + 4 * G) * sizeof(K) + 2 * 256, sout = round256(chunk * sizeof(K));
    unsigned char* pst = nullptr;
    if (pg_a || pg_b || pg_o) {
        pst = static_cast<unsigned char*>(pinned_stage(3 * round256(sin + sout)));
        if (!pst) pg_a = pg_b = pg_o = false;  // the driver's own staging instead
    }
    auto slot_in = [&](int sl) { return pst + size_t(sl) * round256(sin + sout); };
    auto copy_out = [&](uint64_t cc) {
        if (!pg_o) return;
        const cudaError_t ce = cudaEventSynchronize(hs.out_done[cc % 3]);
        if (ce != cudaSuccess) {
            if (!rc) rc = cuda_fail(ce, "comerge: host pipeline device->host copy");
            return;
        }
        copy_pool::get().copy(out + cuts[cc], slot_in(int(cc % 3)) + sin,
                              (cuts[cc + 1] - cuts[cc]) * sizeof(K));
    };
    std::vector<uint64_t> js(nchunks + 1), ss(nchunks + 1);
    js[0] = 0;
    ss[0] = 0;
    bool first = true;
    const uint64_t lag = host_drain_lag(nchunks);
    for (uint64_t c = 0; c < nchunks && rc == COMERGE_OK; ++c) {
        const int sl = int(c % 3);
        unsigned char* base = slots + sl * slot_bytes;
        K* dA = reinterpret_cast<K*>(base);
        K* dB = reinterpret_cast<K*>(base + kb);
        K* dO = reinterpret_cast<K*>(base + 2 * kb);
        uint64_t* dAo = reinterpret_cast<uint64_t*>(base + 3 * kb);
        uint64_t* dBo = reinterpret_cast<uint64_t*>(base + 3 * kb + ob);
        const uint64_t i0 = cuts[c], i1 = cuts[c + 1];
        if (c + 1 < nchunks)
            split(i1, js[c + 1], ss[c + 1]);
        else
            js[c + 1] = m, ss[c + 1] = nseg - 1;
        const uint64_t j0 = js[c], j1 = js[c + 1], k0 = i0 - j0, k1 = i1 - j1;
        const uint64_t sa = j0 / G * G, ea = std::min(m, div_up(j1, G) * G);
        const uint64_t sb = k0 / G * G, eb = std::min(n, div_up(k1, G) * G);
        if (c >= 3) cudaStreamWaitEvent(hs.h2d, hs.out_done[sl], 0);
        const void* srcA = a + sa;
        const void* srcB = b + sb;
        if (pg_a || pg_b) {
            if (c >= 3) {  // the slot's previous chunk has been copied to the device
                const cudaError_t ce = cudaEventSynchronize(hs.in_done[sl]);
                if (ce != cudaSuccess) {
                    rc = cuda_fail(ce, "comerge: host pipeline host->device copy");
                    break;
                }
            }
            unsigned char* in = slot_in(sl);
            if (pg_a && ea > sa) {
                copy_pool::get().copy(in, srcA, (ea - sa) * sizeof(K));
                srcA = in;
            }
            if (pg_b && eb > sb) {
                unsigned char* inb = in + round256((ea - sa) * sizeof(K));
                copy_pool::get().copy(inb, srcB, (eb - sb) * sizeof(K));
                srcB = inb;
            }
        }
        h2d_copy(dA, srcA, (ea - sa) * sizeof(K));
        h2d_copy(dB, srcB, (eb - sb) * sizeof(K));
        *h2d += (i1 - i0) * sizeof(K);
        cudaEventRecord(hs.in_done[sl], hs.h2d);
        if (rc) break;
        cudaStreamWaitEvent(hs.comp, hs.in_done[sl], 0);
        if (first) {
            cudaEventRecord(hs.t0, hs.comp);
            first = false;
        }
        // the segments the windows touch, rebased onto them
        const uint64_t s_lo = std::min(first_seg(a_off, sa), first_seg(b_off, sb));
        const uint64_t s_hi = std::max(ss[c + 1], s_lo);
        const uint64_t ns = s_hi - s_lo + 1;
        const uint64_t la = j1 - sa, lb = k1 - sb;
        rebase_offsets_kernel<<<unsigned(div_up(ns + 1, 256)), 256, 0, hs.comp>>>(
            dAoff, dBoff, s_lo, ns, sa, la, sb, lb, dAo, dBo);
        if ((rc = check_launch("comerge: offsets rebase launch"))) break;
        pipe_pieces range;
        range.out_base = (j0 - sa) + (k0 - sb);
        range.out_end = range.out_base + (i1 - i0);
        rc = launch_pipe<K, false, 1>(dA, nullptr, la, dB, nullptr, lb, dO, nullptr, dAo, dBo, ns,
                                      nullptr, 0, hs.comp, 0, &range);
        cudaEventRecord(hs.merged[sl], hs.comp);
        cudaStreamWaitEvent(hs.d2h, hs.merged[sl], 0);
        const uint64_t h = std::min(i1, i0 + (j1 - j0 + G / 2) / G * G) - i0;
        K* dstO = pg_o ? reinterpret_cast<K*>(slot_in(sl) + sin) : out + i0;
        d2h_copy(dstO, dO, h * sizeof(K));
        d2h_copy(dstO + h, dO + h, (i1 - i0 - h) * sizeof(K));
        *d2h += (i1 - i0) * sizeof(K);
        cudaEventRecord(hs.out_done[sl], hs.d2h);
        if (c >= lag && !rc) copy_out(c - lag);  // as merge_host_pipeline
    }
    for (uint64_t q = std::min<uint64_t>(lag, nchunks); q >= 1 && !rc; --q) copy_out(nchunks - q);
    cudaEventRecord(hs.t1, hs.comp);
    cudaEventRecord(hs.in_done[0], hs.d2h);
    cudaStreamWaitEvent(hs.comp, hs.in_done[0], 0);
    cudaFreeAsync(buf, hs.comp);
    e = cudaStreamSynchronize(hs.d2h);
    if (e == cudaSuccess) e = cudaStreamSynchronize(hs.comp);
    if (e != cudaSuccess) return cuda_fail(e, "comerge: segmented host pipeline");
    if (rc) return rc;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, hs.t0, hs.t1);
    *merge_ns = uint64_t(double(ms) * 1e6);
    return COMERGE_OK;
}

// comerge_merge_segmented_host_*: host (or device) buffers, synchronous
template <typename K>
int merge_segmented_sync(const K* a, const uint64_t* a_off, size_t m, const K* b,
                         const uint64_t* b_off, size_t n, size_t nseg, K* out, size_t out_len,
                         comerge_merge_report* rep) {
    if (m > SIZE_MAX - n)
        return fail(COMERGE_E_LENGTH, "comerge: combined input length exceeds index range");
    if (out_len != m + n)
        return fail(COMERGE_E_INVALID, "merge_segmented: output length must equal |a| + |b|");
    if (int rc = check_merge_args<K>("merge_segmented", a, m, b, n, out, nullptr, nullptr, nullptr,
                                     false))
        return rc;
    const uint64_t total = uint64_t(m) + n;
    if (nseg == 0) {
        if (total) return fail(COMERGE_E_INVALID, "merge_segmented: no segments for nonempty input");
        if (rep) *rep = comerge_merge_report{};
        return COMERGE_OK;
    }
    if (!a_off || !b_off) return fail(COMERGE_E_INVALID, "merge_segmented: null offsets");
    const bool dev_off = is_device_ptr(a_off) || is_device_ptr(b_off);
    std::vector<uint64_t> ha, hb;
    const uint64_t* pa = a_off;
    const uint64_t* pb = b_off;
    if (dev_off) {  // offsets on the device: a host copy for the checks and cuts
        ha.resize(nseg + 1);
        hb.resize(nseg + 1);
        cudaError_t e = cudaMemcpy(ha.data(), a_off, (nseg + 1) * 8, cudaMemcpyDefault);
        if (e == cudaSuccess) e = cudaMemcpy(hb.data(), b_off, (nseg + 1) * 8, cudaMemcpyDefault);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: segment offsets copy");
        pa = ha.data();
        pb = hb.data();
    }
    for (size_t q = 0; q < nseg; ++q)
        if (pa[q] > pa[q + 1] || pb[q] > pb[q + 1])
            return fail(COMERGE_E_INVALID, "merge_segmented: offsets must be nondecreasing");
    if (pa[nseg] > m || pb[nseg] > n || pa[0] != 0 || pb[0] != 0)
        return fail(COMERGE_E_INVALID,
                    "merge_segmented: offsets must start at 0 and end within the inputs");
    const bool all_host = total >= (uint64_t(1) << 20) && !dev_off && !is_device_ptr(a) &&
                          !is_device_ptr(b) && !is_device_ptr(out) && pa[nseg] == m &&
                          pb[nseg] == n;
    if (all_host) {
        const auto w0 = std::chrono::steady_clock::now();
        uint64_t h2d = 0, d2h = 0, merge_ns = 0;
        if (int rc = merge_segmented_host_pipeline<K>(a, pa, m, b, pb, n, nseg, out, &h2d, &d2h,
                                                      &merge_ns))
            return rc;
        const auto w1 = std::chrono::steady_clock::now();
        if (rep) {
            *rep = comerge_merge_report{};
            rep->m = m;
            rep->n = n;
            rep->workers = 1;
            rep->wall_ns = merge_ns;
            rep->e2e_ns = uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(w1 - w0).count());
            rep->h2d_bytes = h2d;
            rep->d2h_bytes = d2h;
            rep->tiles = div_up(total, pipe_layout<K, false, 1>::T);
        }
        return COMERGE_OK;
    }
    // small or mixed: stage, merge on the device, copy back
    cudaStream_t s = sync_stream();
    event_pair e2e, dv;
    uint64_t h2d = 0, d2h = 0;
    cudaEventRecord(e2e.a, s);
    {
        staged da, db, dao, dbo, dout;
        int rc;
        if ((rc = da.in(a, m * sizeof(K), s, &h2d))) return rc;
        if ((rc = db.in(b, n * sizeof(K), s, &h2d))) return rc;
        if ((rc = dao.in(a_off, (nseg + 1) * 8, s, &h2d))) return rc;
        if ((rc = dbo.in(b_off, (nseg + 1) * 8, s, &h2d))) return rc;
        if ((rc = dout.out_alloc(out, total * sizeof(K), s))) return rc;
        cudaEventRecord(dv.a, s);
        if ((rc = merge_segmented_device<K>(static_cast<const K*>(da.dev),
                                            static_cast<const uint64_t*>(dao.dev), m,
                                            static_cast<const K*>(db.dev),
                                            static_cast<const uint64_t*>(dbo.dev), n, nseg,
                                            static_cast<K*>(dout.dev), nullptr, 0, s)))
            return rc;
        cudaEventRecord(dv.b, s);
        if ((rc = dout.back(out, total * sizeof(K), &d2h))) return rc;
        cudaEventRecord(e2e.b, s);
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: merge_segmented");
    }
    if (rep) {
        *rep = comerge_merge_report{};
        rep->m = m;
        rep->n = n;
        rep->workers = 1;
        rep->wall_ns = total ? dv.ns() : 0;
        rep->e2e_ns = e2e.ns();
        rep->h2d_bytes = h2d;
        rep->d2h_bytes = d2h;
        rep->tiles = div_up(total, pipe_layout<K, false, 1>::T);
    }
    return COMERGE_OK;
}

// The reference's merge_report bookkeeping (parallel.hpp:262-281) from the
// co-ranks of every worker-block boundary r = 0..workers: block sizes, the
// co_rank_stats iterations (begin and end per worker; synced: begin only,
// :269-275) and, when counting, the total comparisons -- every co-rank's
// (Algorithm 1's own count) plus every block's merge_into (merge_comparisons,
// corank.cuh: exact, no counted merge needed).
struct block_report {
    std::vector<uint64_t> ranks, js, merge_cmps;
    std::vector<uint32_t> its, cmps;
    void emit(size_t workers, int synced, uint64_t* block_sizes, uint32_t* iters,
              uint64_t* comparisons) const {
        if (block_sizes)
            for (size_t r = 0; r < workers; ++r) block_sizes[r] = ranks[r + 1] - ranks[r];
        if (iters) {
            for (size_t r = 0; r < workers; ++r) {
                if (synced) {
                    iters[r] = its[r];
                } else {
                    iters[2 * r] = its[r];
                    iters[2 * r + 1] = its[r + 1];
                }
            }
        }
        if (comparisons) {
            uint64_t total = 0;
            for (size_t r = 0; r < workers; ++r)
                total += cmps[r] + (synced ? 0 : cmps[r + 1]) + merge_cmps[r];
            *comparisons = total;
        }
    }
};

// ... with Algorithm 1 over host-resident inputs
template <typename K>
void host_block_report(const K* a, size_t m, const K* b, size_t n, size_t workers, bool count,
                       block_report& br) {
    const uint64_t total = uint64_t(m) + n;
    br.ranks.resize(workers + 1);
    br.js.resize(workers + 1);
    br.its.resize(workers + 1);
    br.cmps.resize(workers + 1);
    auto rd = [](const K* p) { return *p; };
    for (size_t r = 0; r <= workers; ++r) {
        partition_output_impl(total, workers, r, &br.ranks[r]);
        corank_stats st{};
        br.js[r] = co_rank_alg1(br.ranks[r], a, m, b, n, rd, &st);
        br.its[r] = st.iterations;
        br.cmps[r] = st.comparisons;
    }
    if (count) {
        br.merge_cmps.resize(workers);
        for (size_t r = 0; r < workers; ++r)
            br.merge_cmps[r] = merge_comparisons(a, br.js[r], br.js[r + 1], b,
                                                 br.ranks[r] - br.js[r],
                                                 br.ranks[r + 1] - br.js[r + 1], rd);
    }
}

template <typename K, bool HAS_V>
int merge_parallel_sync(const K* a, const uint32_t* av, size_t m, const K* b, const uint32_t* bv,
                        size_t n, K* out, uint32_t* outv, size_t out_len, size_t workers,
                        int synced, comerge_merge_report* rep, uint64_t* block_sizes,
                        uint32_t* corank_iterations, uint64_t* comparisons = nullptr) {
    const char* who = synced ? "merge_parallel_synced" : "merge_parallel";
    // checked_output (parallel.hpp:284-295), then workers (:185-186)
    if (m > SIZE_MAX - n)
        return fail(COMERGE_E_LENGTH, "comerge: combined input length exceeds index range");
    if (out_len != m + n)
        return fail(COMERGE_E_INVALID, std::string(who) + ": output length must equal |a| + |b|");
    if (overlaps(a, m * sizeof(K), out, out_len * sizeof(K)) ||
        overlaps(b, n * sizeof(K), out, out_len * sizeof(K)))
        return fail(COMERGE_E_INVALID, std::string(who) + ": output must not alias an input");
    if (HAS_V) {  // the payload arrays, as check_merge_args (every path below)
        const size_t ob = out_len * sizeof(K), vb = out_len * sizeof(uint32_t);
        if (overlaps(av, m * 4, outv, vb) || overlaps(bv, n * 4, outv, vb) ||
            overlaps(a, m * sizeof(K), outv, vb) || overlaps(b, n * sizeof(K), outv, vb) ||
            overlaps(av, m * 4, out, ob) || overlaps(bv, n * 4, out, ob) || overlaps(out, ob, outv, vb))
            return fail(COMERGE_E_INVALID, std::string(who) + ": output must not alias an input");
    }
    if (workers == 0)
        return fail(COMERGE_E_INVALID, "merge_parallel: worker count must be positive");
    const uint64_t total = m + n;
    // opt-in zero-copy for pinned host (or device) buffers: the merge kernel
    // loads its tile windows from and stores its tiles to host memory over
    // PCIe (measured ~36 GB/s per direction on B200 PCIe Gen5 x16, below the
    // copy engines' ~50, so the chunked pipeline below is the default)
    auto pinned_or_dev = [](const void* p, size_t bytes) {
        return bytes == 0 || is_pinned_host(p) || is_device_ptr(p);
    };
    const bool any_host = !is_device_ptr(a) || !is_device_ptr(b) || !is_device_ptr(out);
    const bool host_in = !is_device_ptr(a) && !is_device_ptr(b);
    if (total >= (uint64_t(1) << 20) && any_host && host_in && g_host_mode == 1 &&
        pinned_or_dev(a, m * sizeof(K)) && pinned_or_dev(b, n * sizeof(K)) &&
        pinned_or_dev(out, total * sizeof(K)) &&
        (!HAS_V || (pinned_or_dev(av, m * 4) && pinned_or_dev(bv, n * 4) &&
                    pinned_or_dev(outv, total * 4)))) {
        cudaStream_t s = sync_stream();
        event_pair e2e;
        cudaEventRecord(e2e.a, s);
        if (int rc = merge_device<K, HAS_V>(a, av, m, b, bv, n, out, outv, nullptr, 0, s)) return rc;
        cudaEventRecord(e2e.b, s);
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: zero-copy merge");
        block_report br;
        host_block_report(a, m, b, n, workers, comparisons != nullptr, br);
        br.emit(workers, synced, block_sizes, corank_iterations, comparisons);
        if (rep) {
            const uint64_t eb = sizeof(K) + (HAS_V ? 4 : 0);
            rep->m = m;
            rep->n = n;
            rep->workers = workers;
            rep->wall_ns = e2e.ns();
            rep->e2e_ns = e2e.ns();
            rep->h2d_bytes = (is_device_ptr(a) ? 0 : m * eb) + (is_device_ptr(b) ? 0 : n * eb);
            rep->d2h_bytes = is_device_ptr(out) ? 0 : total * eb;
            rep->tiles = div_up(total, pipe_layout<K, HAS_V>::T);
        }
        return COMERGE_OK;
    }
    // all-host buffers: chunked, overlapped H2D / merge / D2H pipeline
    const bool all_host = total >= (uint64_t(1) << 20) && g_host_mode == 0 && !is_device_ptr(a) && !is_device_ptr(b) &&
                          !is_device_ptr(out) &&
                          (!HAS_V || (!is_device_ptr(av) && !is_device_ptr(bv) && !is_device_ptr(outv)));
    if (all_host && (m == 0 || a) && (n == 0 || b) && (!HAS_V || ((m == 0 || av) && (n == 0 || bv) && outv))) {
        const auto w0 = std::chrono::steady_clock::now();
        uint64_t h2d = 0, d2h = 0, merge_ns = 0;
        if (int rc = merge_host_pipeline<K, HAS_V>(a, av, m, b, bv, n, out, outv, &h2d, &d2h,
                                                   &merge_ns))
            return rc;
        const auto w1 = std::chrono::steady_clock::now();
        block_report br;  // Algorithm 1 over the host-resident inputs (bookkeeping only)
        host_block_report(a, m, b, n, workers, comparisons != nullptr, br);
        br.emit(workers, synced, block_sizes, corank_iterations, comparisons);
        if (rep) {
            rep->m = m;
            rep->n = n;
            rep->workers = workers;
            rep->wall_ns = merge_ns;
            rep->e2e_ns = uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(w1 - w0).count());
            rep->h2d_bytes = h2d;
            rep->d2h_bytes = d2h;
            rep->tiles = div_up(total, pipe_layout<K, HAS_V>::T);
        }
        return COMERGE_OK;
    }
    cudaStream_t s = sync_stream();
    event_pair e2e, dev;
    uint64_t h2d = 0, d2h = 0;
    cudaEventRecord(e2e.a, s);
    int rc = COMERGE_OK;
    {
        staged da, db, dav, dbv, dout, doutv;
        if ((rc = da.in(a, m * sizeof(K), s, &h2d))) return rc;
        if ((rc = db.in(b, n * sizeof(K), s, &h2d))) return rc;
        if (HAS_V) {
            if ((rc = dav.in(av, m * 4, s, &h2d))) return rc;
            if ((rc = dbv.in(bv, n * 4, s, &h2d))) return rc;
            if ((rc = doutv.out_alloc(outv, total * 4, s))) return rc;
        }
        if ((rc = dout.out_alloc(out, total * sizeof(K), s))) return rc;
        cudaEventRecord(dev.a, s);
        rc = merge_device<K, HAS_V>(static_cast<const K*>(da.dev),
                                    static_cast<const uint32_t*>(dav.dev), m,
                                    static_cast<const K*>(db.dev),
                                    static_cast<const uint32_t*>(dbv.dev), n,
                                    static_cast<K*>(dout.dev), static_cast<uint32_t*>(doutv.dev),
                                    nullptr, 0, s);
        if (rc) return rc;
        cudaEventRecord(dev.b, s);
        // report: co-rank every reference worker-block boundary with
        // Algorithm 1 on the device (parallel.hpp:201-207, :273-275)
        const size_t nq = workers + 1;
        block_report br;
        br.ranks.resize(nq);
        br.js.resize(nq);
        br.its.resize(nq);
        br.cmps.resize(nq);
        for (size_t r = 0; r <= workers; ++r) partition_output_impl(total, workers, r, &br.ranks[r]);
        const bool count = comparisons != nullptr;
        if (corank_iterations || count) {
            staged dr, dj, dit, dcmp, dmc;
            if ((rc = dr.in(br.ranks.data(), nq * 8, s, nullptr))) return rc;
            if ((rc = dj.out_alloc(br.js.data(), nq * 8, s))) return rc;
            if ((rc = dit.out_alloc(br.its.data(), nq * 4, s))) return rc;
            if ((rc = dcmp.out_alloc(br.cmps.data(), nq * 4, s))) return rc;
            if ((rc = co_rank_batch_device<K>(static_cast<const uint64_t*>(dr.dev), nq,
                                              static_cast<const K*>(da.dev), m,
                                              static_cast<const K*>(db.dev), n,
                                              static_cast<uint64_t*>(dj.dev),
                                              static_cast<uint32_t*>(dit.dev),
                                              static_cast<uint32_t*>(dcmp.dev), s)))
                return rc;
            if (count) {
                br.merge_cmps.resize(workers);
                if ((rc = dmc.out_alloc(br.merge_cmps.data(), workers * 8, s))) return rc;
                block_comparisons_kernel<K><<<unsigned(div_up(workers, 128)), 128, 0, s>>>(
                    static_cast<const K*>(da.dev), static_cast<const K*>(db.dev),
                    static_cast<const uint64_t*>(dr.dev), static_cast<const uint64_t*>(dj.dev),
                    workers, static_cast<uint64_t*>(dmc.dev));
                if ((rc = check_launch("comerge: block comparisons launch"))) return rc;
                if ((rc = dmc.back(br.merge_cmps.data(), workers * 8, nullptr))) return rc;
            }
            if ((rc = dit.back(br.its.data(), nq * 4, nullptr))) return rc;
            if ((rc = dcmp.back(br.cmps.data(), nq * 4, nullptr))) return rc;
            if ((rc = dj.back(br.js.data(), nq * 8, nullptr))) return rc;
        }
        if ((rc = dout.back(out, total * sizeof(K), &d2h))) return rc;
        if (HAS_V && (rc = doutv.back(outv, total * 4, &d2h))) return rc;
        cudaEventRecord(e2e.b, s);
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: merge_parallel");
        br.emit(workers, synced, block_sizes, corank_iterations, comparisons);
    }
    if (rep) {
        rep->m = m;
        rep->n = n;
        rep->workers = workers;
        rep->wall_ns = total ? dev.ns() : 0;
        rep->e2e_ns = e2e.ns();
        rep->h2d_bytes = h2d;
        rep->d2h_bytes = d2h;
        rep->tiles = div_up(total, tile_cfg<K>::kTile);
    }
    return COMERGE_OK;
}

template <typename K>
int co_rank_sync(uint64_t target, const K* a, size_t m, const K* b, size_t n, uint64_t* j,
                 uint64_t* k, uint32_t* iterations, uint32_t* comparisons) {
    if (m > SIZE_MAX - n)
        return fail(COMERGE_E_LENGTH, "comerge: combined input length exceeds index range");
    if (target > m + n)  // corank.hpp:78-79
        return fail(COMERGE_E_RANGE, "co_rank: rank out of range (exceeds m+n)");
    if (!j || !k) return fail(COMERGE_E_INVALID, "co_rank: null result pointer");
    cudaStream_t s = sync_stream();
    int rc;
    uint64_t hj = 0;
    uint32_t hit = 0, hcmp = 0;
    {
        staged da, db, dr, dj, dit, dcmp;
        if ((rc = da.in(a, m * sizeof(K), s, nullptr))) return rc;
        if ((rc = db.in(b, n * sizeof(K), s, nullptr))) return rc;
        if ((rc = dr.in(&target, 8, s, nullptr))) return rc;
        if ((rc = dj.out_alloc(&hj, 8, s))) return rc;
        if ((rc = dit.out_alloc(&hit, 4, s))) return rc;
        if ((rc = dcmp.out_alloc(&hcmp, 4, s))) return rc;
        if ((rc = co_rank_batch_device<K>(
                 static_cast<const uint64_t*>(dr.dev), 1, static_cast<const K*>(da.dev), m,
                 static_cast<const K*>(db.dev), n, static_cast<uint64_t*>(dj.dev),
                 static_cast<uint32_t*>(dit.dev), static_cast<uint32_t*>(dcmp.dev), s)))
            return rc;
        if ((rc = dj.back(&hj, 8, nullptr)) || (rc = dit.back(&hit, 4, nullptr)) ||
            (rc = dcmp.back(&hcmp, 4, nullptr)))
            return rc;
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: co_rank");
    }
    *j = hj;
    *k = target - hj;
    if (iterations) *iterations = hit;
    if (comparisons) *comparisons = hcmp;
    return COMERGE_OK;
}

// comerge::plan (parallel.hpp:94-115): both co-ranks of every block from one
// batched Algorithm-1 launch over inputs staged once (host or device).
template <typename K>
int plan_sync(const K* a, size_t m, const K* b, size_t n, size_t workers, uint64_t* blocks) {
    if (m > SIZE_MAX - n)
        return fail(COMERGE_E_LENGTH, "comerge: combined input length exceeds index range");
    if (workers == 0) return fail(COMERGE_E_INVALID, "plan: worker count must be positive");
    if (!blocks) return fail(COMERGE_E_INVALID, "plan: null result pointer");
    if ((m && !a) || (n && !b)) return fail(COMERGE_E_INVALID, "plan: null input");
    const uint64_t total = uint64_t(m) + n;
    const size_t nq = workers + 1;
    std::vector<uint64_t> ranks(nq), js(nq);
    for (size_t r = 0; r <= workers; ++r) partition_output_impl(total, workers, r, &ranks[r]);
    cudaStream_t s = sync_stream();
    int rc;
    {
        staged da, db, dr, dj;
        if ((rc = da.in(a, m * sizeof(K), s, nullptr))) return rc;
        if ((rc = db.in(b, n * sizeof(K), s, nullptr))) return rc;
        if ((rc = dr.in(ranks.data(), nq * 8, s, nullptr))) return rc;
        if ((rc = dj.out_alloc(js.data(), nq * 8, s))) return rc;
        if ((rc = co_rank_batch_device<K>(static_cast<const uint64_t*>(dr.dev), nq,
                                          static_cast<const K*>(da.dev), m,
                                          static_cast<const K*>(db.dev), n,
                                          static_cast<uint64_t*>(dj.dev), nullptr, nullptr, s)))
            return rc;
        if ((rc = dj.back(js.data(), nq * 8, nullptr))) return rc;
        const cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: plan");
    }
    for (size_t r = 0; r < workers; ++r) {
        uint64_t* o = blocks + 7 * r;  // block_assignment, parallel.hpp:70-84
        o[0] = r;
        o[1] = ranks[r];
        o[2] = ranks[r + 1];
        o[3] = js[r];
        o[4] = js[r + 1];
        o[5] = ranks[r] - js[r];
        o[6] = ranks[r + 1] - js[r + 1];
    }
    return COMERGE_OK;
}

// comerge::merge_parallel over records (host or device pointers)
template <typename KT, int S>
int merge_parallel_records_sync(const void* a, size_t m, const void* b, size_t n, void* out,
                                size_t out_len, size_t workers, int synced,
                                comerge_merge_report* rep, uint64_t* block_sizes,
                                uint32_t* corank_iterations, uint64_t* comparisons = nullptr) {
    const int A = records_align_class<KT, S>(a, m, b, n, out);
    if (A == 0)
        return fail(COMERGE_E_INVALID, "merge_parallel: arrays must be aligned to their record type");
    auto run = [&](auto tag) {
        using R = decltype(tag);
        return merge_parallel_sync<R, false>(static_cast<const R*>(a), nullptr, m,
                                             static_cast<const R*>(b), nullptr, n,
                                             static_cast<R*>(out), nullptr, out_len, workers,
                                             synced, rep, block_sizes, corank_iterations,
                                             comparisons);
    };
    if constexpr (S == 16) {
        return A >= 16 ? run(rec<KT, 16, 16>{}) : run(rec<KT, 16, 8>{});
    } else if constexpr (S == 12) {
        return run(rec<KT, 12, 4>{});
    } else {
        return A >= 8 ? run(rec<KT, 8, 8>{}) : run(rec<KT, 8, 4>{});
    }
}

// The reference's generic co_rank / plan / full-report merge_parallel over
// records with a key-only less (corank.hpp:128-147 and parallel.hpp:94-115,
// :304-336 instantiated with tagged<K> / tagged_key_less, oracle.hpp:22-37;
// the comparator KAT of corank_test.cpp:205-214).  The record size arrives at
// run time: 8 or 12 bytes with a 32-bit key, 16 with a 64-bit one.  Co-ranks
// only read keys, so the narrowest-alignment instantiation serves every view.
template <typename KT, typename Fn>
int with_record_type(const char* who, size_t record_bytes, const void* a, size_t m, const void* b,
                     size_t n, Fn&& fn) {
    constexpr uintptr_t nat = sizeof(KT) - 1;  // the record struct's own alignment
    if ((m && (reinterpret_cast<uintptr_t>(a) & nat)) || (n && (reinterpret_cast<uintptr_t>(b) & nat)))
        return fail(COMERGE_E_INVALID, std::string(who) + ": arrays must be aligned to their record type");
    if constexpr (sizeof(KT) == 8) {
        if (record_bytes == 16) return fn(rec<KT, 16, 8>{});
        return fail(COMERGE_E_INVALID, std::string(who) + ": records with a 64-bit key are 16 bytes");
    } else {
        if (record_bytes == 8) return fn(rec<KT, 8, 4>{});
        if (record_bytes == 12) return fn(rec<KT, 12, 4>{});
        return fail(COMERGE_E_INVALID, std::string(who) + ": records with a 32-bit key are 8 or 12 bytes");
    }
}

template <typename KT>
int co_rank_records_sync(uint64_t target, const void* a, size_t m, const void* b, size_t n,
                         size_t record_bytes, uint64_t* j, uint64_t* k, uint32_t* iterations,
                         uint32_t* comparisons) {
    return with_record_type<KT>("co_rank", record_bytes, a, m, b, n, [&](auto tag) {
        using R = decltype(tag);
        return co_rank_sync<R>(target, static_cast<const R*>(a), m, static_cast<const R*>(b), n, j,
                               k, iterations, comparisons);
    });
}

template <typename KT>
int plan_records_sync(const void* a, size_t m, const void* b, size_t n, size_t record_bytes,
                      size_t workers, uint64_t* blocks) {
    return with_record_type<KT>("plan", record_bytes, a, m, b, n, [&](auto tag) {
        using R = decltype(tag);
        return plan_sync<R>(static_cast<const R*>(a), m, static_cast<const R*>(b), n, workers,
                            blocks);
    });
}

template <typename KT>
int co_rank_batch_records_device(const uint64_t* ranks, size_t count, const void* a, size_t m,
                                 const void* b, size_t n, size_t record_bytes, uint64_t* out_j,
                                 uint32_t* out_it, uint32_t* out_cmp, cudaStream_t s) {
    return with_record_type<KT>("co_rank", record_bytes, a, m, b, n, [&](auto tag) {
        using R = decltype(tag);
        return co_rank_batch_device<R>(ranks, count, static_cast<const R*>(a), m,
                                       static_cast<const R*>(b), n, out_j, out_it, out_cmp, s);
    });
}

template <typename KT>
int merge_parallel_records_ex(const void* a, size_t m, const void* b, size_t n, void* out,
                              size_t out_len, size_t record_bytes, size_t workers,
                              const comerge_merge_options* opts, comerge_merge_report* rep,
                              uint64_t* block_sizes, uint32_t* corank_iterations,
                              uint64_t* comparisons) {
    const int synced = opts ? opts->synced : 0;
    if (opts && opts->count_comparisons && !comparisons)
        return fail(COMERGE_E_INVALID, "merge_parallel: count_comparisons needs an output");
    uint64_t* cmp = opts && opts->count_comparisons ? comparisons : nullptr;
    if constexpr (sizeof(KT) == 8) {
        if (record_bytes == 16)
            return merge_parallel_records_sync<KT, 16>(a, m, b, n, out, out_len, workers, synced,
                                                       rep, block_sizes, corank_iterations, cmp);
        return fail(COMERGE_E_INVALID, "merge_parallel: records with a 64-bit key are 16 bytes");
    } else {
        if (record_bytes == 8)
            return merge_parallel_records_sync<KT, 8>(a, m, b, n, out, out_len, workers, synced,
                                                      rep, block_sizes, corank_iterations, cmp);
        if (record_bytes == 12)
            return merge_parallel_records_sync<KT, 12>(a, m, b, n, out, out_len, workers, synced,
                                                       rep, block_sizes, corank_iterations, cmp);
        return fail(COMERGE_E_INVALID, "merge_parallel: records with a 32-bit key are 8 or 12 bytes");
    }
}

}  // namespace

// ------------------------------------------------------------ merge sort
// Stable sort of keys[0, n) into out (may equal keys): block sort of runs of
// R = sort_cfg<K>::R, then log2(n / R) merge passes of the pipeline in
// merge-pass mode (sort.cuh).  Workspace: one n-element buffer (two when out
// is not 16-byte aligned) plus the pipeline's tail slots.
template <typename K>
size_t sort_ws_bytes(size_t n) {
    if (n == 0) return 0;
    const size_t buf = round256(n * sizeof(K));
    const size_t tail = round256(32 * (div_up(n, pipe_layout<K, false, 1>::T) + 4));
    return 2 * buf + tail;
}

template <typename K>
size_t sort_pairs_ws_bytes(size_t n) {
    if (n == 0) return 0;
    const size_t buf = round256(n * sizeof(K)) + round256(n * 4);
    const size_t tail = round256(32 * (div_up(n, pipe_layout<K, true, 2>::T) + 4));
    return 2 * buf + tail;
}

// Merge passes launch with programmatic dependent launch (flags bit 24: off,
// an A/B knob): each pass's grid is scheduled while the previous kernel
// drains instead of after it.
inline bool sort_pdl() { return !(g_tune_flags & 16777216); }

// Stable key-value merge sort: as sort_device, the payload moving with its key.
// block sorts: dynamic shared memory, opted in once per device
template <typename K, bool SMALL>
void launch_block_sort_pairs(const K* in, const uint32_t* in_v, K* out, uint32_t* out_v,
                             uint64_t n, cudaStream_t s) {
    using C = sort_pairs_cfg<K, SMALL>;
    static std::once_flag once[kMaxDevices];
    std::call_once(once[current_device()], [] {
        cudaFuncSetAttribute(block_sort_pairs_kernel<K, SMALL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem));
    });
    block_sort_pairs_kernel<K, SMALL><<<unsigned(div_up(n, C::R)), C::NT, C::kSmem, s>>>(
        in, in_v, out, out_v, n);
}

// Base run of a sort of n elements: the full-size run, or half of it (twice the
// CTAs) while the input is under one full-size run per SM.
template <typename CFG_BIG, typename CFG_SMALL>
bool sort_small_runs(uint64_t n) {
    return n < uint64_t(CFG_BIG::R) * uint64_t(sm_count());
}

template <typename K>
int sort_pairs_device(const K* keys, const uint32_t* vals, size_t n, K* out, uint32_t* out_v,
                      void* ws, size_t ws_bytes, cudaStream_t s) {
    if (n && (!keys || !vals || !out || !out_v))
        return fail(COMERGE_E_INVALID, "sort_pairs: null pointer");
    if (n == 0) return COMERGE_OK;
    if (n > (size_t(1) << 40)) return fail(COMERGE_E_LENGTH, "sort_pairs: more than 2^40 elements");
    if ((keys != out && overlaps(keys, n * sizeof(K), out, n * sizeof(K))) ||
        (vals != out_v && overlaps(vals, n * 4, out_v, n * 4)) ||
        overlaps(out, n * sizeof(K), out_v, n * 4))
        return fail(COMERGE_E_INVALID, "sort_pairs: outputs must not partially overlap the inputs or each other");
    const bool small = sort_small_runs<sort_pairs_cfg<K, false>, sort_pairs_cfg<K, true>>(n);
    const uint64_t R = small ? sort_pairs_cfg<K, true>::R : sort_pairs_cfg<K, false>::R;
    auto block_sort = [&](K* ok, uint32_t* ov) {
        if (small)
            launch_block_sort_pairs<K, true>(keys, vals, ok, ov, n, s);
        else
            launch_block_sort_pairs<K, false>(keys, vals, ok, ov, n, s);
    };
    uint32_t passes = 0;
    while ((R << passes) < n) ++passes;
    if (passes == 0) {
        block_sort(out, out_v);
        return check_launch("comerge: block sort launch");
    }
    scratch sc;
    if (int rc = sc.acquire(ws, ws_bytes, sort_pairs_ws_bytes<K>(n), s)) return rc;
    unsigned char* w = static_cast<unsigned char*>(sc.ptr);
    const size_t kb = round256(n * sizeof(K)), vb = round256(n * 4);
    K* tk[2] = {reinterpret_cast<K*>(w), reinterpret_cast<K*>(w + kb + vb)};
    uint32_t* tv[2] = {reinterpret_cast<uint32_t*>(w + kb),
                       reinterpret_cast<uint32_t*>(w + 2 * kb + vb)};
    unsigned char* tail = w + 2 * (kb + vb);
    const size_t tail_bytes = sort_pairs_ws_bytes<K>(n) - 2 * (kb + vb);
    const bool direct = aligned16(out) && aligned16(out_v);
    K* bk[2] = {direct ? out : tk[1], tk[0]};
    uint32_t* bv[2] = {direct ? out_v : tv[1], tv[0]};
    K* ck = bk[passes & 1];
    uint32_t* cv = bv[passes & 1];
    block_sort(ck, cv);
    if (int rc = check_launch("comerge: block sort launch")) return rc;
    uint64_t L = R;
    for (uint32_t p = 0; p < passes; ++p, L *= 2) {
        K* dk = bk[(passes - p - 1) & 1];
        uint32_t* dv = bv[(passes - p - 1) & 1];
        const uint64_t full = n / (2 * L), rem = n % (2 * L);
        const uint64_t ma = full * L + (rem < L ? rem : L), mb = n - ma;
        if (int rc = launch_pipe<K, true, 2>(ck, cv, ma, ck, cv, mb, dk, dv, nullptr, nullptr,
                                             div_up(n, 2 * L), tail, tail_bytes, s, L, nullptr,
                                             sort_pdl()))
            return rc;
        ck = dk;
        cv = dv;
    }
    if (ck != out) {
        cudaError_t e = cudaMemcpyAsync(out, ck, n * sizeof(K), cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out_v, cv, n * 4, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: sort result copy");
    }
    return COMERGE_OK;
}

template <typename K, bool SMALL>
void launch_block_sort(const K* in, K* out, uint64_t n, cudaStream_t s) {
    using C = sort_cfg<K, SMALL>;
    static std::once_flag once[kMaxDevices];
    std::call_once(once[current_device()], [] {
        cudaFuncSetAttribute(block_sort_kernel<K, SMALL>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::kSmem));
    });
    block_sort_kernel<K, SMALL><<<unsigned(div_up(n, C::R)), C::NT, C::kSmem, s>>>(in, out, n);
}

template <typename K>
int sort_device(const K* keys, size_t n, K* out, void* ws, size_t ws_bytes, cudaStream_t s) {
    if (n && (!keys || !out)) return fail(COMERGE_E_INVALID, "sort: null pointer");
    if (n == 0) return COMERGE_OK;
    if (n > (size_t(1) << 40)) return fail(COMERGE_E_LENGTH, "sort: more than 2^40 elements");
    if (keys != out && overlaps(keys, n * sizeof(K), out, n * sizeof(K)))
        return fail(COMERGE_E_INVALID, "sort: output must not partially overlap the input");
    const bool small = sort_small_runs<sort_cfg<K, false>, sort_cfg<K, true>>(n);
    const uint64_t R = small ? sort_cfg<K, true>::R : sort_cfg<K, false>::R;
    auto block_sort = [&](K* dst) {
        if (small)
            launch_block_sort<K, true>(keys, dst, n, s);
        else
            launch_block_sort<K, false>(keys, dst, n, s);
    };
    uint32_t passes = 0;
    while ((R << passes) < n) ++passes;
    if (passes == 0) {
        block_sort(out);
        return check_launch("comerge: block sort launch");
    }
    scratch sc;
    if (int rc = sc.acquire(ws, ws_bytes, sort_ws_bytes<K>(n), s)) return rc;
    unsigned char* w = static_cast<unsigned char*>(sc.ptr);
    const size_t buf = round256(n * sizeof(K));
    K* t0 = reinterpret_cast<K*>(w);
    K* t1 = reinterpret_cast<K*>(w + buf);
    unsigned char* tail = w + 2 * buf;
    const size_t tail_bytes = sort_ws_bytes<K>(n) - 2 * buf;
    // ping-pong so the last pass lands in out (or in t0, then one copy when out
    // is not 16-byte aligned for the pipeline's bulk stores)
    const bool direct = aligned16(out);
    K* bufs[2] = {direct ? out : t1, t0};  // bufs[x]: the result of a stage with passes-left parity x
    K* cur = bufs[passes & 1];
    block_sort(cur);
    if (int rc = check_launch("comerge: block sort launch")) return rc;
    uint64_t L = R;
    for (uint32_t p = 0; p < passes; ++p, L *= 2) {
        K* dst = bufs[(passes - p - 1) & 1];
        const uint64_t full = n / (2 * L), rem = n % (2 * L);
        const uint64_t ma = full * L + (rem < L ? rem : L), mb = n - ma;
        const uint64_t nseg = div_up(n, 2 * L);
        if (int rc = launch_pipe<K, false, 2>(cur, nullptr, ma, cur, nullptr, mb, dst, nullptr,
                                                 nullptr, nullptr, nseg, tail, tail_bytes, s, L,
                                                 nullptr, sort_pdl()))
            return rc;
        cur = dst;
    }
    if (cur != out) {
        const cudaError_t e = cudaMemcpyAsync(out, cur, n * sizeof(K), cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "comerge: sort result copy");
    }
    return COMERGE_OK;
}

extern "C" {

const char* comerge_cuda_last_error(void) { return g_error.c_str(); }

void comerge_cuda_set_path(int path) { g_path = path; }
void comerge_cuda_set_host_mode(int mode) { g_host_mode = mode; }
int comerge_cuda_last_path(void) { return g_last_path; }
void comerge_cuda_set_trace(unsigned long long* device_buffer) { g_trace = device_buffer; }
void comerge_cuda_set_tuning(int static_pct, int flags, int lookahead) {
    g_tune_static_pct = static_pct;
    g_tune_flags = flags;
    g_tune_lookahead = lookahead;
}

void comerge_cuda_set_kernel_events(void* before, void* after) {
    g_ev_before = static_cast<cudaEvent_t>(before);
    g_ev_after = static_cast<cudaEvent_t>(after);
}
int comerge_cuda_abi_version(void) { return 10000; }

int comerge_cuda_host_alloc(size_t bytes, void** ptr) {
    if (!ptr) return fail(COMERGE_E_INVALID, "host_alloc: null result pointer");
    *ptr = nullptr;
    if (bytes == 0) return COMERGE_OK;
    const cudaError_t e = cudaHostAlloc(ptr, bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        *ptr = nullptr;
        return cuda_fail(e, "comerge: page-locked host allocation");
    }
    return COMERGE_OK;
}

int comerge_cuda_host_free(void* ptr) {
    if (!ptr) return COMERGE_OK;
    const cudaError_t e = cudaFreeHost(ptr);
    return e == cudaSuccess ? COMERGE_OK : cuda_fail(e, "comerge: page-locked host free");
}

size_t comerge_cuda_merge_workspace_bytes(size_t m, size_t n, int key_kind, int) {
    return with_slack(key_kind == COMERGE_KEY_U64 ? merge_ws_bytes<uint64_t>(m, n)
                                                  : merge_ws_bytes<uint32_t>(m, n));
}
size_t comerge_cuda_segmented_workspace_bytes(size_t total, size_t, int key_kind) {
    return with_slack(key_kind == COMERGE_KEY_U64 ? seg_ws_bytes<uint64_t>(total)
                                                  : seg_ws_bytes<uint32_t>(total));
}

#define COMERGE_KEYS(SUF, K)                                                                     \
    int comerge_cuda_merge_keys_##SUF(const K* a, size_t m, const K* b, size_t n, K* out,       \
                                      void* ws, size_t ws_bytes, comerge_stream_t stream) {      \
        return merge_device<K, false>(a, nullptr, m, b, nullptr, n, out, nullptr, ws, ws_bytes,  \
                                      stream);                                                   \
    }                                                                                            \
    int comerge_cuda_merge_pairs_##SUF(const K* ak, const uint32_t* av, size_t m, const K* bk,   \
                                       const uint32_t* bv, size_t n, K* ok, uint32_t* ov,        \
                                       void* ws, size_t ws_bytes, comerge_stream_t stream) {     \
        return merge_device<K, true>(ak, av, m, bk, bv, n, ok, ov, ws, ws_bytes, stream);        \
    }                                                                                            \
    int comerge_cuda_co_rank_batch_##SUF(const uint64_t* ranks, size_t count, const K* a,       \
                                         size_t m, const K* b, size_t n, uint64_t* out_j,        \
                                         uint32_t* out_it, uint32_t* out_cmp,                    \
                                         comerge_stream_t stream) {                              \
        return co_rank_batch_device<K>(ranks, count, a, m, b, n, out_j, out_it, out_cmp,         \
                                       stream);                                                  \
    }                                                                                            \
    int comerge_merge_parallel_##SUF(const K* a, size_t m, const K* b, size_t n, K* out,        \
                                     size_t out_len, size_t workers, int synced,                 \
                                     comerge_merge_report* report, uint64_t* block_sizes,        \
                                     uint32_t* corank_iterations) {                              \
        return merge_parallel_sync<K, false>(a, nullptr, m, b, nullptr, n, out, nullptr,         \
                                             out_len, workers, synced, report, block_sizes,      \
                                             corank_iterations);                                 \
    }                                                                                            \
    int comerge_merge_parallel_ex_##SUF(const K* a, const uint32_t* av, size_t m, const K* b,    \
                                        const uint32_t* bv, size_t n, K* out, uint32_t* outv,    \
                                        size_t out_len, size_t workers,                          \
                                        const comerge_merge_options* opts,                       \
                                        comerge_merge_report* report, uint64_t* block_sizes,     \
                                        uint32_t* corank_iterations, uint64_t* comparisons) {    \
        const int synced = opts ? opts->synced : 0;                                              \
        uint64_t* cmp = opts && opts->count_comparisons ? comparisons : nullptr;                 \
        if (opts && opts->count_comparisons && !comparisons)                                     \
            return fail(COMERGE_E_INVALID, "merge_parallel: count_comparisons needs an output"); \
        if (av || bv || outv) {                                                                  \
            if (!(av || m == 0) || !(bv || n == 0) || !(outv || m + n == 0))                     \
                return fail(COMERGE_E_INVALID, "merge_parallel: payloads need all three arrays"); \
            return merge_parallel_sync<K, true>(a, av, m, b, bv, n, out, outv, out_len, workers, \
                                                synced, report, block_sizes, corank_iterations,  \
                                                cmp);                                            \
        }                                                                                        \
        return merge_parallel_sync<K, false>(a, nullptr, m, b, nullptr, n, out, nullptr,         \
                                             out_len, workers, synced, report, block_sizes,      \
                                             corank_iterations, cmp);                            \
    }                                                                                            \
    int comerge_merge_parallel_pairs_##SUF(const K* ak, const uint32_t* av, size_t m,            \
                                           const K* bk, const uint32_t* bv, size_t n, K* ok,     \
                                           uint32_t* ov, size_t out_len, size_t workers,         \
                                           comerge_merge_report* report) {                       \
        return merge_parallel_sync<K, true>(ak, av, m, bk, bv, n, ok, ov, out_len, workers, 0,   \
                                            report, nullptr, nullptr);                           \
    }                                                                                            \
    int comerge_cuda_merge_keys_pieces_##SUF(const K* const* a_pieces, const uint64_t* a_lens,  \
                                             int na, const K* const* b_pieces,                   \
                                             const uint64_t* b_lens, int nb, uint64_t out_begin, \
                                             uint64_t out_end, K* out, void* ws,                 \
                                             size_t ws_bytes, comerge_stream_t stream) {         \
        return merge_pieces_device<K, false>(a_pieces, nullptr, a_lens, na, b_pieces, nullptr,  \
                                             b_lens, nb, out_begin, out_end, out, nullptr, ws,   \
                                             ws_bytes, stream);                                  \
    }                                                                                            \
    int comerge_cuda_merge_pairs_pieces_##SUF(                                                   \
        const K* const* a_pieces, const uint32_t* const* a_val_pieces, const uint64_t* a_lens,  \
        int na, const K* const* b_pieces, const uint32_t* const* b_val_pieces,                  \
        const uint64_t* b_lens, int nb, uint64_t out_begin, uint64_t out_end, K* out_keys,       \
        uint32_t* out_vals, void* ws, size_t ws_bytes, comerge_stream_t stream) {                \
        return merge_pieces_device<K, true>(a_pieces, a_val_pieces, a_lens, na, b_pieces,        \
                                            b_val_pieces, b_lens, nb, out_begin, out_end,        \
                                            out_keys, out_vals, ws, ws_bytes, stream);           \
    }                                                                                            \
    int comerge_plan_##SUF(const K* a, size_t m, const K* b, size_t n, size_t workers,          \
                           uint64_t* blocks) {                                                   \
        return plan_sync<K>(a, m, b, n, workers, blocks);                                        \
    }                                                                                            \
    int comerge_co_rank_##SUF(uint64_t target, const K* a, size_t m, const K* b, size_t n,       \
                              uint64_t* j, uint64_t* k, uint32_t* iterations,                    \
                              uint32_t* comparisons) {                                           \
        return co_rank_sync<K>(target, a, m, b, n, j, k, iterations, comparisons);               \
    }

COMERGE_KEYS(i32, int32_t)
COMERGE_KEYS(u32, uint32_t)
COMERGE_KEYS(u64, uint64_t)

int comerge_cuda_merge_segmented_i32(const int32_t* a, const uint64_t* a_off, size_t m,
                                     const int32_t* b, const uint64_t* b_off, size_t n,
                                     size_t nseg, int32_t* out, void* ws, size_t ws_bytes,
                                     comerge_stream_t stream) {
    return merge_segmented_device<int32_t>(a, a_off, m, b, b_off, n, nseg, out, ws, ws_bytes,
                                           stream);
}
int comerge_cuda_merge_segmented_u32(const uint32_t* a, const uint64_t* a_off, size_t m,
                                     const uint32_t* b, const uint64_t* b_off, size_t n,
                                     size_t nseg, uint32_t* out, void* ws, size_t ws_bytes,
                                     comerge_stream_t stream) {
    return merge_segmented_device<uint32_t>(a, a_off, m, b, b_off, n, nseg, out, ws, ws_bytes,
                                            stream);
}

int comerge_merge_segmented_host_i32(const int32_t* a, const uint64_t* a_off, size_t m,
                                     const int32_t* b, const uint64_t* b_off, size_t n,
                                     size_t nseg, int32_t* out, size_t out_len,
                                     comerge_merge_report* report) {
    return merge_segmented_sync<int32_t>(a, a_off, m, b, b_off, n, nseg, out, out_len, report);
}
int comerge_merge_segmented_host_u32(const uint32_t* a, const uint64_t* a_off, size_t m,
                                     const uint32_t* b, const uint64_t* b_off, size_t n,
                                     size_t nseg, uint32_t* out, size_t out_len,
                                     comerge_merge_report* report) {
    return merge_segmented_sync<uint32_t>(a, a_off, m, b, b_off, n, nseg, out, out_len, report);
}

size_t comerge_cuda_sort_workspace_bytes(size_t n, int key_kind) {
    return with_slack(key_kind == COMERGE_KEY_U64 ? sort_ws_bytes<uint64_t>(n)
                                                  : sort_ws_bytes<uint32_t>(n));
}
size_t comerge_cuda_sort_pairs_workspace_bytes(size_t n, int key_kind) {
    return with_slack(key_kind == COMERGE_KEY_U64 ? sort_pairs_ws_bytes<uint64_t>(n)
                                                  : sort_pairs_ws_bytes<uint32_t>(n));
}
int comerge_cuda_sort_pairs_i32(const int32_t* keys, const uint32_t* vals, size_t n,
                                int32_t* out_keys, uint32_t* out_vals, void* ws, size_t ws_bytes,
                                comerge_stream_t stream) {
    return sort_pairs_device<int32_t>(keys, vals, n, out_keys, out_vals, ws, ws_bytes, stream);
}
int comerge_cuda_sort_pairs_u32(const uint32_t* keys, const uint32_t* vals, size_t n,
                                uint32_t* out_keys, uint32_t* out_vals, void* ws, size_t ws_bytes,
                                comerge_stream_t stream) {
    return sort_pairs_device<uint32_t>(keys, vals, n, out_keys, out_vals, ws, ws_bytes, stream);
}
int comerge_cuda_sort_pairs_u64(const uint64_t* keys, const uint32_t* vals, size_t n,
                                uint64_t* out_keys, uint32_t* out_vals, void* ws, size_t ws_bytes,
                                comerge_stream_t stream) {
    return sort_pairs_device<uint64_t>(keys, vals, n, out_keys, out_vals, ws, ws_bytes, stream);
}
int comerge_cuda_sort_keys_i32(const int32_t* keys, size_t n, int32_t* out, void* ws,
                               size_t ws_bytes, comerge_stream_t stream) {
    return sort_device<int32_t>(keys, n, out, ws, ws_bytes, stream);
}
int comerge_cuda_sort_keys_u32(const uint32_t* keys, size_t n, uint32_t* out, void* ws,
                               size_t ws_bytes, comerge_stream_t stream) {
    return sort_device<uint32_t>(keys, n, out, ws, ws_bytes, stream);
}
int comerge_cuda_sort_keys_u64(const uint64_t* keys, size_t n, uint64_t* out, void* ws,
                               size_t ws_bytes, comerge_stream_t stream) {
    return sort_device<uint64_t>(keys, n, out, ws, ws_bytes, stream);
}

size_t comerge_cuda_records_workspace_bytes(size_t m, size_t n, int key_kind) {
    return with_slack(key_kind == COMERGE_KEY_U64 ? records_ws_bytes<uint64_t, 16>(m, n)
                                                  : records_ws_bytes<uint32_t, 8>(m, n));
}

#define COMERGE_RECORDS(SUF, KT, S)                                                              \
    int comerge_cuda_merge_records_##SUF(const comerge_rec_##SUF* a, size_t m,                   \
                                         const comerge_rec_##SUF* b, size_t n,                   \
                                         comerge_rec_##SUF* out, void* ws, size_t ws_bytes,      \
                                         comerge_stream_t stream) {                              \
        return merge_records_device<KT, S>(a, m, b, n, out, ws, ws_bytes, stream);              \
    }                                                                                            \
    int comerge_merge_parallel_records_##SUF(                                                    \
        const comerge_rec_##SUF* a, size_t m, const comerge_rec_##SUF* b, size_t n,              \
        comerge_rec_##SUF* out, size_t out_len, size_t workers, int synced,                      \
        comerge_merge_report* report, uint64_t* block_sizes, uint32_t* corank_iterations) {      \
        return merge_parallel_records_sync<KT, S>(a, m, b, n, out, out_len, workers, synced,     \
                                                  report, block_sizes, corank_iterations);       \
    }

COMERGE_RECORDS(i32, int32_t, 8)
COMERGE_RECORDS(u32, uint32_t, 8)
COMERGE_RECORDS(u64, uint64_t, 16)

size_t comerge_cuda_records12_workspace_bytes(size_t m, size_t n) {
    return with_slack(records_ws_bytes<uint32_t, 12>(m, n));
}

#define COMERGE_RECORDS12(SUF, KT)                                                               \
    int comerge_cuda_merge_records12_##SUF(const comerge_rec12_##SUF* a, size_t m,               \
                                           const comerge_rec12_##SUF* b, size_t n,               \
                                           comerge_rec12_##SUF* out, void* ws, size_t ws_bytes,  \
                                           comerge_stream_t stream) {                            \
        return merge_records_device<KT, 12>(a, m, b, n, out, ws, ws_bytes, stream);             \
    }                                                                                            \
    int comerge_merge_parallel_records12_##SUF(                                                  \
        const comerge_rec12_##SUF* a, size_t m, const comerge_rec12_##SUF* b, size_t n,          \
        comerge_rec12_##SUF* out, size_t out_len, size_t workers, int synced,                    \
        comerge_merge_report* report, uint64_t* block_sizes, uint32_t* corank_iterations) {      \
        return merge_parallel_records_sync<KT, 12>(a, m, b, n, out, out_len, workers, synced,    \
                                                   report, block_sizes, corank_iterations);      \
    }

COMERGE_RECORDS12(i32, int32_t)
COMERGE_RECORDS12(u32, uint32_t)

#define COMERGE_RECORDS_GENERIC(SUF, KT)                                                         \
    int comerge_co_rank_records_##SUF(uint64_t target, const void* a, size_t m, const void* b,   \
                                      size_t n, size_t record_bytes, uint64_t* j, uint64_t* k,   \
                                      uint32_t* iterations, uint32_t* comparisons) {             \
        return co_rank_records_sync<KT>(target, a, m, b, n, record_bytes, j, k, iterations,      \
                                        comparisons);                                            \
    }                                                                                            \
    int comerge_plan_records_##SUF(const void* a, size_t m, const void* b, size_t n,             \
                                   size_t record_bytes, size_t workers, uint64_t* blocks) {      \
        return plan_records_sync<KT>(a, m, b, n, record_bytes, workers, blocks);                 \
    }                                                                                            \
    int comerge_cuda_co_rank_batch_records_##SUF(                                                \
        const uint64_t* ranks, size_t count, const void* a, size_t m, const void* b, size_t n,   \
        size_t record_bytes, uint64_t* out_j, uint32_t* out_it, uint32_t* out_cmp,               \
        comerge_stream_t stream) {                                                               \
        return co_rank_batch_records_device<KT>(ranks, count, a, m, b, n, record_bytes, out_j,   \
                                                out_it, out_cmp, stream);                        \
    }                                                                                            \
    int comerge_merge_parallel_records_ex_##SUF(                                                 \
        const void* a, size_t m, const void* b, size_t n, void* out, size_t out_len,             \
        size_t record_bytes, size_t workers, const comerge_merge_options* opts,                  \
        comerge_merge_report* report, uint64_t* block_sizes, uint32_t* corank_iterations,        \
        uint64_t* comparisons) {                                                                 \
        return merge_parallel_records_ex<KT>(a, m, b, n, out, out_len, record_bytes, workers,    \
                                             opts, report, block_sizes, corank_iterations,       \
                                             comparisons);                                       \
    }

COMERGE_RECORDS_GENERIC(i32, int32_t)
COMERGE_RECORDS_GENERIC(u32, uint32_t)
COMERGE_RECORDS_GENERIC(u64, uint64_t)

static_assert(sizeof(comerge_rec_i32) == sizeof(rec<int32_t, 8, 8>) &&
                  sizeof(comerge_rec_u64) == sizeof(rec<uint64_t, 16, 16>) &&
                  offsetof(comerge_rec_u64, val) == 8 &&
                  sizeof(comerge_rec12_i32) == sizeof(rec<int32_t, 12, 4>) &&
                  sizeof(comerge_rec12_u32) == 12,
              "record layouts");

int comerge_partition_output(uint64_t total, uint64_t workers, uint64_t r, uint64_t* out) {
    if (!out) return fail(COMERGE_E_INVALID, "partition_output: null result pointer");
    return partition_output_impl(total, workers, r, out);
}

}  // extern "C"
