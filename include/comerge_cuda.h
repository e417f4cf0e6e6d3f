/*
 * comerge_cuda.h -- C ABI of the B200 (sm_100a) stable parallel merge.
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/proj/include/comerge/{corank,merge,parallel}.hpp).  The
 * reference is header-only C++ with no C ABI of its own; every entry point
 * below names the reference interface it replaces.  All indices are size_t
 * / uint64_t, all memory is caller-owned, and nothing here takes a torch or
 * CUDA-runtime type: the stream argument is a `struct CUstream_st*`, which is
 * exactly `cudaStream_t`.
 *
 * Two tiers:
 *   comerge_cuda_*   asynchronous, DEVICE pointers, enqueued on `stream`,
 *                    scratch from a caller workspace (or NULL: stream-ordered
 *                    allocation inside the call).
 *   comerge_merge_parallel_* / comerge_co_rank_*
 *                    synchronous mirrors of the reference's templates taking
 *                    HOST or DEVICE pointers (detected per call), filling a
 *                    merge report like comerge::merge_report.
 *
 * Error behaviour mirrors the reference's exceptions as status codes; the
 * message (same substrings as the reference's what()) is available from
 * comerge_cuda_last_error() on the calling thread.
 */
#ifndef COMERGE_CUDA_H
#define COMERGE_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

struct CUstream_st;
typedef struct CUstream_st* comerge_stream_t; /* == cudaStream_t */

typedef enum comerge_status {
    COMERGE_OK = 0,
    COMERGE_E_INVALID = 1, /* std::invalid_argument: length, alias, null, workers==0 */
    COMERGE_E_RANGE = 2,   /* std::out_of_range: "rank out of range (exceeds m+n)"   */
    COMERGE_E_LENGTH = 3,  /* std::length_error: m+n beyond the index range          */
    COMERGE_E_CUDA = 4     /* launch / runtime failure (detail in last_error)         */
} comerge_status;

typedef enum comerge_key_kind {
    COMERGE_KEY_I32 = 0,
    COMERGE_KEY_U32 = 1,
    COMERGE_KEY_U64 = 2
} comerge_key_kind;

/* Thread-local message of the last failing call ("" if none). */
const char* comerge_cuda_last_error(void);
/* ABI version (major*10000 + minor*100 + patch). */
int comerge_cuda_abi_version(void);

/* Page-locked host memory for the host-buffer entry points.  The host
 * pipeline's copies run at PCIe rate only from page-locked buffers (measured
 * on C4: 69 ms pinned; from pageable std::vector storage 467 ms through the
 * driver's synchronous staging, 132 ms through the library's staging pool);
 * comerge::cuda::pinned_allocator<T> wraps
 * these for std::vector.  Returns COMERGE_OK or COMERGE_E_CUDA. */
int comerge_cuda_host_alloc(size_t bytes, void** ptr);
int comerge_cuda_host_free(void* ptr);

/* Instrumentation (bench / profiling): when set on the calling thread, every
 * comerge_cuda_merge_* call records `before` on its stream right before the
 * dominant merge kernel and `after` right after it, so a caller can time that
 * kernel alone with cudaEventElapsedTime.  Pass NULLs to disable.  The
 * arguments are cudaEvent_t handles. */
void comerge_cuda_set_kernel_events(void* before, void* after);

/* Kernel selection on the calling thread (testing / benchmarking every
 * device path): 0 = automatic (default: 4 up to one wave of tiles, i.e.
 * 2 x #SMs pipeline tiles, else 3), 1 = tile kernel (partition + one CTA per
 * tile), 3 = persistent tile-pipeline kernel, 4 = one-wave small-merge kernel
 * (one CTA per tile, both boundaries co-ranked in the CTA).  All take arrays
 * at any element offset.  Segmented batches: 1 or else the pipeline. */
void comerge_cuda_set_path(int path);
/* Kernel used by the last merge on this thread: 1 = tile kernel (partition
 * + merge launches), 3 = tile pipeline (one launch), 4 = segmented tile
 * kernel (partition + merge), 5 = segmented tile pipeline (one launch),
 * 6 = merge pass of the sort (tile pipeline over runs), 7 = pieced-input
 * range merge, 8 = small-merge kernel (one launch), 0 = none yet. */
int comerge_cuda_last_path(void);
/* Host-buffer strategy of the synchronous entry points on this thread
 * (testing / benchmarking): 0 = chunked pipeline (default: output chunks
 * co-ranked on the host, H2D / device merge / D2H overlapped on three
 * streams), 1 = zero-copy for pinned host memory (the kernel reads and writes
 * host memory over PCIe), 2 = plain staging (copy in, merge, copy out). */
void comerge_cuda_set_host_mode(int mode);
/* Debug tracing of the persistent kernels: when non-NULL (at least
 * 20*4096 uint64), CTA c writes %globaltimer stamps and counters to
 * device_buffer[8c .. 8c+7], consumer phase sums to
 * device_buffer[8*4096 + 4c ..], producer starvation (static range / tail)
 * to device_buffer[12*4096 + 4c ..] and scheduler tail counters to
 * device_buffer[16*4096 + 4c ..].  NULL disables. */
void comerge_cuda_set_trace(unsigned long long* device_buffer);
/* Tuning knobs of the tile pipeline (benchmarking only, per host thread;
 * 0 = default): the statically assigned share of tiles in percent (default
 * 70; the rest is the dynamic tail), experiment flags, and the claim
 * look-ahead (queued tiles below which the next tail tile is claimed,
 * default 2).  Flags: bit 0 co-rank the start-up boundaries one after the
 * other; bits 2-3 scheduler pass cap (1: 8, 2: 16, 3: 32); bits 4-7
 * scheduler look-ahead / 4; bit 8 / 9 output stores evict-first on / off;
 * bit 10 no concurrent start-up searches for segmented batches; bit 12 no L2
 * pull of small inputs; bit 13 no L2 pull of segment offsets; bit 14 the
 * small-merge kernel's searches to the end (no superset windows); bits 15-17
 * dynamic-tail anchor unit (1-7, default 4); bit 24 merge passes without
 * programmatic dependent launch. */
void comerge_cuda_set_tuning(int static_pct, int flags, int lookahead);

/* ------------------------------------------------------------ workspace */

/* Bytes of scratch the merge entry points need for (m, n): the tile
 * boundary co-ranks / the pipeline's dynamic-tail state.  Replaces nothing in
 * the reference (which allocates per-worker slots itself, parallel.hpp:189);
 * CUB-style query.  A workspace may have any alignment: the library uses it
 * from its first 256-byte boundary, and every *_workspace_bytes figure
 * includes those 256 bytes of slack (also for the sort queries below). */
size_t comerge_cuda_merge_workspace_bytes(size_t m, size_t n, int key_kind, int has_payload);
size_t comerge_cuda_segmented_workspace_bytes(size_t total, size_t nseg, int key_kind);

/* ------------------------------------------- asynchronous, device memory */

/* Stable merge of sorted a[0,m) and b[0,n) into out[0,m+n), ties A-first.
 * Replaces comerge::merge_parallel / merge_parallel_synced /
 * stable_merge for keys with std::less<> (parallel.hpp:304-336,
 * merge.hpp:52-68).  `out` must not overlap a or b (E_INVALID). */
int comerge_cuda_merge_keys_i32(const int32_t* a, size_t m, const int32_t* b, size_t n,
                                int32_t* out, void* ws, size_t ws_bytes, comerge_stream_t stream);
int comerge_cuda_merge_keys_u32(const uint32_t* a, size_t m, const uint32_t* b, size_t n,
                                uint32_t* out, void* ws, size_t ws_bytes,
                                comerge_stream_t stream);
int comerge_cuda_merge_keys_u64(const uint64_t* a, size_t m, const uint64_t* b, size_t n,
                                uint64_t* out, void* ws, size_t ws_bytes,
                                comerge_stream_t stream);

/* Key-value merge (SoA keys + uint32 payload): the same decisions as the
 * keys-only merge, payload moved with its key.  Replaces merge_parallel over
 * a {key, val} struct with a key-only less (the reference's
 * tagged<K>/tagged_key_less pattern, oracle.hpp:22-37). */
int comerge_cuda_merge_pairs_i32(const int32_t* a_keys, const uint32_t* a_vals, size_t m,
                                 const int32_t* b_keys, const uint32_t* b_vals, size_t n,
                                 int32_t* out_keys, uint32_t* out_vals, void* ws, size_t ws_bytes,
                                 comerge_stream_t stream);
int comerge_cuda_merge_pairs_u32(const uint32_t* a_keys, const uint32_t* a_vals, size_t m,
                                 const uint32_t* b_keys, const uint32_t* b_vals, size_t n,
                                 uint32_t* out_keys, uint32_t* out_vals, void* ws,
                                 size_t ws_bytes, comerge_stream_t stream);
int comerge_cuda_merge_pairs_u64(const uint64_t* a_keys, const uint32_t* a_vals, size_t m,
                                 const uint64_t* b_keys, const uint32_t* b_vals, size_t n,
                                 uint64_t* out_keys, uint32_t* out_vals, void* ws,
                                 size_t ws_bytes, comerge_stream_t stream);

/* Key-value RECORDS merged by key -- the reference's own key-value call
 * shape: merge_parallel<T>(a, b, out, workers, less) over a struct with a
 * key-only less (tagged<K> / tagged_key_less, oracle.hpp:22-37;
 * parallel.hpp:304-317).  A record is the key at offset 0 followed by its
 * payload bytes, which travel with it untouched (padding included):
 *   comerge_rec_i32 / _u32  8 bytes  {key, uint32 val}
 *   comerge_rec_u64        16 bytes  {uint64 key, uint32 val, uint32 pad}
 *                                    (the C/C++ layout of {uint64_t, uint32_t})
 * Ties go to A (stable).  Arrays may start at any record offset into an
 * allocation (4-byte aligned for 8-byte records, 8-byte aligned for 16-byte
 * ones).  Workspace from comerge_cuda_records_workspace_bytes. */
typedef struct comerge_rec_i32 { int32_t key; uint32_t val; } comerge_rec_i32;
typedef struct comerge_rec_u32 { uint32_t key; uint32_t val; } comerge_rec_u32;
typedef struct comerge_rec_u64 { uint64_t key; uint32_t val; uint32_t pad; } comerge_rec_u64;
size_t comerge_cuda_records_workspace_bytes(size_t m, size_t n, int key_kind);
int comerge_cuda_merge_records_i32(const comerge_rec_i32* a, size_t m, const comerge_rec_i32* b,
                                   size_t n, comerge_rec_i32* out, void* ws, size_t ws_bytes,
                                   comerge_stream_t stream);
int comerge_cuda_merge_records_u32(const comerge_rec_u32* a, size_t m, const comerge_rec_u32* b,
                                   size_t n, comerge_rec_u32* out, void* ws, size_t ws_bytes,
                                   comerge_stream_t stream);
int comerge_cuda_merge_records_u64(const comerge_rec_u64* a, size_t m, const comerge_rec_u64* b,
                                   size_t n, comerge_rec_u64* out, void* ws, size_t ws_bytes,
                                   comerge_stream_t stream);

/* 12-byte records {32-bit key, 8 payload bytes}: the layout of the
 * reference's own tagged<int32_t> / tagged<uint32_t> (key, origin byte + 3
 * padding bytes, uint32 index; oracle.hpp:22-27), so a caller's
 * std::vector<tagged<int32_t>> is merged in place of
 * comerge::merge_parallel(a, b, out, workers, tagged_key_less{}).  4-byte
 * aligned arrays.  Workspace from comerge_cuda_records12_workspace_bytes. */
typedef struct comerge_rec12_i32 { int32_t key; uint32_t w[2]; } comerge_rec12_i32;
typedef struct comerge_rec12_u32 { uint32_t key; uint32_t w[2]; } comerge_rec12_u32;
size_t comerge_cuda_records12_workspace_bytes(size_t m, size_t n);
int comerge_cuda_merge_records12_i32(const comerge_rec12_i32* a, size_t m,
                                     const comerge_rec12_i32* b, size_t n, comerge_rec12_i32* out,
                                     void* ws, size_t ws_bytes, comerge_stream_t stream);
int comerge_cuda_merge_records12_u32(const comerge_rec12_u32* a, size_t m,
                                     const comerge_rec12_u32* b, size_t n, comerge_rec12_u32* out,
                                     void* ws, size_t ws_bytes, comerge_stream_t stream);

/* Segmented batch: pair s merges a[a_off[s], a_off[s+1]) with
 * b[b_off[s], b_off[s+1]) into out[a_off[s]+b_off[s], ...).  a_off / b_off
 * hold nseg+1 nondecreasing offsets (device memory) with a_off[0] =
 * b_off[0] = 0, a_off[nseg] = m and b_off[nseg] = n (the caller passes m and
 * n so the call never synchronises).  One launch for all pairs.  The reference has no batched
 * API; this replaces a loop of comerge::stable_merge (merge.hpp:52-68). */
int comerge_cuda_merge_segmented_i32(const int32_t* a, const uint64_t* a_off, size_t m,
                                     const int32_t* b, const uint64_t* b_off, size_t n,
                                     size_t nseg, int32_t* out, void* ws, size_t ws_bytes,
                                     comerge_stream_t stream);
int comerge_cuda_merge_segmented_u32(const uint32_t* a, const uint64_t* a_off, size_t m,
                                     const uint32_t* b, const uint64_t* b_off, size_t n,
                                     size_t nseg, uint32_t* out, void* ws, size_t ws_bytes,
                                     comerge_stream_t stream);

/* Stable merge sort (the merge path's natural consumer; no
 * reference counterpart -- its result is std::stable_sort's, i.e. repeated
 * stable_merge of adjacent runs, merge.hpp:52-68): keys[0, n) -> out[0, n),
 * out may equal keys (in place) but must not partially overlap it.  Block
 * sort of runs in shared memory, then log2(n / run) merge passes of the tile
 * pipeline.  Workspace from comerge_cuda_sort_workspace_bytes (NULL: the
 * library pool).  Up to 2^40 keys. */
size_t comerge_cuda_sort_workspace_bytes(size_t n, int key_kind);
int comerge_cuda_sort_keys_i32(const int32_t* keys, size_t n, int32_t* out, void* ws,
                               size_t ws_bytes, comerge_stream_t stream);
int comerge_cuda_sort_keys_u32(const uint32_t* keys, size_t n, uint32_t* out, void* ws,
                               size_t ws_bytes, comerge_stream_t stream);
int comerge_cuda_sort_keys_u64(const uint64_t* keys, size_t n, uint64_t* out, void* ws,
                               size_t ws_bytes, comerge_stream_t stream);
/* Stable key-value merge sort: the uint32 payload moves with its key, equal
 * keys keep their input order (std::stable_sort of {key, val} by key).  Out
 * arrays may equal the inputs. */
size_t comerge_cuda_sort_pairs_workspace_bytes(size_t n, int key_kind);
int comerge_cuda_sort_pairs_i32(const int32_t* keys, const uint32_t* vals, size_t n,
                                int32_t* out_keys, uint32_t* out_vals, void* ws, size_t ws_bytes,
                                comerge_stream_t stream);
int comerge_cuda_sort_pairs_u32(const uint32_t* keys, const uint32_t* vals, size_t n,
                                uint32_t* out_keys, uint32_t* out_vals, void* ws, size_t ws_bytes,
                                comerge_stream_t stream);
int comerge_cuda_sort_pairs_u64(const uint64_t* keys, const uint32_t* vals, size_t n,
                                uint64_t* out_keys, uint32_t* out_vals, void* ws, size_t ws_bytes,
                                comerge_stream_t stream);

/* Batched co-rank (Algorithm 1 exactly, corank.hpp:72-121): for each
 * ranks[q] (device array) writes j (k = ranks[q] - j) and, if the pointers
 * are non-NULL, the reference's co_rank_stats {iterations, comparisons}.
 * A rank > m+n yields out_j = UINT64_MAX (the reference throws
 * std::out_of_range there; the synchronous comerge_co_rank_* below returns
 * COMERGE_E_RANGE). */
int comerge_cuda_co_rank_batch_i32(const uint64_t* ranks, size_t count, const int32_t* a,
                                   size_t m, const int32_t* b, size_t n, uint64_t* out_j,
                                   uint32_t* out_iterations, uint32_t* out_comparisons,
                                   comerge_stream_t stream);
int comerge_cuda_co_rank_batch_u32(const uint64_t* ranks, size_t count, const uint32_t* a,
                                   size_t m, const uint32_t* b, size_t n, uint64_t* out_j,
                                   uint32_t* out_iterations, uint32_t* out_comparisons,
                                   comerge_stream_t stream);
int comerge_cuda_co_rank_batch_u64(const uint64_t* ranks, size_t count, const uint64_t* a,
                                   size_t m, const uint64_t* b, size_t n, uint64_t* out_j,
                                   uint32_t* out_iterations, uint32_t* out_comparisons,
                                   comerge_stream_t stream);

/* -------------------------------- synchronous mirrors of the templates */

/* comerge::merge_report (parallel.hpp:44-55) in C: the vectors are
 * caller-provided arrays (block_sizes: `workers` entries, corank_iterations:
 * 2*workers, or `workers` when synced), either may be NULL. */
typedef struct comerge_merge_report {
    uint64_t m;
    uint64_t n;
    uint64_t workers;
    uint64_t wall_ns;     /* merge region on the device (CUDA events)        */
    uint64_t e2e_ns;      /* whole call incl. host<->device copies           */
    uint64_t h2d_bytes;   /* bytes copied host->device by this call          */
    uint64_t d2h_bytes;   /* bytes copied device->host by this call          */
    uint64_t tiles;       /* device output tiles (the GPU's unit of work)    */
} comerge_merge_report;

/* comerge::merge_parallel(a, b, out, workers) / merge_parallel_synced
 * (parallel.hpp:304-336).  Pointers may be host or device memory (mixed is
 * allowed); host data is staged through the device inside the call.
 * `workers` >= 1 defines the reported block partition (partition_output,
 * parallel.hpp:60-67) exactly as in the reference; the device always
 * merges in its own fixed-size tiles, so the output is worker-independent
 * (acceptance criterion 6). */
int comerge_merge_parallel_i32(const int32_t* a, size_t m, const int32_t* b, size_t n,
                               int32_t* out, size_t out_len, size_t workers, int synced,
                               comerge_merge_report* report, uint64_t* block_sizes,
                               uint32_t* corank_iterations);
int comerge_merge_parallel_u32(const uint32_t* a, size_t m, const uint32_t* b, size_t n,
                               uint32_t* out, size_t out_len, size_t workers, int synced,
                               comerge_merge_report* report, uint64_t* block_sizes,
                               uint32_t* corank_iterations);
int comerge_merge_parallel_u64(const uint64_t* a, size_t m, const uint64_t* b, size_t n,
                               uint64_t* out, size_t out_len, size_t workers, int synced,
                               comerge_merge_report* report, uint64_t* block_sizes,
                               uint32_t* corank_iterations);
int comerge_merge_parallel_pairs_i32(const int32_t* a_keys, const uint32_t* a_vals, size_t m,
                                     const int32_t* b_keys, const uint32_t* b_vals, size_t n,
                                     int32_t* out_keys, uint32_t* out_vals, size_t out_len,
                                     size_t workers, comerge_merge_report* report);
int comerge_merge_parallel_pairs_u32(const uint32_t* a_keys, const uint32_t* a_vals, size_t m,
                                     const uint32_t* b_keys, const uint32_t* b_vals, size_t n,
                                     uint32_t* out_keys, uint32_t* out_vals, size_t out_len,
                                     size_t workers, comerge_merge_report* report);
int comerge_merge_parallel_pairs_u64(const uint64_t* a_keys, const uint32_t* a_vals, size_t m,
                                     const uint64_t* b_keys, const uint32_t* b_vals, size_t n,
                                     uint64_t* out_keys, uint32_t* out_vals, size_t out_len,
                                     size_t workers, comerge_merge_report* report);

/* comerge::merge_parallel over key-value records (see comerge_rec_*): host or
 * device pointers, the report as comerge_merge_parallel_*. */
int comerge_merge_parallel_records_i32(const comerge_rec_i32* a, size_t m,
                                       const comerge_rec_i32* b, size_t n, comerge_rec_i32* out,
                                       size_t out_len, size_t workers, int synced,
                                       comerge_merge_report* report, uint64_t* block_sizes,
                                       uint32_t* corank_iterations);
int comerge_merge_parallel_records_u32(const comerge_rec_u32* a, size_t m,
                                       const comerge_rec_u32* b, size_t n, comerge_rec_u32* out,
                                       size_t out_len, size_t workers, int synced,
                                       comerge_merge_report* report, uint64_t* block_sizes,
                                       uint32_t* corank_iterations);
int comerge_merge_parallel_records_u64(const comerge_rec_u64* a, size_t m,
                                       const comerge_rec_u64* b, size_t n, comerge_rec_u64* out,
                                       size_t out_len, size_t workers, int synced,
                                       comerge_merge_report* report, uint64_t* block_sizes,
                                       uint32_t* corank_iterations);
int comerge_merge_parallel_records12_i32(const comerge_rec12_i32* a, size_t m,
                                         const comerge_rec12_i32* b, size_t n,
                                         comerge_rec12_i32* out, size_t out_len, size_t workers,
                                         int synced, comerge_merge_report* report,
                                         uint64_t* block_sizes, uint32_t* corank_iterations);
int comerge_merge_parallel_records12_u32(const comerge_rec12_u32* a, size_t m,
                                         const comerge_rec12_u32* b, size_t n,
                                         comerge_rec12_u32* out, size_t out_len, size_t workers,
                                         int synced, comerge_merge_report* report,
                                         uint64_t* block_sizes, uint32_t* corank_iterations);

/* Segmented batch with HOST (or device) buffers -- the reference's C5
 * baseline is a loop of comerge::stable_merge over independent pairs
 * (merge.hpp:52-68); this is the same batch in one call: pair s merges
 * a[a_off[s], a_off[s+1]) with b[b_off[s], b_off[s+1]) into
 * out[a_off[s] + b_off[s], ...).  Offsets (nseg + 1 each, host or device)
 * must be nondecreasing, start at 0 and end within the inputs (E_INVALID
 * otherwise).  Host inputs of >= 2^20 elements stream through a chunked
 * H2D / merge / D2H pipeline; report fields as comerge_merge_parallel_*
 * (workers = 1, no block sizes). */
int comerge_merge_segmented_host_i32(const int32_t* a, const uint64_t* a_off, size_t m,
                                     const int32_t* b, const uint64_t* b_off, size_t n,
                                     size_t nseg, int32_t* out, size_t out_len,
                                     comerge_merge_report* report);
int comerge_merge_segmented_host_u32(const uint32_t* a, const uint64_t* a_off, size_t m,
                                     const uint32_t* b, const uint64_t* b_off, size_t n,
                                     size_t nseg, uint32_t* out, size_t out_len,
                                     comerge_merge_report* report);

/* merge_options (parallel.hpp:38-42) for the full-report entry points. */
typedef struct comerge_merge_options {
    int synced;             /* merge_parallel_synced semantics (parallel.hpp:323-336)  */
    int count_comparisons;  /* merge_options::count_comparisons: fill *comparisons      */
} comerge_merge_options;

/* merge_parallel / merge_parallel_synced with every report field, keys only
 * (payload pointers NULL) or keys + uint32 payloads (all three non-NULL).
 * With opts->count_comparisons, *comparisons receives the reference's total
 * (parallel.hpp:270-280): Algorithm 1's comparisons at every co-rank its
 * workers make plus every block's merge_into (merge.hpp:18-33), computed
 * exactly from the block windows (one binary search per block).  opts may be
 * NULL (unsynced, no counting). */
int comerge_merge_parallel_ex_i32(const int32_t* a, const uint32_t* a_vals, size_t m,
                                  const int32_t* b, const uint32_t* b_vals, size_t n,
                                  int32_t* out, uint32_t* out_vals, size_t out_len,
                                  size_t workers, const comerge_merge_options* opts,
                                  comerge_merge_report* report, uint64_t* block_sizes,
                                  uint32_t* corank_iterations, uint64_t* comparisons);
int comerge_merge_parallel_ex_u32(const uint32_t* a, const uint32_t* a_vals, size_t m,
                                  const uint32_t* b, const uint32_t* b_vals, size_t n,
                                  uint32_t* out, uint32_t* out_vals, size_t out_len,
                                  size_t workers, const comerge_merge_options* opts,
                                  comerge_merge_report* report, uint64_t* block_sizes,
                                  uint32_t* corank_iterations, uint64_t* comparisons);
int comerge_merge_parallel_ex_u64(const uint64_t* a, const uint32_t* a_vals, size_t m,
                                  const uint64_t* b, const uint32_t* b_vals, size_t n,
                                  uint64_t* out, uint32_t* out_vals, size_t out_len,
                                  size_t workers, const comerge_merge_options* opts,
                                  comerge_merge_report* report, uint64_t* block_sizes,
                                  uint32_t* corank_iterations, uint64_t* comparisons);

/* Output ranks [out_begin, out_end) of the stable merge of A and B into
 * out[0, out_end - out_begin), where A (B) is the concatenation of na (nb) <= 8
 * device arrays -- e.g. every GPU's piece of a distributed input, peer
 * pointers mapped over NVLink (CUDA IPC): the multi-GPU split of Algorithm 2,
 * one launch per GPU for its own output range, no data-path collective.
 * Pieces and out 16-byte aligned; every piece but the last a multiple of 16
 * bytes.  Piece pointer / length arrays are host memory.  Workspace: the
 * tail slots of the pipeline (comerge_cuda_merge_workspace_bytes(m, n, ...)
 * is enough), NULL = library pool. */
int comerge_cuda_merge_keys_pieces_i32(const int32_t* const* a_pieces, const uint64_t* a_lens,
                                       int na, const int32_t* const* b_pieces,
                                       const uint64_t* b_lens, int nb, uint64_t out_begin,
                                       uint64_t out_end, int32_t* out, void* ws, size_t ws_bytes,
                                       comerge_stream_t stream);
int comerge_cuda_merge_keys_pieces_u32(const uint32_t* const* a_pieces, const uint64_t* a_lens,
                                       int na, const uint32_t* const* b_pieces,
                                       const uint64_t* b_lens, int nb, uint64_t out_begin,
                                       uint64_t out_end, uint32_t* out, void* ws, size_t ws_bytes,
                                       comerge_stream_t stream);
int comerge_cuda_merge_keys_pieces_u64(const uint64_t* const* a_pieces, const uint64_t* a_lens,
                                       int na, const uint64_t* const* b_pieces,
                                       const uint64_t* b_lens, int nb, uint64_t out_begin,
                                       uint64_t out_end, uint64_t* out, void* ws, size_t ws_bytes,
                                       comerge_stream_t stream);

/* Key-value form: payload pieces cut like their key pieces; every piece but
 * the last a multiple of 4 elements and of 16 bytes of keys. */
int comerge_cuda_merge_pairs_pieces_i32(const int32_t* const* a_pieces,
                                        const uint32_t* const* a_val_pieces,
                                        const uint64_t* a_lens, int na,
                                        const int32_t* const* b_pieces,
                                        const uint32_t* const* b_val_pieces,
                                        const uint64_t* b_lens, int nb, uint64_t out_begin,
                                        uint64_t out_end, int32_t* out_keys, uint32_t* out_vals,
                                        void* ws, size_t ws_bytes, comerge_stream_t stream);
int comerge_cuda_merge_pairs_pieces_u32(const uint32_t* const* a_pieces,
                                        const uint32_t* const* a_val_pieces,
                                        const uint64_t* a_lens, int na,
                                        const uint32_t* const* b_pieces,
                                        const uint32_t* const* b_val_pieces,
                                        const uint64_t* b_lens, int nb, uint64_t out_begin,
                                        uint64_t out_end, uint32_t* out_keys, uint32_t* out_vals,
                                        void* ws, size_t ws_bytes, comerge_stream_t stream);
int comerge_cuda_merge_pairs_pieces_u64(const uint64_t* const* a_pieces,
                                        const uint32_t* const* a_val_pieces,
                                        const uint64_t* a_lens, int na,
                                        const uint64_t* const* b_pieces,
                                        const uint32_t* const* b_val_pieces,
                                        const uint64_t* b_lens, int nb, uint64_t out_begin,
                                        uint64_t out_end, uint64_t* out_keys, uint32_t* out_vals,
                                        void* ws, size_t ws_bytes, comerge_stream_t stream);

/* comerge::plan(a, b, workers) (parallel.hpp:94-115): blocks[7*r .. 7*r+6] =
 * {worker, out_begin, out_end, a_begin, a_end, b_begin, b_end} for every
 * worker r (block_assignment, parallel.hpp:70-84).  Host or device inputs,
 * staged once; all co-ranks in one batched device launch. */
int comerge_plan_i32(const int32_t* a, size_t m, const int32_t* b, size_t n, size_t workers,
                     uint64_t* blocks);
int comerge_plan_u32(const uint32_t* a, size_t m, const uint32_t* b, size_t n, size_t workers,
                     uint64_t* blocks);
int comerge_plan_u64(const uint64_t* a, size_t m, const uint64_t* b, size_t n, size_t workers,
                     uint64_t* blocks);

/* comerge::co_rank(target, a, b, less, stats) (corank.hpp:128-133); host or
 * device pointers; iterations / comparisons may be NULL. */
int comerge_co_rank_i32(uint64_t target, const int32_t* a, size_t m, const int32_t* b, size_t n,
                        uint64_t* j, uint64_t* k, uint32_t* iterations, uint32_t* comparisons);
int comerge_co_rank_u32(uint64_t target, const uint32_t* a, size_t m, const uint32_t* b,
                        size_t n, uint64_t* j, uint64_t* k, uint32_t* iterations,
                        uint32_t* comparisons);
int comerge_co_rank_u64(uint64_t target, const uint64_t* a, size_t m, const uint64_t* b,
                        size_t n, uint64_t* j, uint64_t* k, uint32_t* iterations,
                        uint32_t* comparisons);

/* The same templates instantiated with a record type and a key-only less
 * (the reference's tagged<K> / tagged_key_less, oracle.hpp:22-37; the
 * comparator known-answer test of corank_test.cpp:205-214): arrays of
 * `record_bytes`-byte records with the key at offset 0 -- 8 or 12 bytes for
 * _i32 / _u32, 16 for _u64 (COMERGE_E_INVALID otherwise) -- host or device
 * pointers.  Only keys are compared, so j, k, iterations, comparisons and the
 * plan equal those of the records' key arrays.
 *   comerge_co_rank_records_*         co_rank / co_rank_counted  corank.hpp:128-147
 *   comerge_plan_records_*            plan                       parallel.hpp:94-115
 *   comerge_cuda_co_rank_batch_records_*  batched, device arrays, async
 *   comerge_merge_parallel_records_ex_*   merge_parallel / _synced with
 *       merge_options (count_comparisons) and every report field,
 *       parallel.hpp:304-336 */
int comerge_co_rank_records_i32(uint64_t target, const void* a, size_t m, const void* b,
                                size_t n, size_t record_bytes, uint64_t* j, uint64_t* k,
                                uint32_t* iterations, uint32_t* comparisons);
int comerge_plan_records_i32(const void* a, size_t m, const void* b, size_t n,
                             size_t record_bytes, size_t workers, uint64_t* blocks);
int comerge_cuda_co_rank_batch_records_i32(const uint64_t* ranks, size_t count, const void* a,
                                           size_t m, const void* b, size_t n,
                                           size_t record_bytes, uint64_t* out_j,
                                           uint32_t* out_iterations, uint32_t* out_comparisons,
                                           comerge_stream_t stream);
int comerge_merge_parallel_records_ex_i32(const void* a, size_t m, const void* b, size_t n,
                                          void* out, size_t out_len, size_t record_bytes,
                                          size_t workers, const comerge_merge_options* opts,
                                          comerge_merge_report* report, uint64_t* block_sizes,
                                          uint32_t* corank_iterations, uint64_t* comparisons);
int comerge_co_rank_records_u32(uint64_t target, const void* a, size_t m, const void* b,
                                size_t n, size_t record_bytes, uint64_t* j, uint64_t* k,
                                uint32_t* iterations, uint32_t* comparisons);
int comerge_plan_records_u32(const void* a, size_t m, const void* b, size_t n,
                             size_t record_bytes, size_t workers, uint64_t* blocks);
int comerge_cuda_co_rank_batch_records_u32(const uint64_t* ranks, size_t count, const void* a,
                                           size_t m, const void* b, size_t n,
                                           size_t record_bytes, uint64_t* out_j,
                                           uint32_t* out_iterations, uint32_t* out_comparisons,
                                           comerge_stream_t stream);
int comerge_merge_parallel_records_ex_u32(const void* a, size_t m, const void* b, size_t n,
                                          void* out, size_t out_len, size_t record_bytes,
                                          size_t workers, const comerge_merge_options* opts,
                                          comerge_merge_report* report, uint64_t* block_sizes,
                                          uint32_t* corank_iterations, uint64_t* comparisons);
int comerge_co_rank_records_u64(uint64_t target, const void* a, size_t m, const void* b,
                                size_t n, size_t record_bytes, uint64_t* j, uint64_t* k,
                                uint32_t* iterations, uint32_t* comparisons);
int comerge_plan_records_u64(const void* a, size_t m, const void* b, size_t n,
                             size_t record_bytes, size_t workers, uint64_t* blocks);
int comerge_cuda_co_rank_batch_records_u64(const uint64_t* ranks, size_t count, const void* a,
                                           size_t m, const void* b, size_t n,
                                           size_t record_bytes, uint64_t* out_j,
                                           uint32_t* out_iterations, uint32_t* out_comparisons,
                                           comerge_stream_t stream);
int comerge_merge_parallel_records_ex_u64(const void* a, size_t m, const void* b, size_t n,
                                          void* out, size_t out_len, size_t record_bytes,
                                          size_t workers, const comerge_merge_options* opts,
                                          comerge_merge_report* report, uint64_t* block_sizes,
                                          uint32_t* corank_iterations, uint64_t* comparisons);

/* comerge::partition_output(total, workers, r) (parallel.hpp:60-67). */
int comerge_partition_output(uint64_t total, uint64_t workers, uint64_t r, uint64_t* out);

#ifdef __cplusplus
}
#endif

#endif /* COMERGE_CUDA_H */
