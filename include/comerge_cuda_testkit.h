/*
 * comerge_cuda_testkit.h -- device-side test/bench utilities exported by
 * libcomerge_cuda.so.  NOT part of the merge path: seeded input generation
 * (the reference's splitmix64 recipe, generate.cpp:17-29 / keys.hpp:17-43)
 * and size-independent verification used by the full-size parity tests.
 */
#ifndef COMERGE_CUDA_TESTKIT_H
#define COMERGE_CUDA_TESTKIT_H

#include "comerge_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

/* out[0,len) = sorted( below(width) draws of stream(seed, lane) ) converted
 * to the key kind (width == 0: next()).  Identical to the reference's
 * sorted_uniform (generate.cpp:21-29) for u64; i32/u32 keep the low 32 bits. */
int comerge_testkit_generate_sorted(int key_kind, uint64_t seed, uint64_t lane, size_t len,
                                    uint64_t width, void* out, comerge_stream_t stream);

/* Unsorted accepted draws (uint64) of stream(seed, lane), in stream order.
 * The seeded generators take at most 2^31 - 2^20 draws per call. */
int comerge_testkit_generate_raw(uint64_t seed, uint64_t lane, size_t len, uint64_t width,
                                 uint64_t* out, comerge_stream_t stream);

/* `total` draws of stream(seed, lane) as int32/uint32 keys, each run
 * [offsets[s], offsets[s+1]) (device offsets, nseg+1 entries) sorted on its
 * own: the inputs of a segmented batch / merge-sort pass. */
int comerge_testkit_generate_runs(int key_kind, uint64_t seed, uint64_t lane,
                                  const uint64_t* offsets, size_t nseg, size_t total,
                                  uint64_t width, void* out, comerge_stream_t stream);

/* out[i] = (i + offset) / run_len as the key kind: sorted runs of equal keys
 * (inputs of any size without a sort, for the 64-bit-index tests). */
int comerge_testkit_fill_runs(int key_kind, size_t len, uint64_t run_len, uint64_t offset,
                              void* out, comerge_stream_t stream);

/* out[i] = i | tag  (payloads: A tag 0, B tag 1u<<31). */
int comerge_testkit_iota(uint32_t* out, size_t len, uint32_t tag, comerge_stream_t stream);

/* Full-size property check of a tagged key-value merge result (tags as in
 * comerge_testkit_iota).  counts (4 uint64, device, zeroed by the call):
 *   [0] positions with key[i] > key[i+1]
 *   [1] equal-key neighbours whose tags do not increase
 *   [2] positions whose key differs from the key its tag points at
 *   [3] tags out of range
 * All four are zero iff the output is the unique stable merge (a repeated
 * tag would appear twice in one equal-key run and trip [1]). */
int comerge_testkit_verify_pairs(int key_kind, const void* a_keys, size_t m, const void* b_keys,
                                 size_t n, const void* out_keys, const uint32_t* out_vals,
                                 unsigned long long* counts, comerge_stream_t stream);

/* Order-independent multiset checksum sum(mix64(key)) (keys.hpp:50-55),
 * int32 keys sign-extended; result added into *acc (device). */
const char* comerge_testkit_last_error(void);

int comerge_testkit_checksum(int key_kind, const void* keys, size_t len,
                             unsigned long long* acc, comerge_stream_t stream);

/* count of i with key[i] > key[i+1], added into *acc (device). */
int comerge_testkit_count_unsorted(int key_kind, const void* keys, size_t len,
                                   unsigned long long* acc, comerge_stream_t stream);

/* Library baselines for the merge sort (bench.py "sorts"): CUB on int32 keys
 * (+ uint32 payloads).  alg 0: DeviceRadixSort::SortKeys, 1: SortPairs,
 * 2: DeviceMergeSort::SortKeysCopy (std::less), 3: SortPairsCopy.  tmp holds
 * comerge_testkit_cub_sort_bytes(n) bytes (the largest of the four). */
size_t comerge_testkit_cub_sort_bytes(size_t n);
int comerge_testkit_cub_sort(int alg, const int32_t* keys, const uint32_t* vals,
                             int32_t* out_keys, uint32_t* out_vals, size_t n, void* tmp,
                             size_t tmp_bytes, comerge_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
