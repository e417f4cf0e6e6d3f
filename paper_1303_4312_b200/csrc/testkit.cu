// testkit.cu -- device-side input generation and full-size verification for
// tests and bench (include/comerge_cuda_testkit.h).  Not on the merge path.
//
// Generation restates the reference's seeded recipe on the GPU:
//   stream(seed, lane) = splitmix64{mix64(seed) ^ mix64(lane+1)}  generate.cpp:17-19
//   draw t (t = 1, 2, ...) = finaliser(state0 + t * golden)        keys.hpp:28-34
//   below(width): reject draws >= width * (2^64-1 / width)         keys.hpp:36-42
// The t-th raw draw is counter-based, so draws are produced in parallel;
// rejection is reproduced exactly by a stable compaction of accepted draws.
// The result is sorted with cub radix sort (a keys-only sort is unique, so
// it equals the reference's std::sort, generate.cpp:27).
#include <cuda_runtime.h>

#include <cub/device/device_merge_sort.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cstdint>
#include <string>

#include "../../include/comerge_cuda_testkit.h"

namespace {

thread_local std::string g_tk_error;

int tk_fail(cudaError_t e, const char* where) {
    g_tk_error = std::string(where) + ": " + cudaGetErrorString(e);
    return COMERGE_E_CUDA;
}

__host__ __device__ __forceinline__ uint64_t fin64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    return fin64(x + 0x9e3779b97f4a7c15ULL);
}

__global__ void draw_kernel(uint64_t state0, uint64_t count, uint64_t width, uint64_t limit,
                            uint64_t* __restrict__ vals, uint8_t* __restrict__ keep) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const uint64_t r = fin64(state0 + (t + 1) * 0x9e3779b97f4a7c15ULL);
    const bool ok = width == 0 || r < limit;
    keep[t] = ok;
    vals[t] = width == 0 ? r : r % width;
}

template <typename K>
__global__ void narrow_kernel(const uint64_t* __restrict__ in, uint64_t len, K* __restrict__ out) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < len) out[t] = K(uint32_t(in[t]));
}

// out[i] = (i + offset) / run_len: sorted keys in runs of equal values
template <typename K>
__global__ void fill_runs_kernel(K* out, uint64_t len, uint64_t run_len, uint64_t offset) {
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len;
         i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = K((i + offset) / run_len);
}

__global__ void iota_kernel(uint32_t* out, uint64_t len, uint32_t tag) {
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < len) out[t] = uint32_t(t) | tag;
}

template <typename K>
__device__ __forceinline__ uint64_t widen(K k) {
    if constexpr (sizeof(K) == 4 && K(-1) < K(0))
        return uint64_t(int64_t(k));
    else
        return uint64_t(k);
}

template <typename K>
__global__ void checksum_kernel(const K* __restrict__ keys, uint64_t len,
                                unsigned long long* acc) {
    uint64_t sum = 0;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < len;
         t += uint64_t(gridDim.x) * blockDim.x)
        sum += mix64(widen(keys[t]));
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(acc, (unsigned long long)sum);
}

template <typename K>
__global__ void unsorted_kernel(const K* __restrict__ keys, uint64_t len, unsigned long long* acc) {
    unsigned long long bad = 0;
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t + 1 < len;
         t += uint64_t(gridDim.x) * blockDim.x)
        bad += keys[t + 1] < keys[t];
    for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(acc, bad);
}

// counts: [0] unsorted, [1] equal-key neighbours whose tags do not increase,
// [2] key != source key, [3] tag out of range.  All zero <=> the output is the
// unique stable merge: a repeated tag would sit twice in one equal-key run
// (same source key) and break [1], so tags form a permutation, and within
// every equal-key run A tags (< 2^31) precede B tags in source order.
template <typename K>
__global__ void verify_pairs_kernel(const K* __restrict__ a, uint64_t m, const K* __restrict__ b,
                                    uint64_t n, const K* __restrict__ ok,
                                    const uint32_t* __restrict__ ov, unsigned long long* counts) {
    const uint64_t total = m + n;
    unsigned long long c[4] = {0, 0, 0, 0};
    for (uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += uint64_t(gridDim.x) * blockDim.x) {
        const K key = ok[t];
        const uint32_t tag = ov[t];
        const bool from_b = tag & 0x80000000u;
        const uint64_t idx = tag & 0x7fffffffu;
        if (from_b ? idx >= n : idx >= m) {
            c[3]++;
        } else if ((from_b ? b[idx] : a[idx]) != key) {
            c[2]++;
        }
        if (t + 1 < total) {
            const K nk = ok[t + 1];
            const uint32_t nt = ov[t + 1];
            if (nk < key) c[0]++;
            if (nk == key && !(nt > tag)) c[1]++;
        }
    }
    for (int i = 0; i < 4; ++i) {
        unsigned long long v = c[i];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(counts + i, v);
    }
}

unsigned grid_for(uint64_t n, unsigned threads) {
    uint64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > 148u * 16u) g = 148u * 16u;
    return unsigned(g);
}

// Accepted draws 0..len-1 of stream(seed, lane) (below(width) / next()),
// in stream order, into a fresh device buffer *out (caller frees).
int draw_accepted(uint64_t seed, uint64_t lane, size_t len, uint64_t width, uint64_t** out,
                  cudaStream_t s) {
    *out = nullptr;
    if (len > (uint64_t(1) << 31) - (uint64_t(1) << 20)) {  // CUB selects count in int
        g_tk_error = "testkit: at most 2^31 - 2^20 draws per call";
        return COMERGE_E_LENGTH;
    }
    const uint64_t state0 = mix64(seed) ^ mix64(lane + 1);
    const uint64_t limit = width ? width * (UINT64_MAX / width) : 0;
    const long double p_rej =
        width ? (long double)(UINT64_MAX - limit) / 18446744073709551616.0L : 0;
    uint64_t slack = uint64_t(len * p_rej * 2.0L) + 1024;
    for (int attempt = 0; attempt < 4; ++attempt, slack *= 4) {
        const uint64_t count = len + slack;
        uint64_t *vals = nullptr, *sel = nullptr;
        uint8_t* keep = nullptr;
        int* nsel = nullptr;
        void* tmp = nullptr;
        size_t tmp_bytes = 0;
        cudaError_t e = cudaMallocAsync(&vals, count * 8, s);
        if (!e) e = cudaMallocAsync(&sel, count * 8, s);
        if (!e) e = cudaMallocAsync(&keep, count, s);
        if (!e) e = cudaMallocAsync(&nsel, sizeof(int), s);
        if (e) return tk_fail(e, "testkit: alloc");
        draw_kernel<<<unsigned((count + 255) / 256), 256, 0, s>>>(state0, count, width, limit,
                                                                 vals, keep);
        cub::DeviceSelect::Flagged(nullptr, tmp_bytes, vals, keep, sel, nsel, int(count), s);
        e = cudaMallocAsync(&tmp, tmp_bytes, s);
        if (e) return tk_fail(e, "testkit: alloc");
        cub::DeviceSelect::Flagged(tmp, tmp_bytes, vals, keep, sel, nsel, int(count), s);
        int h_nsel = 0;
        cudaMemcpyAsync(&h_nsel, nsel, sizeof(int), cudaMemcpyDeviceToHost, s);
        e = cudaStreamSynchronize(s);
        cudaFreeAsync(tmp, s);
        cudaFreeAsync(vals, s);
        cudaFreeAsync(keep, s);
        cudaFreeAsync(nsel, s);
        if (e) return tk_fail(e, "testkit: select");
        if (uint64_t(h_nsel) >= len) {
            *out = sel;
            return COMERGE_OK;
        }
        cudaFreeAsync(sel, s);
    }
    g_tk_error = "testkit: too many rejections";
    return COMERGE_E_CUDA;
}

template <typename K>
int generate_sorted(uint64_t seed, uint64_t lane, size_t len, uint64_t width, K* out,
                    cudaStream_t s) {
    if (len == 0) return COMERGE_OK;
    uint64_t* sel = nullptr;
    if (int rc = draw_accepted(seed, lane, len, width, &sel, s)) return rc;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cudaError_t e = cudaSuccess;
    if constexpr (sizeof(K) == 8) {
        cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, sel, reinterpret_cast<uint64_t*>(out),
                                       int(len), 0, 64, s);
        e = cudaMallocAsync(&tmp, tmp_bytes, s);
        if (e) return tk_fail(e, "testkit: alloc");
        cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, sel, reinterpret_cast<uint64_t*>(out),
                                       int(len), 0, 64, s);
    } else {
        K* narrow = nullptr;
        e = cudaMallocAsync(&narrow, len * sizeof(K), s);
        if (e) return tk_fail(e, "testkit: alloc");
        narrow_kernel<K><<<unsigned((len + 255) / 256), 256, 0, s>>>(sel, len, narrow);
        cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, narrow, out, int(len), 0, 32, s);
        e = cudaMallocAsync(&tmp, tmp_bytes, s);
        if (e) return tk_fail(e, "testkit: alloc");
        cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, narrow, out, int(len), 0, 32, s);
        cudaFreeAsync(narrow, s);
    }
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(sel, s);
    e = cudaGetLastError();
    return e ? tk_fail(e, "testkit: generate") : COMERGE_OK;
}

// Draw `total` keys of stream(seed, lane), narrow to K, sort each run
// [offsets[s], offsets[s+1]) independently (segmented batch inputs).
template <typename K>
int generate_runs(uint64_t seed, uint64_t lane, const uint64_t* offsets, size_t nseg,
                  size_t total, uint64_t width, K* out, cudaStream_t s) {
    if (total == 0) return COMERGE_OK;
    uint64_t* sel = nullptr;
    if (int rc = draw_accepted(seed, lane, total, width, &sel, s)) return rc;
    K* narrow = nullptr;
    cudaError_t e = cudaMallocAsync(&narrow, total * sizeof(K), s);
    if (e) return tk_fail(e, "testkit: alloc");
    narrow_kernel<K><<<unsigned((total + 255) / 256), 256, 0, s>>>(sel, total, narrow);
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tmp_bytes, narrow, out, int(total),
                                            int(nseg), offsets, offsets + 1, 0,
                                            int(8 * sizeof(K)), s);
    e = cudaMallocAsync(&tmp, tmp_bytes, s);
    if (e) return tk_fail(e, "testkit: alloc");
    cub::DeviceSegmentedRadixSort::SortKeys(tmp, tmp_bytes, narrow, out, int(total), int(nseg),
                                            offsets, offsets + 1, 0, int(8 * sizeof(K)), s);
    cudaFreeAsync(tmp, s);
    cudaFreeAsync(narrow, s);
    cudaFreeAsync(sel, s);
    e = cudaGetLastError();
    return e ? tk_fail(e, "testkit: generate runs") : COMERGE_OK;
}

}  // namespace

extern "C" {

const char* comerge_testkit_last_error(void) { return g_tk_error.c_str(); }

int comerge_testkit_generate_sorted(int key_kind, uint64_t seed, uint64_t lane, size_t len,
                                    uint64_t width, void* out, comerge_stream_t stream) {
    if (len > (size_t(1) << 31) - 4096) {
        g_tk_error = "testkit: len too large for one generation call";
        return COMERGE_E_INVALID;
    }
    switch (key_kind) {
    case COMERGE_KEY_I32:
        return generate_sorted<int32_t>(seed, lane, len, width, static_cast<int32_t*>(out), stream);
    case COMERGE_KEY_U32:
        return generate_sorted<uint32_t>(seed, lane, len, width, static_cast<uint32_t*>(out),
                                         stream);
    case COMERGE_KEY_U64:
        return generate_sorted<uint64_t>(seed, lane, len, width, static_cast<uint64_t*>(out),
                                         stream);
    }
    return COMERGE_E_INVALID;
}

int comerge_testkit_generate_raw(uint64_t seed, uint64_t lane, size_t len, uint64_t width,
                                 uint64_t* out, comerge_stream_t stream) {
    if (len == 0) return COMERGE_OK;
    uint64_t* sel = nullptr;
    if (int rc = draw_accepted(seed, lane, len, width, &sel, stream)) return rc;
    cudaMemcpyAsync(out, sel, len * 8, cudaMemcpyDeviceToDevice, stream);
    cudaFreeAsync(sel, stream);
    const cudaError_t e = cudaGetLastError();
    return e ? tk_fail(e, "testkit: raw") : COMERGE_OK;
}

int comerge_testkit_generate_runs(int key_kind, uint64_t seed, uint64_t lane,
                                  const uint64_t* offsets, size_t nseg, size_t total,
                                  uint64_t width, void* out, comerge_stream_t stream) {
    if (total > (size_t(1) << 31) - 4096) {
        g_tk_error = "testkit: total too large for one generation call";
        return COMERGE_E_INVALID;
    }
    switch (key_kind) {
    case COMERGE_KEY_I32:
        return generate_runs<int32_t>(seed, lane, offsets, nseg, total, width,
                                      static_cast<int32_t*>(out), stream);
    case COMERGE_KEY_U32:
        return generate_runs<uint32_t>(seed, lane, offsets, nseg, total, width,
                                       static_cast<uint32_t*>(out), stream);
    }
    return COMERGE_E_INVALID;
}

int comerge_testkit_fill_runs(int key_kind, size_t len, uint64_t run_len, uint64_t offset,
                              void* out, comerge_stream_t stream) {
    if (len == 0) return COMERGE_OK;
    if (run_len == 0) return tk_fail(cudaErrorInvalidValue, "testkit: run length 0");
    const unsigned g = grid_for(len, 256);
    switch (key_kind) {
    case COMERGE_KEY_I32:
        fill_runs_kernel<int32_t><<<g, 256, 0, stream>>>(static_cast<int32_t*>(out), len, run_len, offset);
        break;
    case COMERGE_KEY_U32:
        fill_runs_kernel<uint32_t><<<g, 256, 0, stream>>>(static_cast<uint32_t*>(out), len, run_len, offset);
        break;
    default:
        fill_runs_kernel<uint64_t><<<g, 256, 0, stream>>>(static_cast<uint64_t*>(out), len, run_len, offset);
        break;
    }
    const cudaError_t e = cudaGetLastError();
    return e ? tk_fail(e, "testkit: fill_runs") : COMERGE_OK;
}

int comerge_testkit_iota(uint32_t* out, size_t len, uint32_t tag, comerge_stream_t stream) {
    if (len == 0) return COMERGE_OK;
    iota_kernel<<<unsigned((len + 255) / 256), 256, 0, stream>>>(out, len, tag);
    const cudaError_t e = cudaGetLastError();
    return e ? tk_fail(e, "testkit: iota") : COMERGE_OK;
}

int comerge_testkit_verify_pairs(int key_kind, const void* a, size_t m, const void* b, size_t n,
                                 const void* ok, const uint32_t* ov, unsigned long long* counts,
                                 comerge_stream_t s) {
    cudaMemsetAsync(counts, 0, 4 * sizeof(unsigned long long), s);
    const unsigned g = grid_for(m + n, 256);
    switch (key_kind) {
    case COMERGE_KEY_I32:
        verify_pairs_kernel<int32_t><<<g, 256, 0, s>>>((const int32_t*)a, m, (const int32_t*)b, n,
                                                       (const int32_t*)ok, ov, counts);
        break;
    case COMERGE_KEY_U32:
        verify_pairs_kernel<uint32_t><<<g, 256, 0, s>>>((const uint32_t*)a, m, (const uint32_t*)b,
                                                        n, (const uint32_t*)ok, ov, counts);
        break;
    case COMERGE_KEY_U64:
        verify_pairs_kernel<uint64_t><<<g, 256, 0, s>>>((const uint64_t*)a, m, (const uint64_t*)b,
                                                        n, (const uint64_t*)ok, ov, counts);
        break;
    default: return COMERGE_E_INVALID;
    }
    const cudaError_t e = cudaGetLastError();
    return e ? tk_fail(e, "testkit: verify") : COMERGE_OK;
}

int comerge_testkit_checksum(int key_kind, const void* keys, size_t len, unsigned long long* acc,
                             comerge_stream_t s) {
    const unsigned g = grid_for(len, 256);
    switch (key_kind) {
    case COMERGE_KEY_I32: checksum_kernel<<<g, 256, 0, s>>>((const int32_t*)keys, len, acc); break;
    case COMERGE_KEY_U32: checksum_kernel<<<g, 256, 0, s>>>((const uint32_t*)keys, len, acc); break;
    case COMERGE_KEY_U64: checksum_kernel<<<g, 256, 0, s>>>((const uint64_t*)keys, len, acc); break;
    default: return COMERGE_E_INVALID;
    }
    const cudaError_t e = cudaGetLastError();
    return e ? tk_fail(e, "testkit: checksum") : COMERGE_OK;
}

int comerge_testkit_count_unsorted(int key_kind, const void* keys, size_t len,
                                   unsigned long long* acc, comerge_stream_t s) {
    const unsigned g = grid_for(len, 256);
    switch (key_kind) {
    case COMERGE_KEY_I32: unsorted_kernel<<<g, 256, 0, s>>>((const int32_t*)keys, len, acc); break;
    case COMERGE_KEY_U32: unsorted_kernel<<<g, 256, 0, s>>>((const uint32_t*)keys, len, acc); break;
    case COMERGE_KEY_U64: unsorted_kernel<<<g, 256, 0, s>>>((const uint64_t*)keys, len, acc); break;
    default: return COMERGE_E_INVALID;
    }
    const cudaError_t e = cudaGetLastError();
    return e ? tk_fail(e, "testkit: unsorted") : COMERGE_OK;
}

namespace {
struct less_i32 {
    __device__ bool operator()(int32_t x, int32_t y) const { return x < y; }
};

cudaError_t cub_sort(int alg, const int32_t* k, const uint32_t* v, int32_t* ok, uint32_t* ov,
                     size_t n, void* tmp, size_t& bytes, cudaStream_t s) {
    const int nn = int(n);
    switch (alg) {
        case 0: return cub::DeviceRadixSort::SortKeys(tmp, bytes, k, ok, nn, 0, 32, s);
        case 1: return cub::DeviceRadixSort::SortPairs(tmp, bytes, k, ok, v, ov, nn, 0, 32, s);
        case 2:
            return cub::DeviceMergeSort::SortKeysCopy(tmp, bytes, k, ok, nn, less_i32(), s);
        default:
            return cub::DeviceMergeSort::SortPairsCopy(tmp, bytes, k, v, ok, ov, nn, less_i32(), s);
    }
}
}  // namespace

size_t comerge_testkit_cub_sort_bytes(size_t n) {
    size_t most = 0;
    for (int alg = 0; alg < 4; ++alg) {
        size_t b = 0;
        if (cub_sort(alg, nullptr, nullptr, nullptr, nullptr, n, nullptr, b, nullptr) == cudaSuccess)
            most = b > most ? b : most;
    }
    return most;
}

int comerge_testkit_cub_sort(int alg, const int32_t* keys, const uint32_t* vals,
                             int32_t* out_keys, uint32_t* out_vals, size_t n, void* tmp,
                             size_t tmp_bytes, comerge_stream_t stream) {
    if (n > (size_t(1) << 31) - 1 || alg < 0 || alg > 3) {
        g_tk_error = "testkit: cub_sort arguments";
        return COMERGE_E_INVALID;
    }
    size_t b = tmp_bytes;
    const cudaError_t e = cub_sort(alg, keys, vals, out_keys, out_vals, n, tmp, b, stream);
    return e ? tk_fail(e, "testkit: cub sort") : COMERGE_OK;
}

}  // extern "C"
