/*
 * comerge_oracle.c -- TEST ORACLE (CPU restatement of the reference path).
 *
 * Test infrastructure only: imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the checker.  Never part of the product.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj.  Parity is pinned against the
 * reference's own KATs and against the compiled reference (oracle/_ref),
 * see comerge_oracle.h.
 */
#include "comerge_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ keys */

/* include/comerge/keys.hpp:17-22 */
uint64_t oracle_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

typedef struct {
    uint64_t state;
} sm64;

/* include/comerge/keys.hpp:28-34 */
static uint64_t sm64_next(sm64* g) {
    g->state += 0x9e3779b97f4a7c15ULL;
    uint64_t x = g->state;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* include/comerge/keys.hpp:36-42: unbiased draw by rejection */
static uint64_t sm64_below(sm64* g, uint64_t bound) {
    const uint64_t limit = bound * (UINT64_MAX / bound);
    uint64_t x = sm64_next(g);
    while (x >= limit) x = sm64_next(g);
    return x % bound;
}

/* src/generate.cpp:17-19 */
static sm64 stream(uint64_t seed, uint64_t lane) {
    sm64 g;
    g.state = oracle_mix64(seed) ^ oracle_mix64(lane + 1);
    return g;
}

void oracle_generate_raw(uint64_t seed, uint64_t lane, uint64_t len, uint64_t width,
                         uint64_t* out) {
    sm64 g = stream(seed, lane);
    for (uint64_t i = 0; i < len; ++i) out[i] = width == 0 ? sm64_next(&g) : sm64_below(&g, width);
}

/* LSD radix sort on order-preserving unsigned images (stands in for the
 * reference's std::sort, generate.cpp:27; a keys-only sort is unique). */
static void radix_sort_u64(uint64_t* v, uint64_t len, int bytes) {
    uint64_t* tmp = (uint64_t*)malloc(len * sizeof(uint64_t) + 1);
    uint64_t* src = v;
    uint64_t* dst = tmp;
    for (int pass = 0; pass < bytes; ++pass) {
        uint64_t count[257];
        memset(count, 0, sizeof(count));
        const int sh = pass * 8;
        for (uint64_t i = 0; i < len; ++i) count[((src[i] >> sh) & 0xff) + 1]++;
        for (int d = 0; d < 256; ++d) count[d + 1] += count[d];
        for (uint64_t i = 0; i < len; ++i) dst[count[(src[i] >> sh) & 0xff]++] = src[i];
        uint64_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != v) memcpy(v, src, len * sizeof(uint64_t));
    free(tmp);
}

void oracle_generate_sorted(int kind, uint64_t seed, uint64_t lane, uint64_t len,
                            uint64_t width, void* out) {
    uint64_t* raw = (uint64_t*)malloc(len * sizeof(uint64_t) + 1);
    oracle_generate_raw(seed, lane, len, width, raw);
    if (kind == ORACLE_U64) {
        radix_sort_u64(raw, len, 8);
        memcpy(out, raw, len * sizeof(uint64_t));
    } else {
        /* map the key kind's order to unsigned 32-bit order */
        const uint32_t flip = kind == ORACLE_I32 ? 0x80000000u : 0u;
        for (uint64_t i = 0; i < len; ++i) raw[i] = (uint32_t)((uint32_t)raw[i] ^ flip);
        radix_sort_u64(raw, len, 4);
        uint32_t* o = (uint32_t*)out;
        for (uint64_t i = 0; i < len; ++i) o[i] = (uint32_t)raw[i] ^ flip;
    }
    free(raw);
}

/* include/comerge/keys.hpp:50-55 */
uint64_t oracle_multiset_checksum(int kind, const void* keys, uint64_t len) {
    uint64_t sum = 0;
    for (uint64_t i = 0; i < len; ++i) {
        uint64_t k;
        if (kind == ORACLE_I32) k = (uint64_t)(int64_t)((const int32_t*)keys)[i];
        else if (kind == ORACLE_U32) k = ((const uint32_t*)keys)[i];
        else k = ((const uint64_t*)keys)[i];
        sum += oracle_mix64(k);
    }
    return sum;
}

/* ------------------------------------------------------- typed algorithms */

#define DEFINE_TYPED(SUFFIX, K)                                                               \
    /* include/comerge/corank.hpp:72-121 (Algorithm 1) */                    \
    static void co_rank_##SUFFIX(uint64_t target, const K* a, uint64_t m, const K* b,          \
                                 uint64_t n, uint64_t* j_out, uint64_t* k_out, uint32_t* it,   \
                                 uint32_t* cmp) {                                              \
        uint64_t take_a = target < m ? target : m; /* :83 */                                   \
        uint64_t take_b = target - take_a;         /* :84 */                                   \
        uint64_t floor_a = target > n ? target - n : 0; /* :86 */                              \
        uint64_t floor_b = target > m ? target - m : 0; /* :87 */                              \
        uint32_t iterations = 0, comparisons = 0;                                              \
        for (;;) {                                                                             \
            /* guard 1 (strict), :93-94 */                                                     \
            if (take_a > 0 && take_b < n && (++comparisons, b[take_b] < a[take_a - 1])) {      \
                const uint64_t step = (take_a - floor_a + 1) / 2; /* :98 */                    \
                floor_b = take_b;                                                              \
                take_a -= step;                                                                \
                take_b += step;                                                                \
                ++iterations;                                                                  \
                /* guard 2 (non-strict), :103-104 */                                           \
            } else if (take_b > 0 && take_a < m &&                                             \
                       (++comparisons, !(b[take_b - 1] < a[take_a]))) {                        \
                const uint64_t step = (take_b - floor_b + 1) / 2; /* :108 */                   \
                floor_a = take_a;                                                              \
                take_a += step;                                                                \
                take_b -= step;                                                                \
                ++iterations;                                                                  \
            } else {                                                                           \
                break; /* :113-115 */                                                          \
            }                                                                                  \
        }                                                                                      \
        *j_out = take_a;                                                                       \
        *k_out = take_b;                                                                       \
        if (it) *it = iterations;                                                              \
        if (cmp) *cmp = comparisons;                                                           \
    }                                                                                          \
    /* include/comerge/merge.hpp:18-33: take from b only when b < a */                         \
    static void merge_into_##SUFFIX(const K* a, const uint32_t* av, uint64_t m, const K* b,    \
                                    const uint32_t* bv, uint64_t n, K* out, uint32_t* outv) {  \
        uint64_t x = 0, y = 0, o = 0;                                                          \
        while (x < m && y < n) {                                                               \
            if (b[y] < a[x]) {                                                                 \
                if (outv) outv[o] = bv[y];                                                     \
                out[o++] = b[y++];                                                             \
            } else {                                                                           \
                if (outv) outv[o] = av[x];                                                     \
                out[o++] = a[x++];                                                             \
            }                                                                                  \
        }                                                                                      \
        for (; x < m; ++x) {                                                                   \
            if (outv) outv[o] = av[x];                                                         \
            out[o++] = a[x];                                                                   \
        }                                                                                      \
        for (; y < n; ++y) {                                                                   \
            if (outv) outv[o] = bv[y];                                                         \
            out[o++] = b[y];                                                                   \
        }                                                                                      \
    }                                                                                          \
    /* the same loop with counting_compare (parallel.hpp:253-256): the number */               \
    /* of less() calls, i.e. loop passes before one side runs out */                           \
    static uint64_t merge_count_##SUFFIX(const K* a, uint64_t m, const K* b, uint64_t n) {     \
        uint64_t x = 0, y = 0, c = 0;                                                          \
        while (x < m && y < n) {                                                               \
            ++c;                                                                               \
            if (b[y] < a[x])                                                                   \
                ++y;                                                                           \
            else                                                                               \
                ++x;                                                                           \
        }                                                                                      \
        return c;                                                                              \
    }

DEFINE_TYPED(i32, int32_t)
DEFINE_TYPED(u32, uint32_t)
DEFINE_TYPED(u64, uint64_t)

static size_t key_size(int kind) { return kind == ORACLE_U64 ? 8 : 4; }

/* include/comerge/corank.hpp:67-70 */
static int check_total_length(uint64_t m, uint64_t n) {
    return m > UINT64_MAX - n ? ORACLE_E_LENGTH : ORACLE_OK;
}

int oracle_co_rank(int kind, uint64_t target, const void* a, uint64_t m, const void* b,
                   uint64_t n, uint64_t* j, uint64_t* k, uint32_t* iterations,
                   uint32_t* comparisons) {
    if (check_total_length(m, n)) return ORACLE_E_LENGTH;
    if (target > m + n) return ORACLE_E_RANGE; /* corank.hpp:78-79 */
    switch (kind) {
    case ORACLE_I32: co_rank_i32(target, a, m, b, n, j, k, iterations, comparisons); break;
    case ORACLE_U32: co_rank_u32(target, a, m, b, n, j, k, iterations, comparisons); break;
    case ORACLE_U64: co_rank_u64(target, a, m, b, n, j, k, iterations, comparisons); break;
    default: return ORACLE_E_INVALID;
    }
    return ORACLE_OK;
}

/* include/comerge/parallel.hpp:60-67 */
int oracle_partition_output(uint64_t total, uint64_t workers, uint64_t r, uint64_t* out) {
    if (workers == 0 || r > workers) return ORACLE_E_INVALID;
    *out = (uint64_t)((unsigned __int128)r * total / workers);
    return ORACLE_OK;
}

void oracle_merge_into(int kind, const void* a, const uint32_t* av, uint64_t m, const void* b,
                       const uint32_t* bv, uint64_t n, void* out, uint32_t* outv) {
    switch (kind) {
    case ORACLE_I32: merge_into_i32(a, av, m, b, bv, n, out, outv); break;
    case ORACLE_U32: merge_into_u32(a, av, m, b, bv, n, out, outv); break;
    case ORACLE_U64: merge_into_u64(a, av, m, b, bv, n, out, outv); break;
    }
}

/* merge_report with count_comparisons (parallel.hpp:180-282, simulated
 * mode): per worker r, co_rank both block ends (unsynced) or its begin only
 * (synced: the end is the next worker's begin, parallel.hpp:209-219), then the
 * counted merge of its block.  Writes block_sizes[workers],
 * iterations[2*workers or workers] and the total comparisons (any may be NULL). */
int oracle_merge_report(int kind, const void* a, uint64_t m, const void* b, uint64_t n,
                        uint64_t workers, int synced, uint64_t* block_sizes,
                        uint32_t* iterations, uint64_t* comparisons) {
    if (check_total_length(m, n)) return ORACLE_E_LENGTH;
    if (workers == 0) return ORACLE_E_INVALID;
    const size_t s = key_size(kind);
    const char* ca = (const char*)a;
    const char* cb = (const char*)b;
    const uint64_t total = m + n;
    uint64_t sum = 0;
    for (uint64_t r = 0; r < workers; ++r) {
        uint64_t lo, hi, j0, k0, j1, k1;
        uint32_t it0 = 0, c0 = 0, it1 = 0, c1 = 0;
        oracle_partition_output(total, workers, r, &lo);
        oracle_partition_output(total, workers, r + 1, &hi);
        oracle_co_rank(kind, lo, a, m, b, n, &j0, &k0, &it0, &c0);
        if (!synced || r + 1 < workers) {
            oracle_co_rank(kind, hi, a, m, b, n, &j1, &k1, &it1, &c1);
        } else {
            j1 = m;
            k1 = n;
        }
        if (synced) c1 = 0; /* the next worker's begin co-rank: counted there */
        uint64_t kc = 0;
        switch (kind) {
        case ORACLE_I32:
            kc = merge_count_i32((const int32_t*)(ca + j0 * s), j1 - j0,
                                 (const int32_t*)(cb + k0 * s), k1 - k0);
            break;
        case ORACLE_U32:
            kc = merge_count_u32((const uint32_t*)(ca + j0 * s), j1 - j0,
                                 (const uint32_t*)(cb + k0 * s), k1 - k0);
            break;
        default:
            kc = merge_count_u64((const uint64_t*)(ca + j0 * s), j1 - j0,
                                 (const uint64_t*)(cb + k0 * s), k1 - k0);
            break;
        }
        sum += (uint64_t)c0 + c1 + kc;
        if (block_sizes) block_sizes[r] = hi - lo;
        if (iterations) {
            if (synced) {
                iterations[r] = it0;
            } else {
                iterations[2 * r] = it0;
                iterations[2 * r + 1] = it1;
            }
        }
    }
    if (comparisons) *comparisons = sum;
    return ORACLE_OK;
}

/* ------------------------------------------- merge sort (test oracle only) */

int oracle_merge_sort(int kind, const void* in, uint64_t n, void* out) {
    const size_t s = key_size(kind);
    char* x = (char*)malloc(n ? n * s : 1);
    char* y = (char*)malloc(n ? n * s : 1);
    if (!x || !y) {
        free(x);
        free(y);
        return -1;
    }
    memcpy(x, in, n * s);
    for (uint64_t w = 1; w < n; w *= 2) {  /* merge runs 2q and 2q+1 of length w */
        for (uint64_t lo = 0; lo < n; lo += 2 * w) {
            const uint64_t mid = lo + w < n ? lo + w : n;
            const uint64_t hi = lo + 2 * w < n ? lo + 2 * w : n;
            oracle_merge_into(kind, x + lo * s, NULL, mid - lo, x + mid * s, NULL, hi - mid,
                              y + lo * s, NULL);
        }
        char* t = x;
        x = y;
        y = t;
    }
    memcpy(out, x, n * s);
    free(x);
    free(y);
    return 0;
}

int oracle_merge_sort_pairs(int kind, const void* in, const uint32_t* in_v, uint64_t n,
                            void* out, uint32_t* out_v) {
    const size_t s = key_size(kind);
    char* x = (char*)malloc(n ? n * s : 1);
    char* y = (char*)malloc(n ? n * s : 1);
    uint32_t* xv = (uint32_t*)malloc(n ? n * 4 : 1);
    uint32_t* yv = (uint32_t*)malloc(n ? n * 4 : 1);
    if (!x || !y || !xv || !yv) {
        free(x);
        free(y);
        free(xv);
        free(yv);
        return -1;
    }
    memcpy(x, in, n * s);
    memcpy(xv, in_v, n * 4);
    for (uint64_t w = 1; w < n; w *= 2) {
        for (uint64_t lo = 0; lo < n; lo += 2 * w) {
            const uint64_t mid = lo + w < n ? lo + w : n;
            const uint64_t hi = lo + 2 * w < n ? lo + 2 * w : n;
            oracle_merge_into(kind, x + lo * s, xv + lo, mid - lo, x + mid * s, xv + mid, hi - mid,
                              y + lo * s, yv + lo);
        }
        char* t = x;
        x = y;
        y = t;
        uint32_t* tv = xv;
        xv = yv;
        yv = tv;
    }
    memcpy(out, x, n * s);
    memcpy(out_v, xv, n * 4);
    free(x);
    free(y);
    free(xv);
    free(yv);
    return 0;
}

/* ---------------------------------------------- Algorithm 2 (parallel.hpp) */

typedef struct {
    int kind;
    const char* a;
    const uint32_t* av;
    uint64_t m;
    const char* b;
    const uint32_t* bv;
    uint64_t n;
    char* out;
    uint32_t* outv;
    uint64_t workers;
    uint64_t* block_sizes;
    uint32_t* iters;
    uint64_t first, step; /* worker ids first, first+step, ... */
} par_job;

/* both_ends_worker, parallel.hpp:201-207 */
static void run_worker(const par_job* J, uint64_t r) {
    const size_t s = key_size(J->kind);
    const uint64_t total = J->m + J->n;
    uint64_t lo, hi, j0, k0, j1, k1;
    uint32_t it0, it1;
    oracle_partition_output(total, J->workers, r, &lo);
    oracle_partition_output(total, J->workers, r + 1, &hi);
    oracle_co_rank(J->kind, lo, J->a, J->m, J->b, J->n, &j0, &k0, &it0, NULL);
    oracle_co_rank(J->kind, hi, J->a, J->m, J->b, J->n, &j1, &k1, &it1, NULL);
    oracle_merge_into(J->kind, J->a + j0 * s, J->av ? J->av + j0 : NULL, j1 - j0, J->b + k0 * s,
                      J->bv ? J->bv + k0 : NULL, k1 - k0, J->out + lo * s,
                      J->outv ? J->outv + lo : NULL);
    if (J->block_sizes) J->block_sizes[r] = hi - lo;
    if (J->iters) {
        J->iters[2 * r] = it0;
        J->iters[2 * r + 1] = it1;
    }
}

static void* par_thread(void* arg) {
    const par_job* J = (const par_job*)arg;
    for (uint64_t r = J->first; r < J->workers; r += J->step) run_worker(J, r);
    return NULL;
}

int oracle_merge_parallel(int kind, const void* a, const uint32_t* av, uint64_t m,
                          const void* b, const uint32_t* bv, uint64_t n, void* out,
                          uint32_t* outv, uint64_t workers, int threads,
                          uint64_t* block_sizes, uint32_t* corank_iterations) {
    if (check_total_length(m, n)) return ORACLE_E_LENGTH;
    if (workers == 0) return ORACLE_E_INVALID; /* parallel.hpp:185-186 */
    par_job base = {kind,  (const char*)a, av,          m,    (const char*)b,    bv, n,
                    (char*)out, outv,       workers, block_sizes, corank_iterations, 0, 1};
    if (threads <= 1) {
        par_thread(&base);
        return ORACLE_OK;
    }
    pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    par_job* jobs = (par_job*)malloc(sizeof(par_job) * (size_t)threads);
    for (int t = 0; t < threads; ++t) {
        jobs[t] = base;
        jobs[t].first = (uint64_t)t;
        jobs[t].step = (uint64_t)threads;
        pthread_create(&tids[t], NULL, par_thread, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    free(tids);
    free(jobs);
    return ORACLE_OK;
}

/* ------------------------------------------------------- segmented batch */

typedef struct {
    int kind;
    const char* a;
    const uint64_t* a_off;
    const char* b;
    const uint64_t* b_off;
    uint64_t nseg;
    char* out;
    uint64_t first, step;
} seg_job;

static void* seg_thread(void* arg) {
    const seg_job* J = (const seg_job*)arg;
    const size_t s = key_size(J->kind);
    for (uint64_t p = J->first; p < J->nseg; p += J->step) {
        const uint64_t ma = J->a_off[p + 1] - J->a_off[p];
        const uint64_t nb = J->b_off[p + 1] - J->b_off[p];
        const uint64_t o = J->a_off[p] + J->b_off[p];
        oracle_merge_into(J->kind, J->a + J->a_off[p] * s, NULL, ma, J->b + J->b_off[p] * s,
                          NULL, nb, J->out + o * s, NULL);
    }
    return NULL;
}

int oracle_merge_segmented(int kind, const void* a, const uint64_t* a_off, const void* b,
                           const uint64_t* b_off, uint64_t nseg, void* out, int threads) {
    for (uint64_t p = 0; p < nseg; ++p)
        if (a_off[p + 1] < a_off[p] || b_off[p + 1] < b_off[p]) return ORACLE_E_INVALID;
    seg_job base = {kind, (const char*)a, a_off, (const char*)b, b_off, nseg, (char*)out, 0, 1};
    if (threads <= 1) {
        seg_thread(&base);
        return ORACLE_OK;
    }
    pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    seg_job* jobs = (seg_job*)malloc(sizeof(seg_job) * (size_t)threads);
    for (int t = 0; t < threads; ++t) {
        jobs[t] = base;
        jobs[t].first = (uint64_t)t;
        jobs[t].step = (uint64_t)threads;
        pthread_create(&tids[t], NULL, seg_thread, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    free(tids);
    free(jobs);
    return ORACLE_OK;
}
