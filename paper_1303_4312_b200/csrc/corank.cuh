// corank.cuh -- co-rank searches (Algorithm 1 of arXiv 1303.4312).
//
// Two formulations of the same unique split (Lemma 1):
//
//  * co_rank_alg1: the reference's two-sided halving search, step for step
//    (proj/include/comerge/corank.hpp:72-121), including its
//    iteration/comparison accounting.  Used where the reference's
//    co_rank_stats must be reproduced (batched co-rank API, merge report).
//
//  * co_rank_split: a one-sided binary search over the monotone predicate
//        P(j) = j > 0 && k < n && b[k] < a[j-1]      (k = i - j)
//    i.e. guard 1 of corank.hpp:93-94.  P(lo) is false at the analytic floor
//    lo = max(0, i-n) and P is monotone in j, and guard 2 at j is
//    equivalent to "j == hi or P(j+1)", so the unique Lemma-1 split is the
//    largest j in [lo, hi] with !P(j).  Every probe inside the loop has
//    0 < mid <= min(i, m) and k = i - mid < n, so no index guard is needed
//    and both loads are independent (they issue together).  Used by the
//    partition kernels and inside shared-memory tiles.
#pragma once

#include <cstdint>

namespace comerge_b200 {

#ifdef __CUDA_ARCH__
__device__ __forceinline__ int32_t ldg_key(const int32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint32_t ldg_key(const uint32_t* p) { return __ldg(p); }
__device__ __forceinline__ uint64_t ldg_key(const uint64_t* p) {
    return static_cast<uint64_t>(__ldg(reinterpret_cast<const unsigned long long*>(p)));
}
#endif

struct corank_stats {
    uint32_t iterations;
    uint32_t comparisons;
};

// corank.hpp:72-121, literally.  `rd` reads one key (global or host).
template <typename K, typename Read>
__host__ __device__ __forceinline__ uint64_t co_rank_alg1(uint64_t target, const K* a, uint64_t m,
                                                          const K* b, uint64_t n, Read rd,
                                                          corank_stats* st) {
    uint64_t take_a = target < m ? target : m;       // :83
    uint64_t take_b = target - take_a;               // :84
    uint64_t floor_a = target > n ? target - n : 0;  // :86
    uint64_t floor_b = target > m ? target - m : 0;  // :87
    uint32_t iterations = 0, comparisons = 0;
    for (;;) {
        if (take_a > 0 && take_b < n && (++comparisons, rd(b + take_b) < rd(a + take_a - 1))) {
            const uint64_t step = (take_a - floor_a + 1) / 2;  // :98 ceil halving
            floor_b = take_b;
            take_a -= step;
            take_b += step;
            ++iterations;
        } else if (take_b > 0 && take_a < m &&
                   (++comparisons, !(rd(b + take_b - 1) < rd(a + take_a)))) {
            const uint64_t step = (take_b - floor_b + 1) / 2;  // :108
            floor_a = take_a;
            take_a += step;
            take_b -= step;
            ++iterations;
        } else {
            break;  // :113-115 both guards hold
        }
    }
    (void)floor_b;
    if (st) {
        st->iterations = iterations;
        st->comparisons = comparisons;
    }
    return take_a;
}

// Key comparisons the reference's serial merge (merge.hpp:18-33) makes on the
// windows A[j0, j1), B[k0, k1): its loop compares once per output until one
// side is exhausted.  B runs out first iff B's last key < A's last key (ties
// go to A); the loop then also took every A key <= B_last, else every B key
// < A_last -- one binary search instead of a counted merge.
template <typename K, typename Read>
__host__ __device__ __forceinline__ uint64_t merge_comparisons(const K* a, uint64_t j0, uint64_t j1,
                                                               const K* b, uint64_t k0, uint64_t k1,
                                                               Read rd) {
    if (j1 == j0 || k1 == k0) return 0;
    const K al = rd(a + j1 - 1), bl = rd(b + k1 - 1);
    if (bl < al) {
        uint64_t lo = j0, hi = j1;  // first A key > B_last
        while (lo < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (bl < rd(a + mid))
                hi = mid;
            else
                lo = mid + 1;
        }
        return (k1 - k0) + (lo - j0);
    }
    uint64_t lo = k0, hi = k1;  // first B key >= A_last
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (rd(b + mid) < al)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (j1 - j0) + (lo - k0);
}

// Largest j in [max(0,i-n), min(i,m)] with !P(j): the Lemma-1 split.
template <typename K, typename Index, typename Read>
__host__ __device__ __forceinline__ Index co_rank_split(Index i, const K* a, Index m, const K* b,
                                                        Index n, Read rd) {
    Index lo = i > n ? i - n : 0;
    Index hi = i < m ? i : m;
    while (lo < hi) {
        const Index mid = lo + (hi - lo + 1) / 2;  // mid in (lo, hi]
        if (rd(b + (i - mid)) < rd(a + (mid - 1)))
            hi = mid - 1;
        else
            lo = mid;
    }
    return lo;
}

}  // namespace comerge_b200
