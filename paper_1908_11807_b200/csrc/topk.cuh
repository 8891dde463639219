// topk.cuh -- register-resident k-best list shared by the kNN kernels.
#pragma once

#include "common.cuh"

namespace lbvh {

// Lexicographic (dist^2, ordinal) order, _kernels.py:293-296.
__device__ __forceinline__ bool lex_less(float d1, int32_t i1, float d2, int32_t i2) {
    return d1 < d2 || (d1 == d2 && i1 < i2);
}

// The k best candidates as 64-bit keys (dist^2 bits << 32 | ordinal + 1),
// kept sorted ascending in registers.  Distances are >= +0 (or +inf), so the
// key order is exactly the reference's lexicographic (dist^2, ordinal) order
// (_kernels.py:293-296).  Slots [0, K-kk) hold 0-keys that rank before every
// real candidate; slots [K-kk, K) start empty (all ones: dist bits are NaN, so
// no distance compares greater and nothing is pruned until kk candidates
// are in, matching "size == kk and nd > worst", _kernels.py:367,383).  The
// k-th best is always slot K-1, a compile-time index, so nothing spills.
template <int K>
struct TopK {
    uint64_t key[K];
#ifdef LBVH_KNN_COUNT_VISITS
    int kept = 0;  // instrumentation: insertions that displaced the k-th
#endif

    // `bound` (optional, may be NaN = none): a distance^2 known to have at
    // least kk candidates at or below it.  Empty slots then carry
    // (bound, 0xFFFFFFFF) -- a virtual candidate every real one at the same
    // distance beats -- so nodes farther than the bound are pruned from the
    // start and leaves beyond it are never offered.  All virtual slots are
    // displaced by real candidates by the end, so results are unchanged.
    __device__ __forceinline__ void init(int kk, float bound) {
        const uint64_t empty = isnan(bound)
                                   ? ~0ull
                                   : (((uint64_t)__float_as_uint(bound) << 32) | 0xFFFFFFFFull);
#pragma unroll
        for (int j = 0; j < K; ++j) key[j] = (j < K - kk) ? 0ull : empty;
    }
    __device__ __forceinline__ float worst() const {
        return __uint_as_float((uint32_t)(key[K - 1] >> 32));
    }
    __device__ __forceinline__ static uint64_t make(float d, int32_t obj) {
        return ((uint64_t)__float_as_uint(d) << 32) | (uint32_t)(obj + 1);
    }

    // Keep the candidate iff it beats the current k-th best
    // (_kernels.py:387-395); branch-free sorted insertion dropping slot K-1.
    __device__ __forceinline__ void offer(float cd, int32_t obj) { offer_key(make(cd, obj)); }
    __device__ __forceinline__ void offer_key(const uint64_t c) {
        if (!(c < key[K - 1])) return;
#ifdef LBVH_KNN_COUNT_VISITS
        ++kept;
#endif
        bool lt[K];
#pragma unroll
        for (int j = 0; j < K; ++j) lt[j] = key[j] < c;
#pragma unroll
        for (int j = K - 1; j > 0; --j) key[j] = lt[j] ? key[j] : (lt[j - 1] ? c : key[j - 1]);
        key[0] = lt[0] ? key[0] : c;
    }
    __device__ __forceinline__ float dist(int j) const {
        return __uint_as_float((uint32_t)(key[j] >> 32));
    }
    __device__ __forceinline__ int32_t ordinal(int j) const {
        return (int32_t)((uint32_t)key[j]) - 1;
    }
};


// The same list held as separate 32-bit fields (distance bits, ordinal + 1),
// for the kNN traversal: the shifts move 32-bit words (the 64-bit key costs
// ptxas a >= and a > pair plus two SELs per slot), and the distance shift
// needs no select.  Same order, same results as TopK.
template <int K>
struct TopKSplit {
    uint32_t d[K], o[K];
#ifdef LBVH_KNN_COUNT_VISITS
    int kept = 0;
#endif
    __device__ __forceinline__ void init(int kk, float bound) {
        const bool none = isnan(bound);
        const uint32_t ed = none ? 0xFFFFFFFFu : __float_as_uint(bound);
#pragma unroll
        for (int j = 0; j < K; ++j) {
            d[j] = (j < K - kk) ? 0u : ed;
            o[j] = (j < K - kk) ? 0u : 0xFFFFFFFFu;
        }
    }
    __device__ __forceinline__ float worst() const { return __uint_as_float(d[K - 1]); }
    __device__ __forceinline__ float dist(int j) const { return __uint_as_float(d[j]); }
    __device__ __forceinline__ int32_t ordinal(int j) const { return (int32_t)o[j] - 1; }

    __device__ __forceinline__ void offer(float cd, int32_t obj) {
        const uint32_t cdu = __float_as_uint(cd), cou = (uint32_t)(obj + 1);
        // keep iff (cd, obj) beats the k-th best (_kernels.py:387-395)
        if (!(cdu < d[K - 1] || (cdu == d[K - 1] && cou < o[K - 1]))) return;
#ifdef LBVH_KNN_COUNT_VISITS
        ++kept;
#endif
        // lexicographic (d, o) < (cd, obj+1): one 64-bit compare of the
        // register pair per slot (ISETP + ISETP.EX)
        bool lt[K];
        const uint64_t c = ((uint64_t)cdu << 32) | cou;
#pragma unroll
        for (int j = 0; j < K; ++j) lt[j] = (((uint64_t)d[j] << 32) | o[j]) < c;
        // a slot that moves takes the candidate or its predecessor; with lt
        // lexicographic, that distance is max(d[j-1], cd): one predicated
        // VIMNMX per slot, one predicated SEL for the ordinal
#pragma unroll
        for (int j = K - 1; j > 0; --j) {
            d[j] = lt[j] ? d[j] : max(d[j - 1], cdu);
            o[j] = lt[j] ? o[j] : (lt[j - 1] ? cou : o[j - 1]);
        }
        d[0] = lt[0] ? d[0] : cdu;
        o[0] = lt[0] ? o[0] : cou;
    }
};

}  // namespace lbvh
