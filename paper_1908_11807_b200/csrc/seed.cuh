// seed.cuh -- exact search-radius seed of the kNN kernels.
#pragma once

#include "common.cuh"

namespace lbvh {

#ifndef LBVH_SEED_WINDOW
#define LBVH_SEED_WINDOW 2  // leaves per k in the Morton window
#endif

// Search-radius seed for one query: the kk-th smallest distance^2 among the
// 2*kk leaves that neighbour the query's Morton code in leaf order (a real
// upper bound of the true k-th distance).  Leaves are found by a lower_bound
// over the build's sorted leaf codes.
template <int K>
__device__ __forceinline__ float seed_bound(const lbvh_tree &t, uint32_t qcode, int kk,
                                            float px, float py, float pz) {
    const int64_t n = t.n;
    const uint32_t *__restrict__ codes = t.leaf_codes;
    int64_t lo = 0, hi = n;
    if (t.leaf_dir) {
        // lower_bound(qcode) lies in the bucket of its top leaf_dir_bits
        const uint32_t p = qcode >> (30 - t.leaf_dir_bits);
        lo = __ldg(t.leaf_dir + p);
        hi = __ldg(t.leaf_dir + p + 1);
    }
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(codes + mid) < qcode)
            lo = mid + 1;
        else
            hi = mid;
    }
    const int64_t w = LBVH_SEED_WINDOW * (int64_t)kk;
    int64_t w0 = lo - w / 2;
    w0 = w0 < 0 ? 0 : w0;
    w0 = (w0 + w > n) ? (n - w > 0 ? n - w : 0) : w0;
    const int64_t w1 = (w0 + w < n) ? w0 + w : n;
    float best[K];
#pragma unroll
    for (int j = 0; j < K; ++j) best[j] = (j < K - kk) ? -INFINITY : INFINITY;
    const float *__restrict__ mn = t.node_mins + 3 * (n - 1);
    // point leaves: maxs == mins (a deferred build leaves node_maxs leaf rows
    // unwritten), three loads per leaf, and the box distance of a point box is
    // bit for bit the sum of squared differences (the gap is |v - x| either
    // way round, rounded the same)
    const bool points = (t.flags & LBVH_TREE_POINT_LEAVES) != 0;
    const float *__restrict__ mx = points ? mn : t.node_maxs + 3 * (n - 1);
    for (int64_t p = w0; p < w1; ++p) {
        float d;
        if (points) {
            const float dx = __fsub_rn(px, __ldg(mn + 3 * p));
            const float dy = __fsub_rn(py, __ldg(mn + 3 * p + 1));
            const float dz = __fsub_rn(pz, __ldg(mn + 3 * p + 2));
            d = __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
        } else {
            d = box_dist_sq(px, py, pz, __ldg(mn + 3 * p), __ldg(mn + 3 * p + 1),
                            __ldg(mn + 3 * p + 2), __ldg(mx + 3 * p), __ldg(mx + 3 * p + 1),
                            __ldg(mx + 3 * p + 2));
        }
        if (d < best[K - 1]) {
            bool lt[K];
#pragma unroll
            for (int j = 0; j < K; ++j) lt[j] = best[j] <= d;
#pragma unroll
            for (int j = K - 1; j > 0; --j) best[j] = lt[j] ? best[j] : (lt[j - 1] ? d : best[j - 1]);
            best[0] = lt[0] ? best[0] : d;
        }
    }
    return best[K - 1];
}

}  // namespace lbvh
