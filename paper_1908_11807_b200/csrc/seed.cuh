// seed.cuh -- exact search-radius seed of the kNN kernels: the kk-th smallest
// distance^2 among 2*kk real leaves near the query bounds its true k-th
// distance from above, so the traversal prunes from the first node on and
// results cannot change.  Two ways to pick the leaves: the 2x2x2 block of
// leaf-directory cells around the query (seed_bound_block, lists of K >= 8)
// and the Morton window around its code (seed_bound, the fallback).

#pragma once

#include "common.cuh"

namespace lbvh {

#ifndef LBVH_SEED_WINDOW
#define LBVH_SEED_WINDOW 2  // leaves per k in the Morton window
#endif
#ifndef LBVH_SEED_BLOCK_MIN_K
#define LBVH_SEED_BLOCK_MIN_K 2  // smallest k seeded from the 2x2x2 cell block
#endif
#ifndef LBVH_SEED_BLOCK_QUARTERS
#define LBVH_SEED_BLOCK_QUARTERS 8  // leaves scanned by the block seed: kk * QUARTERS / 4, nearest cells first
#endif

// Distance^2 of the query to the leaf at sorted position p (point leaves:
// the sum of squared differences, bit for bit the point-box distance).
__device__ __forceinline__ float seed_leaf_dist(const float *__restrict__ mn,
                                                const float *__restrict__ mx, bool points,
                                                int64_t p, float px, float py, float pz) {
    if (points) {
        const float dx = __fsub_rn(px, __ldg(mn + 3 * p));
        const float dy = __fsub_rn(py, __ldg(mn + 3 * p + 1));
        const float dz = __fsub_rn(pz, __ldg(mn + 3 * p + 2));
        return __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
    }
    return box_dist_sq(px, py, pz, __ldg(mn + 3 * p), __ldg(mn + 3 * p + 1),
                       __ldg(mn + 3 * p + 2), __ldg(mx + 3 * p), __ldg(mx + 3 * p + 1),
                       __ldg(mx + 3 * p + 2));
}

// Sorted list of the K smallest distances (slots j < K - kk hold -inf).
template <int K>
__device__ __forceinline__ void seed_insert(float (&best)[K], float d) {
    if (d < best[K - 1]) {
        bool lt[K];
#pragma unroll
        for (int j = 0; j < K; ++j) lt[j] = best[j] <= d;
#pragma unroll
        for (int j = K - 1; j > 0; --j) best[j] = lt[j] ? best[j] : (lt[j - 1] ? d : best[j - 1]);
        best[0] = lt[0] ? best[0] : d;
    }
}

// x, y or z cell coordinate (10 bits) of a 30-bit Morton code
__device__ __forceinline__ uint32_t compact_bits(uint32_t v) {
    v &= 0x09249249u;
    v = (v | (v >> 2)) & 0x030C30C3u;
    v = (v | (v >> 4)) & 0x0300F00Fu;
    v = (v | (v >> 8)) & 0x030000FFu;
    v = (v | (v >> 16)) & 0x000003FFu;
    return v;
}

// Block seed: when the leaf directory's buckets are cubic cells (bits = 3L),
// the leaves of the 2x2x2 block of level-L cells around the query (the block
// whose centre is the cell corner nearest to it) are eight contiguous runs of
// the sorted leaves.  The first 2*kk of them, the query's own cell first,
// then the cells sharing a face, an edge, the corner, give a bound like any
// kk real leaves do, and it covers the query's neighbourhood on all sides (a
// Morton window follows the curve and is one-sided across its jumps): at C2
// the bound is 1.13x the exact k-th distance on average against 1.55x for
// the 2k-leaf window, for the same number of distance tests.  Returns +inf
// when the block holds fewer than kk leaves (the caller falls back to the
// window).
template <int K>
__device__ __forceinline__ float seed_bound_block(const lbvh_tree &t, uint32_t qcode, int kk,
                                                  float px, float py, float pz) {
    const int L = t.leaf_dir_bits / 3;
    const int sh = 10 - L;  // bits of a level-L cell below its coordinate
    const uint32_t top = (1u << L) - 2;
    uint32_t base[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const uint32_t c = compact_bits(qcode >> (2 - a));  // x, y, z
        const uint32_t cell = c >> sh, upper = sh ? (c >> (sh - 1)) & 1u : 0u;
        uint32_t b = cell + upper;  // block = [b - 1, b]
        b = b < 1 ? 1 : (b > top + 1 ? top + 1 : b);
        base[a] = b - 1;
    }
    float best[K];
#pragma unroll
    for (int j = 0; j < K; ++j) best[j] = (j < K - kk) ? -INFINITY : INFINITY;
    const int64_t n = t.n;
    const float *__restrict__ mn = t.node_mins + 3 * (n - 1);
    const bool points = (t.flags & LBVH_TREE_POINT_LEAVES) != 0;
    const float *__restrict__ mx = points ? mn : t.node_maxs + 3 * (n - 1);
    // the eight cells nearest first: the query's own cell, the three that
    // share a face with it, the three that share an edge, the opposite corner
    // (all directory reads issued up front; the scan stops after `cap` leaves)
    uint32_t sa[3][2];  // spread coordinate of [own, other] cell per axis
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const uint32_t c = compact_bits(qcode >> (2 - a)) >> sh;
        const uint32_t own = c < base[a] ? base[a] : (c > base[a] + 1 ? base[a] + 1 : c);
        const uint32_t other = own == base[a] ? base[a] + 1 : base[a];
        sa[a][0] = spread_bits(own) << (2 - a);
        sa[a][1] = spread_bits(other) << (2 - a);
    }
    constexpr int kOff[8] = {0, 4, 2, 1, 6, 5, 3, 7};  // flip x / y / z bits
    uint32_t lo[8], hi[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int o = kOff[r];
        const uint32_t code = sa[0][(o >> 2) & 1] | sa[1][(o >> 1) & 1] | sa[2][o & 1];
        lo[r] = __ldg(t.leaf_dir + code);
        hi[r] = __ldg(t.leaf_dir + code + 1);
    }
    const int cap = (LBVH_SEED_BLOCK_QUARTERS * kk) >> 2;
    int scanned = 0, left = 7;
    uint32_t p = lo[0], e = hi[0];
    // one flat loop over the runs: the next run shifts into (p, e)
#pragma unroll 1
    while (scanned < cap) {
        if (p < e) {
            seed_insert<K>(best, seed_leaf_dist(mn, mx, points, p, px, py, pz));
            ++p;
            ++scanned;
        } else {
            if (left == 0) break;
            --left;
#pragma unroll
            for (int r = 0; r < 7; ++r) {
                lo[r] = lo[r + 1];
                hi[r] = hi[r + 1];
            }
            p = lo[0];
            e = hi[0];
        }
    }
    return scanned >= kk ? best[K - 1] : INFINITY;
}

// Search-radius seed for one query: the kk-th smallest distance^2 among the
// 2*kk leaves that neighbour the query's Morton code in leaf order (a real
// upper bound of the true k-th distance).  Leaves are found by a lower_bound
// over the build's sorted leaf codes.
template <int K>
__device__ __forceinline__ float seed_bound(const lbvh_tree &t, uint32_t qcode, int kk,
                                            float px, float py, float pz) {
    const int64_t n = t.n;
    // lists of <= 4 (k = 1: 2.28 ms window vs 2.39 block, the eight directory
    // reads and their registers cost more than the 2k leaves save)
    if (K >= 8 && kk >= LBVH_SEED_BLOCK_MIN_K && t.leaf_dir && t.leaf_dir_bits >= 3 &&
        t.leaf_dir_bits % 3 == 0) {
        const float b = seed_bound_block<K>(t, qcode, kk, px, py, pz);
        if (b != INFINITY) return b;
    }
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
    // unwritten), three loads per leaf
    const bool points = (t.flags & LBVH_TREE_POINT_LEAVES) != 0;
    const float *__restrict__ mx = points ? mn : t.node_maxs + 3 * (n - 1);
    for (int64_t p = w0; p < w1; ++p) seed_insert<K>(best, seed_leaf_dist(mn, mx, points, p, px, py, pz));
    return best[K - 1];
}

}  // namespace lbvh
