// shard.cu -- device helpers of the sharded multi-GPU search (SURVEY.md §8e,
// paper_1908_11807_b200/distributed.py).  The reference has no distributed
// path; these kernels replace the tensor-op glue around the NCCL exchanges:
//
//   rank_forward_mask_kernel  which other ranks a query must visit: rank r is
//                             needed iff its box distance^2 <= the home's k-th
//                             distance^2 (kNN) or r*r (radius); same fp32
//                             recipe as the traversal (_kernels.py:146-176)
//   knn_finalize_kernel       home lists -> return arrays (sqrt(d^2), global
//                             ordinal), merged rows from sorted (d^2 bits << 32
//                             | global ordinal) keys (paths without lbvh_knn_kth)
//   scatter_rows_kernel       received rows -> (nq, kk) outputs in query order
//   remap_leaves_kernel       local tree leaves -> global ordinals
//   forward_*_kernel          radius: (query, rank) pairs of the forward mask ->
//                             per-destination rows (x, y, z, r, query id)
//   record_*_kernel           radius merge at the origin: per-query totals from
//                             the returned per-row hit counts, then each
//                             source's hits appended in rank order

#include "common.cuh"
#include "internal.cuh"

namespace lbvh {
namespace {

__global__ void __launch_bounds__(256)
rank_forward_mask_kernel(const float *__restrict__ centers, const float *__restrict__ bound,
                         float radius2, int64_t m, const float *__restrict__ boxes, int world,
                         uint32_t candidates, uint32_t *__restrict__ mask) {
    __shared__ float s_box[32 * 6];
    for (int i = threadIdx.x; i < world * 6; i += blockDim.x) s_box[i] = boxes[i];
    __syncthreads();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m;
         q += (int64_t)gridDim.x * blockDim.x) {
        const float px = __ldg(centers + 3 * q), py = __ldg(centers + 3 * q + 1),
                    pz = __ldg(centers + 3 * q + 2);
        const float b = bound ? __ldg(bound + q) : radius2;
        uint32_t bits = 0;
        for (int r = 0; r < world; ++r) {
            if (!((candidates >> r) & 1u)) continue;
            const float *bx = s_box + 6 * r;
            const float d = box_dist_sq(px, py, pz, bx[0], bx[1], bx[2], bx[3], bx[4], bx[5]);
            if (d <= b) bits |= 1u << r;
        }
        mask[q] = bits;
    }
}

// Home kNN lists -> the two return arrays (sqrt(d^2) f32, global ordinal i32),
// m x kk each, rows in arrival order; a row with remote candidates takes its
// merged keys instead.  Element-wise, fully coalesced.
__global__ void __launch_bounds__(256)
knn_finalize_kernel(int64_t m, int kk, const int32_t *__restrict__ local_idx,
                    const float *__restrict__ d2, const int64_t *__restrict__ gids,
                    const int64_t *__restrict__ merged_pos, const uint64_t *__restrict__ merged,
                    float *__restrict__ out_dist, int32_t *__restrict__ out_gid) {
    const int64_t total = m * kk;
    const bool narrow = total < (1ll << 32);  // 32-bit row/column split
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = narrow ? (int64_t)((uint32_t)e / (uint32_t)kk) : e / kk;
        const int64_t mp = merged_pos ? __ldg(merged_pos + q) : -1;
        float dd;
        int32_t g;
        if (mp >= 0) {
            const uint64_t key = __ldg(merged + mp * kk + (e - q * kk));
            dd = __uint_as_float((uint32_t)(key >> 32));
            g = (int32_t)(uint32_t)key;
        } else {
            dd = __ldg(d2 + e);
            const int32_t li = __ldg(local_idx + e);
            g = gids ? (int32_t)__ldg(gids + li) : li;
        }
        out_dist[e] = __fsqrt_rn(dd);
        out_gid[e] = g;
    }
}

// Received result rows of one source -> final (nq, kk) outputs:
// row i lands at query dst[i] (the origin's partition permutation slice).
__global__ void __launch_bounds__(256)
scatter_rows_kernel(int64_t m, int kk, const int64_t *__restrict__ dst,
                    const float *__restrict__ rd, const int32_t *__restrict__ rg,
                    float *__restrict__ out_d, int32_t *__restrict__ out_g) {
    const int64_t total = m * kk;
    const bool narrow = total < (1ll << 32);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = narrow ? (int64_t)((uint32_t)e / (uint32_t)kk) : e / kk;
        const int64_t q = __ldg(dst + i);
        const int64_t o = q * kk + (e - i * kk);
        out_d[o] = __ldg(rd + e);
        out_g[o] = __ldg(rg + e);
    }
}

// dst[i] = src[idx[i]] for 3-float rows (queries gathered into send order).
__global__ void __launch_bounds__(256)
gather_rows3_kernel(const float *__restrict__ src, const int64_t *__restrict__ idx, int64_t n,
                    float *__restrict__ dst) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = __ldg(idx + i);
        const float x = __ldg(src + 3 * j), y = __ldg(src + 3 * j + 1), z = __ldg(src + 3 * j + 2);
        dst[3 * i] = x;
        dst[3 * i + 1] = y;
        dst[3 * i + 2] = z;
    }
}

// Leaf ordinals of a local tree -> global ordinals (map[local] = global), in
// leaf_obj and in the packed nodes' leaf links.
__global__ void __launch_bounds__(256)
remap_leaves_kernel(int64_t n, int32_t *__restrict__ leaf_obj, PackedNode *__restrict__ nodes,
                    const int64_t *__restrict__ map) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        leaf_obj[i] = (int32_t)__ldg(map + leaf_obj[i]);
        if (i < n - 1) {
            int4 d = nodes[i].d;
            if (d.x < 0) d.x = (int32_t)((uint32_t)__ldg(map + (d.x & 0x7FFFFFFF)) | kLeafTag);
            if (d.y < 0) d.y = (int32_t)((uint32_t)__ldg(map + (d.y & 0x7FFFFFFF)) | kLeafTag);
            nodes[i].d = d;
        }
    }
}


// Radius forwarding (origin): rank d's rows go to its region of `rows`
// (region starts `start`, cursors zeroed), one 5-word row (x, y, z, r,
// query id as bits) per (query, rank) pair of the forward mask.  Positions
// inside a region follow the atomics; the merge below does not depend on them.
__global__ void __launch_bounds__(256)
forward_count_kernel(const uint32_t *__restrict__ mask, int64_t m, int world,
                     uint32_t *__restrict__ per_rank) {
    __shared__ uint32_t s_cnt[32];
    if (threadIdx.x < 32) s_cnt[threadIdx.x] = 0;
    __syncthreads();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m;
         q += (int64_t)gridDim.x * blockDim.x) {
        uint32_t b = __ldg(mask + q);
        while (b) {
            const int r = __ffs(b) - 1;
            b &= b - 1;
            atomicAdd(&s_cnt[r], 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x < world && s_cnt[threadIdx.x])
        atomicAdd(per_rank + threadIdx.x, s_cnt[threadIdx.x]);
}

__global__ void __launch_bounds__(256)
forward_rows_kernel(const float *__restrict__ centers, const float *__restrict__ radii,
                    const uint32_t *__restrict__ mask, int64_t m,
                    const int64_t *__restrict__ start, uint32_t *__restrict__ cursor,
                    float *__restrict__ rows) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < m;
         q += (int64_t)gridDim.x * blockDim.x) {
        uint32_t b = __ldg(mask + q);
        if (!b) continue;
        const float x = __ldg(centers + 3 * q), y = __ldg(centers + 3 * q + 1),
                    z = __ldg(centers + 3 * q + 2), r = __ldg(radii + q);
        while (b) {
            const int d = __ffs(b) - 1;
            b &= b - 1;
            float *row = rows + 5 * (__ldg(start + d) + atomicAdd(cursor + d, 1u));
            row[0] = x;
            row[1] = y;
            row[2] = z;
            row[3] = r;
            row[4] = __int_as_float((int32_t)q);
        }
    }
}

// Origin merge, step 1: each returned record (one per row this rank sent,
// in its send order) adds its hit count to its query's total.
__global__ void __launch_bounds__(256)
record_totals_kernel(const float *__restrict__ sent_rows, const int32_t *__restrict__ rec_counts,
                     int64_t n_rec, int32_t *__restrict__ totals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_rec;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = __ldg(rec_counts + i);
        if (c) atomicAdd(totals + __float_as_int(__ldg(sent_rows + 5 * i + 4)), c);
    }
}

// Origin merge, step 2 (one launch per source rank, in rank order): a query
// appears at most once per source, so its records need no atomics -- each
// appends its hits (the responder's fill order) after the earlier sources'.
__global__ void __launch_bounds__(256)
record_place_kernel(const float *__restrict__ sent_rows, const int32_t *__restrict__ rec_counts,
                    const int64_t *__restrict__ rec_off, int64_t r0, int64_t r1,
                    const int32_t *__restrict__ hits, const int64_t *__restrict__ offsets,
                    int32_t *__restrict__ cursor, int64_t *__restrict__ out) {
    for (int64_t i = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < r1;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = __ldg(rec_counts + i);
        if (!c) continue;
        const int32_t q = __float_as_int(__ldg(sent_rows + 5 * i + 4));
        const int64_t dst = __ldg(offsets + q) + cursor[q];
        const int64_t src = __ldg(rec_off + i);
        for (int32_t j = 0; j < c; ++j) out[dst + j] = __ldg(hits + src + j);
        cursor[q] += c;
    }
}

unsigned grid_of(int64_t n) {
    unsigned g = div_up(n > 0 ? n : 1, 256);
    return g < kNumSMs * 8 ? g : kNumSMs * 8;
}

}  // namespace
}  // namespace lbvh

using namespace lbvh;

extern "C" {

int lbvh_rank_forward_mask(const float *centers, const float *bound, float radius2, int64_t m,
                           const float *boxes, int world, uint32_t candidates, uint32_t *mask,
                           void *stream) {
    if (m < 0 || world < 1 || world > 32 || !boxes || (m > 0 && (!centers || !mask)))
        return LBVH_ERR_INVALID_ARG;
    if (m == 0) return LBVH_OK;
    rank_forward_mask_kernel<<<grid_of(m), 256, 0, (cudaStream_t)stream>>>(
        centers, bound, radius2, m, boxes, world, candidates, mask);
    count_launches(1);
    return check_launch();
}

int lbvh_knn_finalize(int64_t m, int kk, const int32_t *local_idx, const float *d2,
                      const int64_t *gids, const int64_t *merged_pos, const uint64_t *merged,
                      float *out_dist, int32_t *out_gid, void *stream) {
    if (m < 0 || kk < 1 || (m > 0 && (!local_idx || !d2 || !out_dist || !out_gid)) ||
        (merged_pos && !merged))
        return LBVH_ERR_INVALID_ARG;
    if (m == 0) return LBVH_OK;
    unsigned g = div_up(m * kk, 256);
    g = g < kNumSMs * 16 ? g : kNumSMs * 16;
    knn_finalize_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(m, kk, local_idx, d2, gids,
                                                            merged_pos, merged, out_dist,
                                                            out_gid);
    count_launches(1);
    return check_launch();
}

int lbvh_scatter_result_rows(int64_t m, int kk, const int64_t *dst, const float *rd,
                             const int32_t *rg, float *out_d, int32_t *out_g, void *stream) {
    if (m < 0 || kk < 1 || (m > 0 && (!dst || !rd || !rg || !out_d || !out_g)))
        return LBVH_ERR_INVALID_ARG;
    if (m == 0) return LBVH_OK;
    unsigned g = div_up(m * kk, 256);
    g = g < kNumSMs * 16 ? g : kNumSMs * 16;
    scatter_rows_kernel<<<g, 256, 0, (cudaStream_t)stream>>>(m, kk, dst, rd, rg, out_d, out_g);
    count_launches(1);
    return check_launch();
}

int lbvh_gather_rows3(const float *src, const int64_t *idx, int64_t n, float *dst,
                      void *stream) {
    if (n < 0 || (n > 0 && (!src || !idx || !dst))) return LBVH_ERR_INVALID_ARG;
    if (n == 0) return LBVH_OK;
    gather_rows3_kernel<<<grid_of(n), 256, 0, (cudaStream_t)stream>>>(src, idx, n, dst);
    count_launches(1);
    return check_launch();
}

int lbvh_forward_rows(const float *centers, const float *radii, const uint32_t *mask, int64_t m,
                      int world, uint32_t *per_rank, int64_t *start, uint32_t *cursor,
                      float *rows, int phase, void *stream) {
    if (m < 0 || world < 1 || world > 32 || !mask || (m > 0 && (!centers || !radii)))
        return LBVH_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (phase == 0) {  // per-rank pair counts
        if (!per_rank) return LBVH_ERR_INVALID_ARG;
        cudaMemsetAsync(per_rank, 0, sizeof(uint32_t) * world, st);
        if (m) {
            forward_count_kernel<<<grid_of(m), 256, 0, st>>>(mask, m, world, per_rank);
            count_launches(1);
        }
        return check_launch();
    }
    if (!start || !cursor || !rows) return LBVH_ERR_INVALID_ARG;
    cudaMemsetAsync(cursor, 0, sizeof(uint32_t) * world, st);
    if (m) {
        forward_rows_kernel<<<grid_of(m), 256, 0, st>>>(centers, radii, mask, m, start, cursor,
                                                       rows);
        count_launches(1);
    }
    return check_launch();
}

int lbvh_merge_records(const float *sent_rows, const int32_t *rec_counts, const int64_t *rec_off,
                       int64_t n_rec, const int64_t *source_starts, int world,
                       const int32_t *hits, const int64_t *offsets, int32_t *totals_or_cursor,
                       int64_t *out, int phase, void *stream) {
    if (n_rec < 0 || world < 1 || (n_rec > 0 && (!sent_rows || !rec_counts)) || !totals_or_cursor)
        return LBVH_ERR_INVALID_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    if (n_rec == 0) return LBVH_OK;
    if (phase == 0) {  // per-query totals (caller zeroes totals)
        record_totals_kernel<<<grid_of(n_rec), 256, 0, st>>>(sent_rows, rec_counts, n_rec,
                                                            totals_or_cursor);
        count_launches(1);
        return check_launch();
    }
    if (!rec_off || !source_starts || !hits || !offsets || !out) return LBVH_ERR_INVALID_ARG;
    for (int s = 0; s < world; ++s) {  // source order = merge order
        const int64_t r0 = source_starts[s], r1 = source_starts[s + 1];
        if (r1 <= r0) continue;
        record_place_kernel<<<grid_of(r1 - r0), 256, 0, st>>>(
            sent_rows, rec_counts, rec_off, r0, r1, hits, offsets, totals_or_cursor, out);
        count_launches(1);
    }
    return check_launch();
}

int lbvh_remap_leaves(const lbvh_tree *tree, int32_t *leaf_obj, void *nodes, const int64_t *map,
                      void *stream) {
    if (!tree || tree->n < 1 || !leaf_obj || !map || (tree->n > 1 && !nodes))
        return LBVH_ERR_INVALID_ARG;
    remap_leaves_kernel<<<grid_of(tree->n), 256, 0, (cudaStream_t)stream>>>(
        tree->n, leaf_obj, (PackedNode *)nodes, map);
    count_launches(1);
    return check_launch();
}

}  // extern "C"
