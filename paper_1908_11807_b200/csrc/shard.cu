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
