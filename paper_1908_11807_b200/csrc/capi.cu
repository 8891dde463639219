// capi.cu -- extern "C" entry points (include/lbvh_b200.h).

#include <stdio.h>
#include <string.h>

#include <atomic>

#include "common.cuh"
#include "internal.cuh"

namespace lbvh {

static thread_local char g_cuda_err[256] = "";
static std::atomic<uint64_t> g_launches{0};

void count_launches(int k) { g_launches.fetch_add((uint64_t)k, std::memory_order_relaxed); }
uint64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }

void set_cuda_error(cudaError_t e) {
    snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e),
             cudaGetErrorString(e));
}

int check_launch() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_cuda_error(e);
        return LBVH_ERR_CUDA;
    }
    return LBVH_OK;
}

// defined in build.cu / traverse.cu / scan.cu
size_t build_workspace_bytes(int64_t n);
int build(const float *, const float *, int64_t, int, void *, size_t, float *, float *,
          int32_t *, int32_t *, int32_t *, float *, void *, uint32_t *, uint32_t *, int, int,
          const int32_t *, uint32_t *, cudaStream_t);
int finish_rows(const lbvh_tree *, float *, float *, cudaStream_t);
size_t topology_workspace_bytes(int64_t n);
int generate_topology(const uint32_t *, int64_t, int32_t *, int32_t *, int32_t *, void *, size_t,
                      cudaStream_t);
int refit(float *, float *, const int32_t *, const int32_t *, const int32_t *, int64_t, void *,
          size_t, cudaStream_t);
int pack(const lbvh_tree *, void *, float *, uint32_t *, cudaStream_t);
int unpack_boxes(const lbvh_tree *, float *, float *, cudaStream_t);
int morton_codes_f64(const double *, int64_t, const double *, const double *, uint32_t *,
                     cudaStream_t);
size_t query_workspace_bytes(int64_t nq);
// status / offsets (optional): fused value check and uniform CRS offsets
int query_order(const float *, int64_t, const float *, int, uint32_t *, uint32_t *, void *,
                size_t, cudaStream_t, uint32_t *status = nullptr, int64_t *offsets = nullptr,
                int64_t span = 0);
int spatial_count(const lbvh_tree *, const float *, const float *, float, const uint32_t *,
                  int64_t, int32_t *, int32_t *, int64_t, uint32_t *, cudaStream_t,
                  int32_t *spill_heads = nullptr, int32_t *spill_pool = nullptr,
                  int64_t spill_chunks = 0, uint32_t *over_list = nullptr,
                  uint32_t *over_n = nullptr, uint32_t *spill_list = nullptr,
                  uint32_t *spill_n = nullptr);
int spill_copy(const int32_t *, int64_t, const int32_t *, const int64_t *, const int32_t *,
               const int32_t *, const uint32_t *, const uint32_t *, int64_t, int32_t *,
               cudaStream_t);
int spatial_list(const lbvh_tree *, const float *, const float *, float, const uint32_t *,
                 const uint32_t *, int64_t, int32_t *, const int64_t *, int32_t *, bool,
                 uint32_t *, cudaStream_t);

int spatial_fill(const lbvh_tree *, const float *, const float *, float, const uint32_t *,
                 int64_t, const int64_t *, int32_t *, const int32_t *, int64_t, uint32_t *,
                 cudaStream_t);
int spatial_1p(const lbvh_tree *, const float *, const float *, float, const uint32_t *, int64_t,
               int32_t *, int64_t, int32_t *, uint32_t *, cudaStream_t);
int compact(const int32_t *, int64_t, const int32_t *, const int64_t *, int64_t, int32_t *,
            cudaStream_t);
int knn_offsets(const int64_t *, int64_t, int64_t, int64_t, int64_t *, int32_t *, uint32_t *,
                void *, size_t, cudaStream_t);
int leaf_directory(const uint32_t *, int64_t, int, uint32_t *, cudaStream_t);
int morton_codes_f32(const float *, int64_t, const float *, uint32_t *, cudaStream_t);
int knn(const lbvh_tree *, const float *, const uint32_t *, const uint32_t *, int64_t,
        const int64_t *, int64_t, int32_t *, float *, int, void *, size_t, uint32_t *,
        cudaStream_t, float *);
size_t knn_workspace_bytes(int64_t nq);
int select_overflow(const uint32_t *, const int32_t *, int64_t, int64_t, uint32_t *, uint32_t *,
                    cudaStream_t, const int32_t *spill_heads = nullptr,
                    uint32_t *spill_list = nullptr, uint32_t *spill_count = nullptr);
int check_queries(const float *, int64_t, const float *, uint32_t *, cudaStream_t);
int unpack_knn_keys(const uint64_t *, int64_t, int64_t *, float *, cudaStream_t);
int brute_knn(const float *, int64_t, const float *, int64_t, int64_t, int32_t *, float *,
              cudaStream_t);
int brute_radius(const float *, int64_t, const float *, const float *, float, int64_t, int32_t *,
                 const int64_t *, int32_t *, cudaStream_t);

}  // namespace lbvh

using namespace lbvh;

#define S(x) ((cudaStream_t)(x))

extern "C" {

const char *lbvh_strerror(int code) {
    switch (code) {
    case LBVH_OK: return "ok";
    case LBVH_ERR_INVALID_ARG: return "invalid argument";
    case LBVH_ERR_WORKSPACE: return "workspace too small";
    case LBVH_ERR_CUDA: return "CUDA error";
    case LBVH_ERR_EMPTY_SCENE: return "empty scene";
    case LBVH_ERR_TOO_LARGE: return "too many items (limit 2^30 - 1)";
    default: return "unknown error";
    }
}

const char *lbvh_last_cuda_error(void) { return g_cuda_err; }

int lbvh_abi_version(void) { return 5; }

uint64_t lbvh_launch_count(void) { return launch_count(); }

size_t lbvh_build_workspace_bytes(int64_t n) { return build_workspace_bytes(n); }
size_t lbvh_sort_workspace_bytes(int64_t n) { return sort_workspace_bytes(n); }
size_t lbvh_topology_workspace_bytes(int64_t n) { return topology_workspace_bytes(n); }
size_t lbvh_query_workspace_bytes(int64_t nq) { return query_workspace_bytes(nq); }
size_t lbvh_scan_workspace_bytes(int64_t nq) { return scan_workspace_bytes(nq); }

int lbvh_build(const float *mins, const float *maxs, int64_t n, int morton_bits, void *ws,
               size_t ws_bytes, float *node_mins, float *node_maxs, int32_t *left,
               int32_t *right, int32_t *leaf_obj, float *root_box, void *nodes,
               uint32_t *sorted_codes, uint32_t *leaf_dir, int leaf_dir_bits, int flags,
               const int32_t *leaf_ids, uint32_t *status, void *stream) {
    return build(mins, maxs, n, morton_bits, ws, ws_bytes, node_mins, node_maxs, left, right,
                 leaf_obj, root_box, nodes, sorted_codes, leaf_dir, leaf_dir_bits, flags,
                 leaf_ids, status, S(stream));
}

int lbvh_finish_rows(const lbvh_tree *tree, float *node_mins, float *node_maxs, void *stream) {
    return finish_rows(tree, node_mins, node_maxs, S(stream));
}

int lbvh_morton_codes(const double *pts, int64_t n, const double *lo, const double *hi,
                      uint32_t *codes, void *stream) {
    return morton_codes_f64(pts, n, lo, hi, codes, S(stream));
}

int lbvh_morton_codes_f32(const float *points, int64_t n, const float *scene_box,
                          uint32_t *codes, void *stream) {
    return morton_codes_f32(points, n, scene_box, codes, S(stream));
}

int lbvh_sort_pairs(uint32_t *keys, uint32_t *values, int64_t n, int key_bits, void *ws,
                    size_t ws_bytes, void *stream) {
    if (n < 0 || (n > 0 && (!keys || !values))) return LBVH_ERR_INVALID_ARG;
    return sort_pairs(keys, values, n, key_bits, ws, ws_bytes, S(stream));
}

int lbvh_generate_topology(const uint32_t *codes, int64_t n, int32_t *left, int32_t *right,
                           int32_t *parent, void *ws, size_t ws_bytes, void *stream) {
    return generate_topology(codes, n, left, right, parent, ws, ws_bytes, S(stream));
}

int lbvh_refit(float *node_mins, float *node_maxs, const int32_t *left, const int32_t *right,
               const int32_t *parent, int64_t n, void *ws, size_t ws_bytes, void *stream) {
    return refit(node_mins, node_maxs, left, right, parent, n, ws, ws_bytes, S(stream));
}

int lbvh_pack(const lbvh_tree *tree, void *nodes, float *root_box, uint32_t *status,
              void *stream) {
    return pack(tree, nodes, root_box, status, S(stream));
}

int lbvh_unpack_boxes(const lbvh_tree *tree, float *node_mins, float *node_maxs,
                      void *stream) {
    return unpack_boxes(tree, node_mins, node_maxs, S(stream));
}

int lbvh_leaf_directory_bits(int64_t n) {
    // cubic cells (3L bits) of >= 2.5 leaves on average: the kNN block seed
    // scans the 2x2x2 cells around a query (about 20-50 leaves)
    int L = 0;
    while (L < 8 && 5 * ((int64_t)1 << (3 * (L + 1))) <= 2 * n) ++L;
    return 3 * L;
}

int lbvh_leaf_directory(const uint32_t *leaf_codes, int64_t n, int bits, uint32_t *dir,
                        void *stream) {
    return leaf_directory(leaf_codes, n, bits, dir, S(stream));
}

int lbvh_query_order(const float *centers, int64_t nq, const float *scene_box, int order_bits,
                     uint32_t *order, uint32_t *sorted_codes, void *ws, size_t ws_bytes,
                     void *stream) {
    return query_order(centers, nq, scene_box, order_bits, order, sorted_codes, ws, ws_bytes,
                       S(stream));
}

int lbvh_check_queries(const float *centers, int64_t nq, const float *radii, uint32_t *status,
                       void *stream) {
    return check_queries(centers, nq, radii, status, S(stream));
}

int lbvh_spatial_count(const lbvh_tree *tree, const float *centers, const float *radii,
                       float radius, const uint32_t *order, int64_t nq, int32_t *counts,
                       int32_t *buf, int64_t buffer_size, uint32_t *status, void *stream) {
    return spatial_count(tree, centers, radii, radius, order, nq, counts, buf, buffer_size,
                         status, S(stream));
}

int lbvh_spatial_fill(const lbvh_tree *tree, const float *centers, const float *radii,
                      float radius, const uint32_t *order, int64_t nq, const int64_t *offsets,
                      int32_t *out, const int32_t *skip_counts, int64_t buffer_size,
                      uint32_t *status, void *stream) {
    return spatial_fill(tree, centers, radii, radius, order, nq, offsets, out, skip_counts,
                        buffer_size, status, S(stream));
}

int lbvh_exclusive_scan(const int32_t *counts, int64_t nq, int64_t *offsets, void *ws,
                        size_t ws_bytes, void *stream) {
    return scan_counts(counts, nq, offsets, ws, ws_bytes, S(stream));
}

int lbvh_spatial_1p(const lbvh_tree *tree, const float *centers, const float *radii,
                    float radius, const uint32_t *order, int64_t nq, int32_t *buf,
                    int64_t buffer_size, int32_t *counts, uint32_t *status, void *stream) {
    return spatial_1p(tree, centers, radii, radius, order, nq, buf, buffer_size, counts, status,
                      S(stream));
}

int lbvh_compact(const int32_t *buf, int64_t buffer_size, const int32_t *counts,
                 const int64_t *offsets, int64_t nq, int32_t *out, void *stream) {
    return compact(buf, buffer_size, counts, offsets, nq, out, S(stream));
}

int lbvh_knn_offsets(const int64_t *ks, int64_t k, int64_t n, int64_t nq, int64_t *offsets,
                     int32_t *max_span, uint32_t *status, void *ws, size_t ws_bytes,
                     void *stream) {
    return knn_offsets(ks, k, n, nq, offsets, max_span, status, ws, ws_bytes, S(stream));
}

int lbvh_knn(const lbvh_tree *tree, const float *centers, const uint32_t *order,
             const uint32_t *query_codes, int64_t nq, const int64_t *offsets, int64_t max_span,
             int32_t *out_idx, float *out_dist, int flags, void *workspace,
             size_t workspace_bytes, uint32_t *status, void *stream) {
    return knn(tree, centers, order, query_codes, nq, offsets, max_span, out_idx, out_dist,
               flags, workspace, workspace_bytes, status, S(stream), nullptr);
}

/* One device kNN batch with a uniform k in a single call: value checks,
 * CRS offsets, Morton query order on the tree's grid and the search (the
 * drop-in query_knn for device-resident centers without per-call host
 * round trips between the launches). */
size_t lbvh_knn_batch_workspace_bytes(int64_t nq) {
    const size_t n = (size_t)(nq > 0 ? nq : 1);
    size_t a = align_up(4 * n) * 2;  // order + sorted query codes
    size_t q = query_workspace_bytes(nq), sc = scan_workspace_bytes(nq),
           kw = knn_workspace_bytes(nq);
    size_t m = q > sc ? q : sc;
    m = m > kw ? m : kw;
    return a + m + 1024;
}

int lbvh_knn_batch(const lbvh_tree *tree, const float *centers, int64_t nq, int64_t k,
                   int order_bits, int64_t *offsets, int32_t *out_idx, float *out_dist,
                   int flags, void *ws, size_t ws_bytes, uint32_t *status, float *kth_d2,
                   void *ev_before, void *ev_after, void *stream) {
    if (!tree || nq < 0 || k < 1 || !status) return LBVH_ERR_INVALID_ARG;
    if (nq == 0) return LBVH_OK;
    if (!centers || !offsets || !out_idx || !out_dist || !ws) return LBVH_ERR_INVALID_ARG;
    if (ws_bytes < lbvh_knn_batch_workspace_bytes(nq)) return LBVH_ERR_WORKSPACE;
    cudaStream_t st = S(stream);
    Carve c(ws, ws_bytes);
    uint32_t *order = c.take<uint32_t>(nq);
    uint32_t *codes = c.take<uint32_t>(nq);
    void *rest = c.take<char>(1);
    const size_t rest_bytes = ws_bytes - ((char *)rest - (char *)ws);
    const int64_t span = k < tree->n ? k : tree->n;
    const bool sorted = order_bits > 0 && nq > 1;
    int rc;
    if (sorted) {
        // one pass over the centers: value check, uniform offsets, Morton codes
        rc = query_order(centers, nq, tree->root_box, order_bits, order, codes, rest,
                         rest_bytes, st, status, offsets, span);
        if (rc) return rc;
    } else {
        rc = check_queries(centers, nq, nullptr, status, st);
        if (rc) return rc;
        rc = knn_offsets(nullptr, k, tree->n, nq, offsets, nullptr, status, rest, rest_bytes, st);
        if (rc) return rc;
    }
    if (ev_before) cudaEventRecord((cudaEvent_t)ev_before, st);
    rc = knn(tree, centers, sorted ? order : nullptr, sorted ? codes : nullptr, nq, offsets,
             span, out_idx, out_dist, flags | LBVH_KNN_UNIFORM_SPANS, rest, rest_bytes, status,
             st, kth_d2);
    if (ev_after) cudaEventRecord((cudaEvent_t)ev_after, st);
    return rc;
}

size_t lbvh_spatial_count_batch_workspace_bytes(int64_t nq) {
    size_t q = query_workspace_bytes(nq), sc = scan_workspace_bytes(nq);
    return (q > sc ? q : sc) + 1024;
}

int lbvh_spatial_count_batch(const lbvh_tree *tree, const float *centers, const float *radii,
                             float radius, int64_t nq, int order_bits, int64_t rows,
                             uint32_t *order, int32_t *counts, int32_t *buf, int64_t *offsets,
                             uint32_t *over_list, uint32_t *over_n, int32_t *spill_heads,
                             int32_t *spill_pool, int64_t spill_chunks, uint32_t *spill_list,
                             uint32_t *spill_n, void *ws, size_t ws_bytes, uint32_t *status,
                             void *ev_before, void *ev_after, void *stream) {
    if (!tree || nq < 0 || !status) return LBVH_ERR_INVALID_ARG;
    if (nq == 0) return LBVH_OK;
    if (!centers || !counts || !offsets || !order || !ws ||
        (rows > 0 && (!buf || !over_list || !over_n)))
        return LBVH_ERR_INVALID_ARG;
    const bool spill = rows > 0 && spill_pool && spill_chunks > 1;
    if (spill && (!spill_heads || !spill_list || !spill_n)) return LBVH_ERR_INVALID_ARG;
    if (ws_bytes < lbvh_spatial_count_batch_workspace_bytes(nq)) return LBVH_ERR_WORKSPACE;
    cudaStream_t st = S(stream);
    const bool sorted = order_bits > 0 && nq > 1;
    // scalar radius: the centers' value check rides on the query Morton pass
    const bool fused_check = sorted && !radii;
    int rc = LBVH_OK;
    if (!fused_check) {
        rc = check_queries(centers, nq, radii, status, st);
        if (rc) return rc;
    }
    if (sorted) {
        rc = query_order(centers, nq, tree->root_box, order_bits, order, nullptr, ws, ws_bytes,
                         st, fused_check ? status : nullptr);
        if (rc) return rc;
    }
    const uint32_t *ord = sorted ? order : nullptr;
    if (ev_before) cudaEventRecord((cudaEvent_t)ev_before, st);
    // the overflow (fill) and spill lists are appended as queries finish:
    // the fill pass and the spill copy take queries in any order
    rc = spatial_count(tree, centers, radii, radius, ord, nq, counts, rows > 0 ? buf : nullptr,
                       rows, status, st, spill ? spill_heads : nullptr,
                       spill ? spill_pool : nullptr, spill ? spill_chunks : 0,
                       rows > 0 ? over_list : nullptr, rows > 0 ? over_n : nullptr,
                       spill ? spill_list : nullptr, spill ? spill_n : nullptr);
    if (ev_after) cudaEventRecord((cudaEvent_t)ev_after, st);
    if (rc) return rc;
    return scan_counts(counts, nq, offsets, ws, ws_bytes, st);
}

int lbvh_knn_kth(const lbvh_tree *tree, const float *centers, const uint32_t *order,
                 const uint32_t *query_codes, int64_t nq, const int64_t *offsets,
                 int64_t max_span, int32_t *out_idx, float *out_dist, int flags,
                 void *workspace, size_t workspace_bytes, uint32_t *status, float *kth_d2,
                 void *stream) {
    if (!kth_d2) return LBVH_ERR_INVALID_ARG;
    return knn(tree, centers, order, query_codes, nq, offsets, max_span, out_idx, out_dist,
               flags, workspace, workspace_bytes, status, S(stream), kth_d2);
}

size_t lbvh_knn_workspace_bytes(int64_t nq) { return knn_workspace_bytes(nq); }

int lbvh_spatial_fill_list(const lbvh_tree *tree, const float *centers, const float *radii,
                           float radius, const uint32_t *list, const uint32_t *list_len,
                           int64_t n_list, const int64_t *offsets, int32_t *out,
                           uint32_t *status, void *stream) {
    if (!tree || n_list < 0 || !status) return LBVH_ERR_INVALID_ARG;
    if (n_list == 0) return LBVH_OK;
    if (list_len)
        return spatial_list(tree, centers, radii, radius, list, list_len, n_list, nullptr,
                            offsets, out, true, status, S(stream));
    return spatial_fill(tree, centers, radii, radius, list, n_list, offsets, out, nullptr, 0,
                        status, S(stream));
}

int lbvh_spill_copy(const int32_t *buf, int64_t rows, const int32_t *counts,
                    const int64_t *offsets, const int32_t *spill_heads, const int32_t *spill_pool,
                    const uint32_t *spill_list, const uint32_t *spill_n, int64_t max_list,
                    int32_t *out, void *stream) {
    return spill_copy(buf, rows, counts, offsets, spill_heads, spill_pool, spill_list, spill_n,
                      max_list, out, S(stream));
}

int lbvh_select_overflow(const uint32_t *order, const int32_t *counts, int64_t nq,
                         int64_t buffer_size, uint32_t *list, uint32_t *list_len, void *stream) {
    return select_overflow(order, counts, nq, buffer_size, list, list_len, S(stream));
}

int lbvh_unpack_knn_keys(const uint64_t *keys, int64_t n, int64_t *ordinals, float *dist,
                         void *stream) {
    return unpack_knn_keys(keys, n, ordinals, dist, S(stream));
}

int lbvh_brute_knn(const float *points, int64_t n, const float *centers, int64_t nq, int64_t k,
                   int32_t *out_idx, float *out_dist, void *stream) {
    return brute_knn(points, n, centers, nq, k, out_idx, out_dist, S(stream));
}

int lbvh_brute_radius(const float *points, int64_t n, const float *centers, const float *radii,
                      float radius, int64_t nq, int32_t *counts, const int64_t *offsets,
                      int32_t *out, void *stream) {
    return brute_radius(points, n, centers, radii, radius, nq, counts, offsets, out, S(stream));
}

}  // extern "C"
