/*
 * lbvh_b200.h -- C ABI of the B200-native LBVH hot path.
 *
 * Plain pointers and sizes only; no torch or CUDA types in the signatures.
 * All array arguments are DEVICE pointers unless marked "host".  `stream` is
 * a cudaStream_t passed as void*.  The library never allocates, frees or
 * throws: callers own every buffer, including the workspace whose size the
 * matching *_workspace_bytes() function reports.  Calls are stream-ordered
 * and asynchronous; per-element failures are reported through a device
 * status word (LBVH_FLAG_* bits, OR-ed by the kernels) that the caller reads
 * back, mirroring the reference's per-query err/overflow arrays
 * (pkg/src/lbvh/_kernels.py:3-5, traversal.py:168-170).
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to the reference checkout).
 */
#ifndef LBVH_B200_H
#define LBVH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes (host side). */
enum {
    LBVH_OK = 0,
    LBVH_ERR_INVALID_ARG = 1,  /* bad sizes / null pointers                */
    LBVH_ERR_WORKSPACE = 2,    /* workspace smaller than *_workspace_bytes */
    LBVH_ERR_CUDA = 3,         /* a CUDA launch or runtime call failed     */
    LBVH_ERR_EMPTY_SCENE = 4,  /* n == 0 (tree.py:186-188)                 */
    LBVH_ERR_TOO_LARGE = 5     /* n or nq beyond the supported 2^30 - 1    */
};

/* Device status-word bits. */
#define LBVH_FLAG_STACK_EXHAUSTED 0x01u /* _kernels.py:220-223,274-277,397-400 */
#define LBVH_FLAG_BUFFER_OVERFLOW 0x02u /* _kernels.py:267-270 (1P)          */
#define LBVH_FLAG_NONFINITE 0x04u       /* validation.py:18-22               */
#define LBVH_FLAG_INVERTED_BOX 0x08u    /* validation.py:75-77               */
#define LBVH_FLAG_BAD_RADIUS 0x10u      /* validation.py:88-89               */
#define LBVH_FLAG_BAD_K 0x20u           /* validation.py:100-101             */
#define LBVH_FLAG_BAD_TREE 0x40u        /* child / leaf ordinal out of range */

#define LBVH_STACK_CAPACITY 64 /* _kernels.py:15 */
#define LBVH_MAX_ITEMS ((int64_t)1 << 30)

/*
 * Immutable tree view (pkg/src/lbvh/tree.py:122-174).  The reference arrays
 * (node_mins/node_maxs (2n-1)x3 f32, left/right (n-1) i32, leaf_obj n i32)
 * keep the reference's Karras ordinals: internal nodes 0..n-2 (root 0),
 * leaf p at (n-1)+p.  `nodes` is the traversal layout: one 64-byte record
 * per internal node holding both child boxes and both child links (a leaf
 * child is stored as its object ordinal with bit 31 set).  `root_box` points
 * to 6 floats (min xyz, max xyz) of node 0.  `leaf_codes` (optional, n u32)
 * are the Morton codes in leaf order, as produced by lbvh_build; when present
 * (and the query codes are passed) kNN seeds its search radius from the
 * leaves nearest in Morton order.
 */
typedef struct lbvh_tree {
    int64_t n;
    const float *node_mins;
    const float *node_maxs;
    const int32_t *left;
    const int32_t *right;
    const int32_t *leaf_obj;
    const void *nodes;
    const float *root_box;
    const uint32_t *leaf_codes;
    /* Optional (with leaf_codes): (1 << leaf_dir_bits) + 1 u32 entries;
     * entry p = first leaf whose code >> (30 - leaf_dir_bits) >= p
     * (lbvh_leaf_directory).  Turns the kNN seed's lower_bound over
     * leaf_codes into one directory lookup plus a search within a bucket. */
    const uint32_t *leaf_dir;
    int32_t leaf_dir_bits;
    /* LBVH_TREE_* bits describing how the tree was built (0 = unknown). */
    int32_t flags;
} lbvh_tree;

/* Every leaf box is a point (built from (n, 3) input: maxs == mins). */
#define LBVH_TREE_POINT_LEAVES 0x1
/* Leaves ordered by (30-bit code, index) -- the reference's build -- so the
 * Karras node covering any code prefix can be located from leaf_codes. */
#define LBVH_TREE_CODES30 0x2
/* Built by lbvh_build (30- or 63-bit codes; user-built trees: 0). */
#define LBVH_TREE_BUILT 0x4

#define LBVH_NODE_BYTES 64

const char *lbvh_strerror(int code);
/* Last CUDA error string seen by this thread (for LBVH_ERR_CUDA). */
const char *lbvh_last_cuda_error(void);
int lbvh_abi_version(void);
/* Number of kernels this library has launched in this process (diagnostic;
 * lets a harness count device launches inside a timed region). */
uint64_t lbvh_launch_count(void);

/* ---------------------------------------------------------------- build */

/* Workspace for lbvh_build / lbvh_sort_pairs / lbvh_query_order. */
size_t lbvh_build_workspace_bytes(int64_t n);
size_t lbvh_sort_workspace_bytes(int64_t n);

/*
 * build(boxes) -> Bvh          replaces tree.py:177-209
 *   (check_boxes value checks validation.py:43-78, scene reduce tree.py:189-190,
 *    f64 centroids tree.py:191-192, morton_codes morton.py:68-91, stable argsort
 *    tree.py:194, leaf gather tree.py:196-199, generate_topology tree.py:85-105,
 *    refit_bounds tree.py:108-119)
 * mins, maxs: n x 3 f32 (maxs may equal mins for point input).
 * Outputs: node_mins/node_maxs (2n-1)x3, left/right (n-1), leaf_obj n,
 * root_box 6 floats (== scene box), nodes (n-1) x 64 B, status word.
 * sorted_codes (optional, may be NULL): n u32 30-bit Morton codes in leaf order.
 * leaf_dir (optional, may be NULL): the kNN seed's leaf directory over
 * sorted_codes with leaf_dir_bits <= 24 ((1 << bits) + 1 u32, exactly what
 * lbvh_leaf_directory writes), produced inside the hierarchy pass.
 * flags: LBVH_BUILD_DEFER_ROWS leaves the reference-layout rows no query reads
 * unwritten -- the internal rows of node_mins/node_maxs and, for point input
 * (mins == maxs), the node_maxs leaf rows; lbvh_finish_rows writes them
 * (bit-identical) when the caller first needs the reference layout.  The
 * packed records, node_mins leaf rows, left/right and leaf_obj are always
 * written.
 * leaf_ids (optional, may be NULL): n i32 ordinals in [0, 2^31) reported for
 * the inputs -- leaf_obj[p] and the packed leaf links hold leaf_ids[index]
 * instead of the index (a shard of a distributed cloud reports global
 * ordinals; ties still break by input index, which must then follow the
 * ordinals' order).
 * morton_bits: 30 = the reference's codes (bit-exact tree); 63 = 21 bits per
 * axis, the same recipe (north_star "30/63-bit"; not in the reference, so
 * its parity is pinned only by the oracle restatement).  Leaves are then
 * ordered by (63-bit code, index), finer for very large clouds.
 */
int lbvh_build(const float *mins, const float *maxs, int64_t n, int morton_bits,
               void *workspace, size_t workspace_bytes, float *node_mins, float *node_maxs,
               int32_t *left, int32_t *right, int32_t *leaf_obj, float *root_box,
               void *nodes, uint32_t *sorted_codes, uint32_t *leaf_dir, int leaf_dir_bits,
               int flags, const int32_t *leaf_ids, uint32_t *status, void *stream);
#define LBVH_BUILD_DEFER_ROWS 0x1

/* The rows an LBVH_BUILD_DEFER_ROWS build left out (internal rows from the
 * packed records with the refit's left-first fold; node_maxs leaf rows copied
 * from node_mins when tree->flags has LBVH_TREE_POINT_LEAVES). */
int lbvh_finish_rows(const lbvh_tree *tree, float *node_mins, float *node_maxs, void *stream);

/* Leaf directory over the build's sorted 30-bit leaf codes (kNN seed index;
 * no reference counterpart).  lbvh_leaf_directory_bits(n) is the bucket
 * count exponent used by the Python layer: a multiple of 3 (buckets are
 * cubic cells, >= 2.5 leaves each on average, <= 24 bits), which lets the kNN
 * seed scan the 2x2x2 cells around a query; other bit counts fall back to a
 * Morton-window seed. */
int lbvh_leaf_directory_bits(int64_t n);
int lbvh_leaf_directory(const uint32_t *leaf_codes, int64_t n, int bits, uint32_t *dir,
                        void *stream);

/* morton_codes(points, scene_min, scene_max)   replaces morton.py:68-91
 * points n x 3 f64 (device); scene bounds host doubles (smin[3], smax[3]). */
int lbvh_morton_codes(const double *points, int64_t n, const double *scene_min_host,
                      const double *scene_max_host, uint32_t *codes, void *stream);

/* The same 30-bit codes from f32 points (device) on a device scene box of 6
 * f32 (min xyz, max xyz): coordinates convert to f64 exactly. */
int lbvh_morton_codes_f32(const float *points, int64_t n, const float *scene_box,
                          uint32_t *codes, void *stream);

/* Stable LSD radix sort of (key, value) pairs, in place; sorts the low
 * key_bits bits.  Replaces np.argsort(kind="stable") (tree.py:194) when
 * values are the identity. */
int lbvh_sort_pairs(uint32_t *keys, uint32_t *values, int64_t n, int key_bits,
                    void *workspace, size_t workspace_bytes, void *stream);

/* generate_topology(sorted_codes)   replaces tree.py:85-105 / _kernels.py:61-115
 * left/right (n-1) i32, parent (2n-1) i32 (parent[0] = -1).  Workspace:
 * lbvh_topology_workspace_bytes(n). */
size_t lbvh_topology_workspace_bytes(int64_t n);
int lbvh_generate_topology(const uint32_t *sorted_codes, int64_t n, int32_t *left,
                           int32_t *right, int32_t *parent, void *workspace,
                           size_t workspace_bytes, void *stream);

/* refit_bounds(node_mins, node_maxs, topology)   replaces tree.py:108-119 /
 * _kernels.py:118-138: fills internal boxes from leaf boxes in place. */
int lbvh_refit(float *node_mins, float *node_maxs, const int32_t *left,
               const int32_t *right, const int32_t *parent, int64_t n, void *workspace,
               size_t workspace_bytes, void *stream);

/* Pack a reference-layout tree (e.g. a user-constructed Bvh) into the
 * traversal layout.  Sets LBVH_FLAG_BAD_TREE on out-of-range links. */
int lbvh_pack(const lbvh_tree *tree, void *nodes, float *root_box, uint32_t *status,
              void *stream);

/* Unpack: traversal layout + root box -> reference node_mins/node_maxs. */
int lbvh_unpack_boxes(const lbvh_tree *tree, float *node_mins, float *node_maxs,
                      void *stream);

/* ---------------------------------------------------------------- query */

/* Traversal order of a query batch (the role of traversal.py:146-165's
 * pre-sort).  order: nq u32 permutation.  scene_box: 6 floats DEVICE (tree
 * root box).  sorted_codes (optional): the queries' Morton codes in `order`
 * order (kNN seed).  order_bits: sort by the top order_bits of the 30-bit
 * code.  Codes use fp32 cell arithmetic and may differ from the reference's
 * f64 codes on cell boundaries: any order gives identical query results; the
 * exact reference permutation (query_sort_order) is lbvh_morton_codes +
 * lbvh_sort_pairs.  The drivers use 24 bits (3 radix passes). */
size_t lbvh_query_workspace_bytes(int64_t nq);
int lbvh_query_order(const float *centers, int64_t nq, const float *scene_box,
                     int order_bits, uint32_t *order, uint32_t *sorted_codes, void *workspace,
                     size_t workspace_bytes, void *stream);

/* Finite check of nq x 3 query centers and (optional) radii >= 0. */
int lbvh_check_queries(const float *centers, int64_t nq, const float *radii,
                       uint32_t *status, void *stream);

/* spatial_pass(store=False)  replaces _kernels.py:179-228 (count pass of
 * query_spatial_2p, traversal.py:197-201).  radii may be NULL -> radius.
 * order may be NULL -> identity.  counts: nq i32.  buf (optional, nq x
 * buffer_size i32): the first buffer_size hits of every query are kept in
 * its row in traversal order, so the fill pass only has to revisit queries
 * whose count exceeds buffer_size (see lbvh_spatial_fill / lbvh_compact). */
int lbvh_spatial_count(const lbvh_tree *tree, const float *centers, const float *radii,
                       float radius, const uint32_t *order, int64_t nq, int32_t *counts,
                       int32_t *buf, int64_t buffer_size, uint32_t *status, void *stream);

/* spatial_pass(store=True)  replaces _kernels.py:179-228 (fill pass,
 * traversal.py:205-209); writes out[offsets[q] ...].  skip_counts
 * (optional): counts of a buffered count pass; queries with count <=
 * buffer_size are skipped (lbvh_compact copies their rows). */
int lbvh_spatial_fill(const lbvh_tree *tree, const float *centers, const float *radii,
                      float radius, const uint32_t *order, int64_t nq,
                      const int64_t *offsets, int32_t *out, const int32_t *skip_counts,
                      int64_t buffer_size, uint32_t *status, void *stream);

/* _exclusive_scan   replaces traversal.py:173-176: offsets[0]=0,
 * offsets[i+1] = sum(counts[0..i]); offsets is nq+1 i64.  Also copies the
 * total to *total_out (device, may be NULL). */
size_t lbvh_scan_workspace_bytes(int64_t nq);
int lbvh_exclusive_scan(const int32_t *counts, int64_t nq, int64_t *offsets,
                        void *workspace, size_t workspace_bytes, void *stream);

/* spatial_pass_buffered  replaces _kernels.py:231-282 (query_spatial_1p,
 * traversal.py:214-248): buf nq x buffer_size i32, counts nq i32. */
int lbvh_spatial_1p(const lbvh_tree *tree, const float *centers, const float *radii,
                    float radius, const uint32_t *order, int64_t nq, int32_t *buf,
                    int64_t buffer_size, int32_t *counts, uint32_t *status, void *stream);

/* Queries (taken in `order`, may be NULL) whose count exceeds buffer_size:
 * written to list (u32 query ids), *list_len (device u32) = how many.  The
 * fill pass then runs with order = list, nq = *list_len. */
int lbvh_select_overflow(const uint32_t *order, const int32_t *counts, int64_t nq,
                         int64_t buffer_size, uint32_t *list, uint32_t *list_len, void *stream);

/* compact_rows  replaces _kernels.py:285-290.  Rows with counts[q] >
 * buffer_size are skipped (they did not fit; see lbvh_spatial_fill). */
int lbvh_compact(const int32_t *buf, int64_t buffer_size, const int32_t *counts,
                 const int64_t *offsets, int64_t nq, int32_t *out, void *stream);

/* kNN spans  replaces traversal.py:261-262: spans = min(k_q, n), offsets =
 * scan(spans).  ks may be NULL -> uniform k (k < 1 is LBVH_ERR_INVALID_ARG;
 * offsets are written directly, no scan).  Sets LBVH_FLAG_BAD_K for ks < 1 and
 * writes max span to *max_span (device i32). */
int lbvh_knn_offsets(const int64_t *ks, int64_t k, int64_t n, int64_t nq, int64_t *offsets,
                     int32_t *max_span, uint32_t *status, void *workspace,
                     size_t workspace_bytes, void *stream);

/* knn_pass  replaces _kernels.py:328-414 (query_knn, traversal.py:251-272).
 * max_span: host upper bound of min(k_q, n) (selects the kernel variant).
 * query_codes (optional): Morton codes of the queries in `order` order (from
 * lbvh_query_order); with tree->leaf_codes they enable the search-radius
 * seed, which never changes results.  flags: LBVH_KNN_SQUARED writes the
 * squared distances (no sqrt) -- used by the distributed merge, which must
 * order candidates by exact (d^2, ordinal). */
#define LBVH_KNN_SQUARED 0x1
/* offsets[q] == q * max_span for every query (uniform k): the kernel computes
 * span starts instead of reading them (the offsets array is still read by
 * the other paths and must hold the same values). */
#define LBVH_KNN_UNIFORM_SPANS 0x2
/* workspace: reserved for future variants; accepted and unused today
 * (lbvh_knn_workspace_bytes returns 0; NULL / 0 is valid). */
size_t lbvh_knn_workspace_bytes(int64_t nq);
int lbvh_knn(const lbvh_tree *tree, const float *centers, const uint32_t *order,
             const uint32_t *query_codes, int64_t nq, const int64_t *offsets,
             int64_t max_span, int32_t *out_idx, float *out_dist, int flags,
             void *workspace, size_t workspace_bytes, uint32_t *status, void *stream);

/* query_spatial_2p's count stage for device-resident centers in one call:
 * value checks, Morton query order (order_bits; 0 = unsorted, `order` then
 * unused), the count pass keeping the first `rows` hits of every query in
 * buf (rows 0: no row buffer), the exclusive scan into offsets (nq+1) and
 * the list of queries whose hits overflowed their row (over_list, over_n).
 * Spill pool (optional, spill_pool != NULL): the count pass keeps a query's
 * hits beyond its row too, in chunks of LBVH_SPILL_CHUNK ints drawn from
 * spill_pool (spill_chunks chunks, chunk 0 reserved; each chunk holds
 * LBVH_SPILL_CHUNK - 1 hits then the index of the next), the first chunk of
 * query q in spill_heads[q] (nq i32, written for overflowing queries only;
 * -1 = pool exhausted).  Overflowing queries fully held by the pool are
 * listed in spill_list / spill_n (copy them with lbvh_spill_copy); only the
 * rest go to over_list (fill pass).  Hit order is the fill order either way.
 * ev_before / ev_after (optional) bracket the count kernel. */
#define LBVH_SPILL_CHUNK 256
size_t lbvh_spatial_count_batch_workspace_bytes(int64_t nq);
int lbvh_spatial_count_batch(const lbvh_tree *tree, const float *centers, const float *radii,
                             float radius, int64_t nq, int order_bits, int64_t rows,
                             uint32_t *order, int32_t *counts, int32_t *buf, int64_t *offsets,
                             uint32_t *over_list, uint32_t *over_n, int32_t *spill_heads,
                             int32_t *spill_pool, int64_t spill_chunks, uint32_t *spill_list,
                             uint32_t *spill_n, void *workspace, size_t workspace_bytes,
                             uint32_t *status, void *ev_before, void *ev_after, void *stream);

/* The spans of the spilled queries (spill_list, its length spill_n on the
 * device, at most max_list): row hits then pool chunks, into out at
 * offsets[q] -- the complement of lbvh_compact, which skips overflowed rows. */
int lbvh_spill_copy(const int32_t *buf, int64_t rows, const int32_t *counts,
                    const int64_t *offsets, const int32_t *spill_heads, const int32_t *spill_pool,
                    const uint32_t *spill_list, const uint32_t *spill_n, int64_t max_list,
                    int32_t *out, void *stream);

/* spatial_pass(store=True) (_kernels.py:179-228) for the listed queries
 * only (list: query ids, typically over_list of lbvh_spatial_count_batch):
 * writes their whole spans at offsets[q].  list_len (device, optional) holds
 * n_list; with it a persistent grid walks the list in order (the queries in
 * flight stay a contiguous stretch of it), else one thread per entry.  Same
 * bytes either way. */
int lbvh_spatial_fill_list(const lbvh_tree *tree, const float *centers, const float *radii,
                           float radius, const uint32_t *list, const uint32_t *list_len,
                           int64_t n_list, const int64_t *offsets, int32_t *out,
                           uint32_t *status, void *stream);

/* query_knn for device-resident centers and a uniform k in one call: value
 * checks (LBVH_FLAG_NONFINITE), uniform CRS offsets (nq+1), Morton query
 * order on the tree's grid (order_bits of the 30-bit code; 0 = unsorted) and
 * the search.  Workspace: lbvh_knn_batch_workspace_bytes(nq).  kth_d2
 * (optional, k <= 32) receives each query's exact k-th squared distance as
 * lbvh_knn_kth.  ev_before / ev_after (optional cudaEvent_t) are recorded
 * around the search kernel on `stream` (kernel timing inside a caller's
 * timed region). */
size_t lbvh_knn_batch_workspace_bytes(int64_t nq);
int lbvh_knn_batch(const lbvh_tree *tree, const float *centers, int64_t nq, int64_t k,
                   int order_bits, int64_t *offsets, int32_t *out_idx, float *out_dist,
                   int flags, void *workspace, size_t workspace_bytes, uint32_t *status,
                   float *kth_d2, void *ev_before, void *ev_after, void *stream);

/* lbvh_knn that also writes kth_d2[q] = the exact squared distance of query
 * q's last (k-th) neighbour -- the sharded search's forwarding bound -- so
 * the outputs can be the final sqrt'ed lists.  max_span <= 32 only. */
int lbvh_knn_kth(const lbvh_tree *tree, const float *centers, const uint32_t *order,
                 const uint32_t *query_codes, int64_t nq, const int64_t *offsets,
                 int64_t max_span, int32_t *out_idx, float *out_dist, int flags,
                 void *workspace, size_t workspace_bytes, uint32_t *status, float *kth_d2,
                 void *stream);

/* Distributed kNN merge epilogue (no reference counterpart):
 * merged candidate keys (dist^2 bits << 32 | global ordinal) -> ordinals and
 * correctly rounded distances sqrt(dist^2), as knn_pass's final sqrt
 * (_kernels.py:413-414). */
int lbvh_unpack_knn_keys(const uint64_t *keys, int64_t n, int64_t *ordinals, float *dist,
                         void *stream);

/* ---------------------------------------------------------- brute force */

/* brute_knn / brute_knn_batch   replaces oracle.py:35-45, 62-70: O(n) per
 * query; out_idx / out_dist are nq x min(k, n), sorted by (d, ordinal). */
int lbvh_brute_knn(const float *points, int64_t n, const float *centers, int64_t nq, int64_t k,
                   int32_t *out_idx, float *out_dist, void *stream);

/* brute_radius / brute_radius_sets   replaces oracle.py:26-32, 48-59.
 * offsets == NULL: writes counts (nq i32); else fills ascending ordinals at
 * out[offsets[q] ...].  radii may be NULL -> radius. */
int lbvh_brute_radius(const float *points, int64_t n, const float *centers, const float *radii,
                      float radius, int64_t nq, int32_t *counts, const int64_t *offsets,
                      int32_t *out, void *stream);

/* ------------------------------------------------- benchmark clouds */

/* datasets.generate(CloudSpec) on the device (datasets.py:95-153), bit for
 * bit numpy's PCG64 stream: kind 0 cube:filled, 1 cube:hollow, 2
 * sphere:hollow; a = count^(1/3), lim = float32(a); (st, inc) = numpy's
 * PCG64(seed).state.  out: p x 3 f32.  sphere:hollow sets
 * LBVH_FLAG_NONFINITE when numpy would redraw a point (norm < 1e-6). */
int lbvh_generate_cloud(int kind, int64_t p, double a, float lim, uint64_t st_hi,
                        uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, float *out,
                        uint32_t *status, void *stream);

/* ------------------------------------------- sharded search (multi-GPU) */

/* Sharded kNN / radius helpers (distributed.py; no reference counterpart --
 * the reference is single-process).  world <= 32 ranks.
 * rank_forward_mask: mask[q] bit r set iff rank r is in `candidates` and its
 * box (boxes: world x 6 f32) has fp32 distance^2 <= bound[q] (or radius2 when
 * bound is NULL), the traversal's box-distance recipe. */
int lbvh_rank_forward_mask(const float *centers, const float *bound, float radius2, int64_t m,
                           const float *boxes, int world, uint32_t candidates, uint32_t *mask,
                           void *stream);
/* Radius forwarding at the origin.  phase 0: per_rank[d] = number of set
 * bits d over mask[0..m) (world u32).  phase 1: rows (sum(per_rank) x 5
 * f32: x, y, z, radius, query id bits) written into rank d's region starting
 * at start[d] (device i64, world), cursor (world u32) is scratch. */
int lbvh_forward_rows(const float *centers, const float *radii, const uint32_t *mask, int64_t m,
                      int world, uint32_t *per_rank, int64_t *start, uint32_t *cursor,
                      float *rows, int phase, void *stream);
/* Radius merge at the origin.  sent_rows: the rows this rank forwarded
 * (n_rec x 5, as lbvh_forward_rows wrote them); rec_counts[i]: hits the
 * destination found for row i (returned in send order); phase 0 adds them
 * into totals_or_cursor[q] (nq i32, caller-zeroed).  phase 1: rec_off =
 * exclusive scan of rec_counts (positions in `hits`, the sources' hits
 * concatenated in rank order), offsets = exclusive scan of the totals,
 * source_starts (HOST i64, world + 1) = record ranges per source rank;
 * each query's hits are appended source by source (rank order), each
 * source's in its traversal (fill) order, into out (i64); totals_or_cursor
 * must be zeroed again as the cursor. */
int lbvh_merge_records(const float *sent_rows, const int32_t *rec_counts, const int64_t *rec_off,
                       int64_t n_rec, const int64_t *source_starts, int world,
                       const int32_t *hits, const int64_t *offsets, int32_t *totals_or_cursor,
                       int64_t *out, int phase, void *stream);
/* Renumber a local tree's leaves with global ordinals (map[local] ->
 * global, < 2^31) in leaf_obj and in the packed leaf links, so its queries
 * report -- and break distance ties by -- global ordinals. */
int lbvh_remap_leaves(const lbvh_tree *tree, int32_t *leaf_obj, void *nodes, const int64_t *map,
                      void *stream);
/* Home kNN lists -> return arrays out_dist = sqrt(d^2) (f32) and out_gid
 * (i32 global ordinal), m x kk, in row order; rows with merged_pos[q] >= 0
 * take merged[merged_pos[q]] (kk sorted (d^2 bits << 32 | ordinal) keys).
 * gids NULL: local_idx are global already.  merged_pos may be NULL. */
int lbvh_knn_finalize(int64_t m, int kk, const int32_t *local_idx, const float *d2,
                      const int64_t *gids, const int64_t *merged_pos, const uint64_t *merged,
                      float *out_dist, int32_t *out_gid, void *stream);
/* dst row i = src row idx[i] (3 f32 per row): queries into send order. */
int lbvh_gather_rows3(const float *src, const int64_t *idx, int64_t n, float *dst,
                      void *stream);
/* m received rows (rd f32, rg i32; m x kk) -> out_d / out_g rows dst[i]. */
int lbvh_scatter_result_rows(int64_t m, int kk, const int64_t *dst, const float *rd,
                             const int32_t *rg, float *out_d, int32_t *out_g, void *stream);
#ifdef __cplusplus
}
#endif

#endif /* LBVH_B200_H */
