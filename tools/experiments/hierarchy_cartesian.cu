// EXPERIMENT (not compiled into the library): the CTA-local hierarchy as a
// Cartesian tree of the split prefixes -- PSE/NSE by binary descent over a
// min sparse table, node boxes from a leftmost min/max sparse table -- in its
// last (persistent, prefetching) form.  Byte-identical trees, but measured
// slower than the Apetrei climb in csrc/build.cu (DESIGN.md section 4,
// "Explored and rejected"): 0.64-0.69 ms vs 0.63 ms for the local kernel at
// 1e7, bound by shared-memory latency of the descent and table builds.
// Drop-in replacement for the section of csrc/build.cu between the
// "Hierarchy (K4+K5)" banner and frontier_box().

// ---------------------------------------------------------------------------
// Hierarchy (K4+K5), in two levels.
//
// The topology is the Cartesian tree of the split prefixes: with augmented
// keys (code, position) every node range [l, r] has a unique boundary of
// minimal prefix delta (its split g), and the boundaries just outside it,
// l - 1 and r, both have smaller prefixes.  So the node split at boundary g
// spans [PSE(g) + 1, NSE(g)], PSE / NSE = nearest boundary on the left /
// right with a smaller delta -- exactly the node find_split / node_range
// build top-down (tree.py:85-105, _kernels.py:50-98).  Its box, the refit's
// left-first fold (_kernels.py:116-138), is the leftmost minimum / maximum
// over the leaves of the range: min(a, b) keeps a unless b < a, so any
// association order returns the leftmost extreme's bits -- the fold does not
// depend on the tree shape.
//
// hierarchy_local_kernel: CTA c owns leaves [B, B + T).  It stages the
// prefixes of boundaries B - 1 .. B + T - 1 and the leaf boxes in shared
// memory, builds sparse tables over both (min prefix / leftmost box over 2^k
// entries), then every interior boundary finds PSE and NSE by a binary
// descent and, if both lie inside the CTA, writes its node (Karras ordinal,
// packed record with both child boxes from two table lookups each, left /
// right) -- no handshakes, no climb, no divergence beyond the range test.
// Finished nodes whose parent is not local hand over to the global climb:
// a parent split at an interior boundary gets the child's far end published
// in its hand-off slot (the child is its first arrival); a parent split at
// the CTA's edge boundary gets the child appended to the frontier list.
//
// hierarchy_frontier_kernel: the frontier nodes continue with a global
// handshake (release exchange; the second arrival fences acq_rel before it
// reads the sibling's record).  A published slot is indistinguishable from a
// frontier first arrival, so the meeting rule is unchanged.  It also writes
// the leaf-directory runs the local kernel deferred.
// ---------------------------------------------------------------------------
#ifndef LBVH_HIER_T
#define LBVH_HIER_T 128
#endif
constexpr int kHierT = LBVH_HIER_T;
constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }
constexpr int kBoxLevels = ilog2c(kHierT);        // S_k, k < log2 T: local ranges < T leaves
constexpr int kDeltaLevels = ilog2c(kHierT) + 1;  // D_k over the T + 1 boundaries
constexpr int kDPitch = kHierT + 16;
// Leaf-directory runs longer than this (empty buckets between two adjacent
// leaves: clustered clouds) are deferred to the frontier kernel, where the
// whole grid writes them.
constexpr int64_t kDirInline = 32;

struct DirRun {
    uint32_t lo, hi, value, pad;  // dir[lo, hi) = value
};

__device__ __forceinline__ void dir_run(uint32_t *__restrict__ dir, int64_t lo, int64_t hi,
                                        uint32_t value, DirRun *runs, uint32_t *run_count) {
    if (hi - lo <= kDirInline) {
        for (int64_t b = lo; b < hi; ++b) dir[b] = value;
    } else {
        const uint32_t at = atomicAdd(run_count, 1u);
        runs[at] = DirRun{(uint32_t)lo, (uint32_t)hi, value, 0u};
    }
}

// Box of 2^k leaves as {lo.x, lo.y, lo.z, hi.x} + {hi.y, hi.z}: two vector
// shared-memory accesses per box, conflict-free for consecutive entries.
template <typename CodeT>
struct HierSmem {
    float4 box4[kBoxLevels][kHierT];
    float2 box2[kBoxLevels][kHierT];
    int32_t link[kHierT];              // leaf links (obj | kLeafTag)
    CodeT code[kHierT + 2];            // codes[B - 1 + i]
    uint8_t d[kDeltaLevels][kDPitch];  // D_k[i]: boundaries B - 1 + [i, i + 2^k); delta + 1, 0 = none
    uint8_t local[kHierT];             // boundary B + i has a CTA-local node
};

template <typename CodeT>
constexpr size_t hier_smem_bytes() { return sizeof(HierSmem<CodeT>); }

__device__ __forceinline__ void fold_box(const float4 &a4, const float2 &a2, const float4 &b4,
                                         const float2 &b2, float4 &o4, float2 &o2) {
    o4 = make_float4(min_left(a4.x, b4.x), min_left(a4.y, b4.y), min_left(a4.z, b4.z),
                     max_left(a4.w, b4.w));
    o2 = make_float2(max_left(a2.x, b2.x), max_left(a2.y, b2.y));
}

// Box of local leaves [a, b] from two overlapping 2^k blocks (leftmost rule).
template <typename CodeT>
__device__ __forceinline__ void range_box(const HierSmem<CodeT> &S, int a, int b, Box &out) {
    const int k = 31 - __clz(b - a + 1);
    const int b2 = b - (1 << k) + 1;
    float4 o4;
    float2 o2;
    fold_box(S.box4[k][a], S.box2[k][a], S.box4[k][b2], S.box2[k][b2], o4, o2);
    out = Box{{o4.x, o4.y, o4.z}, {o4.w, o2.x, o2.y}};
}

template <typename CodeT>
__global__ void __launch_bounds__(kHierT)
hierarchy_local_kernel(const CodeT *__restrict__ codes, const uint32_t *__restrict__ perm,
                       const float *__restrict__ mins, const float *__restrict__ maxs, int64_t n,
                       uint32_t *__restrict__ slots, float *__restrict__ node_mins,
                       float *__restrict__ node_maxs, bool leaf_maxs_rows,
                       int32_t *__restrict__ left, int32_t *__restrict__ right,
                       int32_t *__restrict__ leaf_obj, PackedNode *__restrict__ nodes,
                       float *__restrict__ root_box, uint32_t *__restrict__ leaf_codes,
                       uint32_t *__restrict__ leaf_dir, int dir_bits, DirRun *runs,
                       uint32_t *run_count, uint2 *__restrict__ frontier,
                       uint32_t *frontier_count, const int32_t *__restrict__ leaf_ids) {
    extern __shared__ __align__(16) unsigned char hier_smem_raw[];
    HierSmem<CodeT> &S = *reinterpret_cast<HierSmem<CodeT> *>(hier_smem_raw);
    const int tid = threadIdx.x;
    const int64_t internal = n - 1;
    const int64_t ntiles = (n + kHierT - 1) / kHierT;
    const bool same = (mins == maxs);
    // Persistent CTAs: the next tile's codes and sorted permutation are
    // loaded while this tile builds its tables, its leaf boxes gathered
    // while this tile builds its nodes (registers, committed next iteration).
    CodeT pc0 = 0, pc1 = 0;
    uint32_t pobj = 0, pgobj = 0;
    Box pb = Box{{0.f, 0.f, 0.f}, {0.f, 0.f, 0.f}};
    auto fetch_ids = [&](int64_t t) {
        const int64_t b = t * kHierT;
        const int64_t j = b - 1 + tid;
        if (j >= 0 && j < n) pc0 = __ldg(codes + j);
        if (tid < 2 && b - 1 + kHierT + tid < n) pc1 = __ldg(codes + b - 1 + kHierT + tid);
        if (b + tid < n) pobj = __ldg(perm + b + tid);
    };
    auto fetch_boxes = [&](int64_t t) {
        if (t * kHierT + tid < n) {
            // the ordinal this leaf reports: its input index, or leaf_ids[index]
            pgobj = leaf_ids ? (uint32_t)__ldg(leaf_ids + pobj) : pobj;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                pb.lo[a] = __ldg(mins + 3 * (int64_t)pobj + a);
                pb.hi[a] = same ? pb.lo[a] : __ldg(maxs + 3 * (int64_t)pobj + a);
            }
        }
    };
    int64_t tile = blockIdx.x;
    if (tile < ntiles) {
        fetch_ids(tile);
        fetch_boxes(tile);
    }
    for (; tile < ntiles; tile += gridDim.x) {
        const int64_t B = tile * kHierT;
        const int nloc = (int)(n - B < kHierT ? n - B : kHierT);
        const int64_t p = B + tid;
        const int64_t next = tile + gridDim.x;
        // this tile's window of the global hand-off slots starts empty
        // (ordered before the publications below by the barriers)
        if (p < n - 1) slots[p] = 0u;
        S.code[tid] = pc0;
        if (tid < 2) S.code[kHierT + tid] = pc1;
        if (tid < nloc) {
            leaf_obj[p] = (int32_t)pgobj;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                node_mins[3 * (internal + p) + a] = pb.lo[a];
                if (leaf_maxs_rows) node_maxs[3 * (internal + p) + a] = pb.hi[a];
            }
            S.link[tid] = (int32_t)(pgobj | kLeafTag);
            if (n == 1) {  // leaf-only tree (tree.py:177-209 with n == 1)
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    root_box[a] = pb.lo[a];
                    root_box[3 + a] = pb.hi[a];
                }
            }
        }
        S.box4[0][tid] = make_float4(pb.lo[0], pb.lo[1], pb.lo[2], pb.hi[0]);
        S.box2[0][tid] = make_float2(pb.hi[1], pb.hi[2]);
        __syncthreads();
        if (next < ntiles) fetch_ids(next);
        if (tid < nloc) {
            const uint32_t c30 = code30(S.code[tid + 1]);
            if (leaf_codes) leaf_codes[p] = c30;
            if (leaf_dir) {
                // dir[b] = first leaf whose code >> (30 - bits) >= b: leaf p owns
                // the buckets after its predecessor's, the last leaf the tail = n
                const int sh = 30 - dir_bits;
                const int64_t cb = (int64_t)(c30 >> sh);
                const int64_t pb_ = p == 0 ? -1 : (int64_t)(code30(S.code[tid]) >> sh);
                dir_run(leaf_dir, pb_ + 1, cb + 1, (uint32_t)p, runs, run_count);
                if (p == n - 1)
                    dir_run(leaf_dir, cb + 1, ((int64_t)1 << dir_bits) + 1, (uint32_t)n, runs,
                            run_count);
            }
        }
        // D_0: boundary B - 1 + i (keys j, j + 1); none before key 0 or after n - 1
        S.d[0][tid + 1] = p < n - 1
                              ? (uint8_t)(delta_of(S.code[tid + 1], S.code[tid + 2], p) + 1)
                              : (uint8_t)0;
        if (tid == 0)
            S.d[0][0] = B > 0 ? (uint8_t)(delta_of(S.code[0], S.code[1], B - 1) + 1) : 0;
#pragma unroll
        for (int k = 1; k < kDeltaLevels; ++k) {
            __syncthreads();
            const int h = 1 << (k - 1);
            if (tid + 2 * h <= kHierT + 1) {
                const uint8_t x = S.d[k - 1][tid], y = S.d[k - 1][tid + h];
                S.d[k][tid] = x < y ? x : y;
            }
            if (k < kBoxLevels && tid + 2 * h <= kHierT)
                fold_box(S.box4[k - 1][tid], S.box2[k - 1][tid], S.box4[k - 1][tid + h],
                         S.box2[k - 1][tid + h], S.box4[k][tid], S.box2[k][tid]);
        }
        __syncthreads();
        if (next < ntiles) fetch_boxes(next);

        // Node split at interior boundary g = B + tid (keys g, g + 1 both local).
        int lo = 0, hi = 0;  // local range [lo, hi] (leaf offsets) when local
        bool local = false;
        if (tid < kHierT - 1 && p < n - 1) {
            const int i0 = tid + 1;
            const uint8_t v = S.d[0][i0];
            int a = i0;      // PSE: largest i < i0 with D_0[i] < v (all of [a, i0) >= v)
            int b = i0 + 1;  // NSE: smallest i > i0 with D_0[i] < v (all of (i0, b) >= v)
#pragma unroll
            for (int k = kDeltaLevels - 1; k >= 0; --k) {
                const int w = 1 << k;
                if (a - w >= 0 && S.d[k][a - w] >= v) a -= w;
                if (b + w - 1 <= kHierT && S.d[k][b] >= v) b += w;
            }
            // D_0 index i is boundary B - 1 + i: PSE index a - 1 is boundary
            // l - 1, NSE index b is boundary r
            local = a >= 1 && b <= kHierT;
            lo = a - 1;
            hi = b - 1;
            if (local) {
                const int64_t g = p, l = B + lo, r = B + hi;
                const int64_t lc = (l == g) ? internal + g : g;
                const int64_t rc = (g + 1 == r) ? internal + g + 1 : g + 1;
                const bool root = (l == 0 && r == n - 1);
                // left child <=> delta(r) > delta(l - 1) (none = 0 covers l == 0 / r == n - 1)
                const bool is_left = S.d[0][hi + 1] > S.d[0][lo];
                const int64_t id = root ? 0 : (is_left ? r : l);
                Box L, R;
                range_box(S, lo, tid, L);
                range_box(S, tid + 1, hi, R);
                const int32_t ll = (l == g) ? S.link[tid] : (int32_t)lc;
                const int32_t rl = (g + 1 == r) ? S.link[tid + 1] : (int32_t)rc;
                store_packed(nodes, id, L, R, ll, rl);
                left[id] = (int32_t)lc;
                right[id] = (int32_t)rc;
                if (root) {
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        root_box[c] = min_left(L.lo[c], R.lo[c]);
                        root_box[3 + c] = max_left(L.hi[c], R.hi[c]);
                    }
                }
            }
        }
        S.local[tid] = local;
        __syncthreads();

        // Hand-over of finished nodes whose parent is not CTA-local: this
        // node (if any) and leaf p.
        auto hand_over = [&](int nl, int nr) {
            if (B + nl == 0 && B + nr == n - 1) return;  // the root
            const bool is_left = S.d[0][nr + 1] > S.d[0][nl];
            const int gp = is_left ? nr : nl - 1;  // the parent's split (local offset)
            const uint32_t known = (uint32_t)(B + (is_left ? nl : nr));
            if (gp >= 0 && gp < kHierT - 1) {       // interior boundary
                if (!S.local[gp]) slots[B + gp] = known + 1u;  // first arrival
            } else {                                // tile edge: global handshake
                const uint32_t at = atomicAdd(frontier_count, 1u);
                frontier[at] = make_uint2((uint32_t)(B + nl), (uint32_t)(B + nr));
            }
        };
        if (local) hand_over(lo, hi);
        if (tid < nloc && n > 1) hand_over(tid, tid);
        __syncthreads();  // the next tile overwrites the shared tables
    }
}

