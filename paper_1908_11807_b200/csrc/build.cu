// build.cu -- LBVH construction on sm_100a.
//
// Pipeline (reference tree.py:177-209):
//   K1 scene_reduce_kernel   scene box + value checks       tree.py:189-190, validation.py:43-78
//   K2 morton_kernel         f64 centroid + 30-bit code     tree.py:191-193, morton.py:68-91
//   K3 sort_pairs            stable (code, index) sort      tree.py:194
//   K4+K5 hierarchy_kernel   leaf gather + single-pass bottom-up hierarchy
//                            emitting Karras ordinals + atomic-flag refit +
//                            packed node records            tree.py:85-119, 196-199
//
// The hierarchy kernel is Apetrei's bottom-up construction: one thread per
// leaf climbs; at every node it decides whether it is a left or right child
// from the two boundary prefix lengths, meets its sibling at the split slot
// through an atomic exchange, and the second arrival builds the parent.  The
// node it builds gets exactly the Karras ordinal of the reference's
// top-down generate_topology: a node [l, r] that is a left child has id r, a
// right child has id l, the root id 0, leaf p id (n-1)+p.  So left/right,
// node boxes and leaf order are byte-identical to the reference.

#include "common.cuh"
#include "internal.cuh"

namespace lbvh {
namespace {

constexpr int kReduceThreads = 256;

__device__ __forceinline__ void warp_minmax(float v[6]) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float lo = __shfl_xor_sync(0xFFFFFFFFu, v[a], o);
            float hi = __shfl_xor_sync(0xFFFFFFFFu, v[3 + a], o);
            v[a] = fminf(v[a], lo);
            v[3 + a] = fmaxf(v[3 + a], hi);
        }
    }
}

// K1: scene box (exact min/max) and the check_boxes value checks.  The last
// CTA to finish folds the per-CTA partials (threadfence reduction).
__global__ void __launch_bounds__(kReduceThreads)
scene_reduce_kernel(const float *__restrict__ mins, const float *__restrict__ maxs, int64_t n,
                    float *__restrict__ partials, uint32_t *counter, float *__restrict__ scene,
                    uint32_t *status) {
    float v[6] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
    uint32_t bad = 0;
    const bool same = (mins == maxs);
    int64_t first = 0;
    if (same && (reinterpret_cast<uintptr_t>(mins) & 15) == 0) {
        // points: 4 points = 3 float4 per step, axes in a fixed pattern
        // (build 1.44 vs 1.46 ms against scalar loads)
        const float4 *m4 = reinterpret_cast<const float4 *>(mins);
        const int64_t chunks = n / 4;
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < chunks;
             c += (int64_t)gridDim.x * blockDim.x) {
            const float4 x = __ldcs(m4 + 3 * c), y = __ldcs(m4 + 3 * c + 1),
                         z = __ldcs(m4 + 3 * c + 2);
            const float f[12] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w, z.x, z.y, z.z, z.w};
#pragma unroll
            for (int j = 0; j < 12; ++j) {
                if (!isfinite(f[j])) bad |= LBVH_FLAG_NONFINITE;
                v[j % 3] = fminf(v[j % 3], f[j]);
                v[3 + j % 3] = fmaxf(v[3 + j % 3], f[j]);
            }
        }
        first = chunks * 4;
    }
    for (int64_t i = first + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            float lo = __ldcs(mins + 3 * i + a);
            float hi = same ? lo : __ldcs(maxs + 3 * i + a);
            if (!isfinite(lo) || !isfinite(hi)) bad |= LBVH_FLAG_NONFINITE;
            if (lo > hi) bad |= LBVH_FLAG_INVERTED_BOX;
            v[a] = fminf(v[a], lo);
            v[3 + a] = fmaxf(v[3 + a], hi);
        }
    }
    bad = __reduce_or_sync(0xFFFFFFFFu, bad);
    if (bad && lane_id() == 0) atomicOr(status, bad);
    warp_minmax(v);
    __shared__ float s_part[kReduceThreads / 32][6];
    __shared__ bool s_last;
    const int warp = threadIdx.x >> 5;
    if (lane_id() == 0)
        for (int a = 0; a < 6; ++a) s_part[warp][a] = v[a];
    __syncthreads();
    if (threadIdx.x < 6) {
        int a = threadIdx.x;
        float r = s_part[0][a];
        for (int w = 1; w < kReduceThreads / 32; ++w)
            r = a < 3 ? fminf(r, s_part[w][a]) : fmaxf(r, s_part[w][a]);
        partials[blockIdx.x * 6 + a] = r;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < 6) {
        int a = threadIdx.x;
        float r = __ldcg(partials + a);
        for (unsigned b = 1; b < gridDim.x; ++b) {
            float x = __ldcg(partials + b * 6 + a);
            r = a < 3 ? fminf(r, x) : fmaxf(r, x);
        }
        scene[a] = r;
    }
}

__device__ __forceinline__ void encode(double x, double y, double z, const double *lo,
                                       const double *ext, uint32_t &out) {
    out = morton3(x, y, z, lo, ext);
}
__device__ __forceinline__ void encode(double x, double y, double z, const double *lo,
                                       const double *ext, uint64_t &out) {
    out = morton63(x, y, z, lo, ext);
}

// K2: codes of the f64 box centroids on the scene grid, plus iota values.
// CodeT = uint32_t: the reference's 30-bit codes; uint64_t: 63-bit codes.
#ifndef LBVH_MORTON_CTAS
#define LBVH_MORTON_CTAS 4  // resident CTAs per SM of the fused Morton + histogram pass
#endif
// hist (30-bit codes, optional): the digit histograms of the 4-pass sort
// that follows (sort_prepare), so it needs no histogram pass of its own.
template <typename CodeT>
__global__ void __launch_bounds__(256)
morton_kernel(const float *__restrict__ mins, const float *__restrict__ maxs, int64_t n,
              const float *__restrict__ scene, CodeT *__restrict__ codes,
              uint32_t *__restrict__ iota, uint32_t *__restrict__ hist = nullptr) {
    __shared__ uint32_t s_hist[4][kSortDigits];
    if (hist) {
        for (int i = threadIdx.x; i < 4 * kSortDigits; i += blockDim.x) (&s_hist[0][0])[i] = 0;
        __syncthreads();
    }
    double lo[3], ext[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = (double)scene[a];
        ext[a] = __dsub_rn((double)scene[3 + a], lo[a]);
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double c[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            // (f64(min) + max) * 0.5 -- tree.py:191-192
            c[a] = __dmul_rn(__dadd_rn((double)__ldg(mins + 3 * i + a),
                                       (double)__ldg(maxs + 3 * i + a)),
                             0.5);
        }
        CodeT code;
        encode(c[0], c[1], c[2], lo, ext, code);
        codes[i] = code;
        if (iota) iota[i] = (uint32_t)i;
        if (sizeof(CodeT) == 4 && hist) hist_accumulate(s_hist, (uint32_t)code, 0, 4);
    }
    if (hist) {
        __syncthreads();
        hist_flush(s_hist, 4, hist);
    }
}

// Common-prefix length of augmented keys i, i+1 (code << 32 | position),
// _kernels.py:50-58.  Keys are distinct, so the xor is never 0.
__device__ __forceinline__ int delta(const uint32_t *__restrict__ codes, int64_t i) {
    uint32_t a = __ldg(codes + i), b = __ldg(codes + i + 1);
    if (a != b) return __clz(a ^ b);
    return 32 + __clz((uint32_t)i ^ (uint32_t)(i + 1));
}

// 63-bit codes: keys (code, position) compare on 64 code bits first.
__device__ __forceinline__ int delta(const uint64_t *__restrict__ codes, int64_t i) {
    uint64_t a = __ldg(codes + i), b = __ldg(codes + i + 1);
    if (a != b) return __clzll(a ^ b);
    return 64 + __clz((uint32_t)i ^ (uint32_t)(i + 1));
}

// Is [l, r] the left child of its parent?  Boundary prefixes are never equal.
template <typename CodeT>
__device__ __forceinline__ bool is_left_child(const CodeT *__restrict__ codes, int64_t n,
                                              int64_t l, int64_t r) {
    if (l == 0) return true;
    if (r == n - 1) return false;
    return delta(codes, r) > delta(codes, l - 1);
}

__device__ __forceinline__ void load_box_cg(const float *mins, const float *maxs, int64_t id,
                                            Box &b) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        b.lo[a] = __ldcg(mins + 3 * id + a);
        b.hi[a] = __ldcg(maxs + 3 * id + a);
    }
}

__device__ __forceinline__ void store_box(float *mins, float *maxs, int64_t id, const Box &b) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        mins[3 * id + a] = b.lo[a];
        maxs[3 * id + a] = b.hi[a];
    }
}

__device__ __forceinline__ void store_packed(PackedNode *nodes, int64_t id, const Box &L,
                                             const Box &R, int32_t lc, int32_t rc) {
    PackedNode *p = nodes + id;
    float4 a, b, c;
    pack_boxes(L, R, a, b, c);
    // two 32-byte stores: full L2 sectors (four 16-byte stores: build +0.06 ms)
    stg256(&p->a, a, b);
    stg256(&p->c, c, make_float4(__int_as_float(lc), __int_as_float(rc), 0.0f, 0.0f));
}

// leaf_codes (optional): the 30-bit code of every leaf in leaf order (for
// 63-bit codes the top 30 bits, which are exactly the 30-bit code).
__device__ __forceinline__ uint32_t code30(uint32_t c) { return c; }
__device__ __forceinline__ uint32_t code30(uint64_t c) { return (uint32_t)(c >> 33); }

// Split prefix of adjacent keys (a, i), (b, i+1): delta() on staged codes.
__device__ __forceinline__ int delta_of(uint32_t a, uint32_t b, int64_t i) {
    if (a != b) return __clz(a ^ b);
    return 32 + __clz((uint32_t)i ^ (uint32_t)(i + 1));
}
__device__ __forceinline__ int delta_of(uint64_t a, uint64_t b, int64_t i) {
    if (a != b) return __clzll(a ^ b);
    return 64 + __clz((uint32_t)i ^ (uint32_t)(i + 1));
}

// Topology only (lbvh_generate_topology, generate_topology tree.py:85-105):
// the bottom-up construction of the build without boxes -- sorted codes in,
// Karras left/right/parent out.  The handshake carries no data besides the
// exchanged range end, so a release-only exchange suffices.
__global__ void __launch_bounds__(256)
topology_kernel(const uint32_t *__restrict__ codes, int64_t n, uint32_t *slots,
                int32_t *__restrict__ left, int32_t *__restrict__ right,
                int32_t *__restrict__ parent) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    if (n == 1) {
        parent[0] = -1;
        return;
    }
    const int64_t internal = n - 1;
    int64_t l = p, r = p;
    bool left_side = is_left_child(codes, n, l, r);
    while (true) {
        const int64_t g = left_side ? r : l - 1;
        const uint32_t known = (uint32_t)(left_side ? l : r);
        const uint32_t other = atomic_exch_release(slots + g, known + 1u);
        if (other == 0) return;  // first arrival: sibling subtree not done
        const int64_t pl = left_side ? l : (int64_t)(other - 1u);
        const int64_t pr = left_side ? (int64_t)(other - 1u) : r;
        const int64_t lc = (pl == g) ? internal + g : g;
        const int64_t rc = (g + 1 == pr) ? internal + g + 1 : g + 1;
        const bool root = (pl == 0 && pr == n - 1);
        const bool parent_left = root ? false : is_left_child(codes, n, pl, pr);
        const int64_t pid = root ? 0 : (parent_left ? pr : pl);
        left[pid] = (int32_t)lc;
        right[pid] = (int32_t)rc;
        parent[lc] = (int32_t)pid;
        parent[rc] = (int32_t)pid;
        if (root) {
            parent[0] = -1;
            return;
        }
        l = pl;
        r = pr;
        left_side = parent_left;
    }
}

// ---------------------------------------------------------------------------
// Hierarchy (K4+K5): Apetrei's bottom-up construction emitting Karras
// ordinals, in two levels split by where the two children of a node meet.
//
// hierarchy_local_kernel: CTA c owns leaves [B, E].  A thread climbs while the
// split slot g of its node satisfies B <= g < E, i.e. both children of the
// parent start or end inside the CTA; the handshake is then a shared-memory
// exchange and the sibling's box and link come from shared memory -- no
// global atomics, no fences.  A node whose slot leaves the CTA is appended to
// the frontier list; a first arrival whose partner never came (the sibling
// subtree crosses the CTA edge) is copied to the global slot array at the end.
// The CTA's codes are staged once in shared memory (coalesced) and the split
// prefixes delta(i), i in [B-1, E], computed from them, so the climb and the
// leaf directory read no global codes.
//
// hierarchy_frontier_kernel: the frontier nodes continue with a global
// handshake (release exchange; the second arrival fences acq_rel before it
// reads the sibling's record).  A local-kernel first arrival is then
// indistinguishable from a global one, so the meeting rule is unchanged.
// It also writes the leaf-directory runs the local kernel deferred.
// ---------------------------------------------------------------------------
#ifndef LBVH_HIER_T
#define LBVH_HIER_T 256
#endif
constexpr int kHierT = LBVH_HIER_T;
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
    __shared__ uint32_t s_slot[kHierT];
    __shared__ float s_box[2][6][kHierT];
    __shared__ int32_t s_link[2][kHierT];
    __shared__ CodeT s_code[kHierT + 2];     // codes[B - 1 + i]
    __shared__ uint8_t s_delta[kHierT + 1];  // delta(B - 1 + i)
    __shared__ int32_t s_pid[kHierT];        // node completed at slot B + i (-1: none)
    const int tid = threadIdx.x;
    // 32-bit indices throughout (trees hold < 2^30 leaves): the climb's
    // range and node arithmetic stays single-instruction
    const int32_t nn = (int32_t)n;
    const int32_t B = (int32_t)blockIdx.x * kHierT;
    const int32_t E = (B + kHierT < nn ? B + kHierT : nn) - 1;
    const int32_t p = B + tid;
    const int32_t internal = nn - 1;
    s_slot[tid] = 0;
    s_pid[tid] = -1;
    // leaf p's box, gathered through the sorted permutation: issued first so
    // its two dependent loads overlap the code loads and barriers below
    bool active = p < nn;
    Box mine;
    uint32_t gobj = 0;
    if (active) {
        const uint32_t obj = __ldg(perm + p);
        // the ordinal this leaf reports: its input index, or leaf_ids[index]
        gobj = leaf_ids ? (uint32_t)__ldg(leaf_ids + obj) : obj;
        const bool same = (mins == maxs);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            mine.lo[a] = __ldg(mins + 3 * (int64_t)obj + a);
            mine.hi[a] = same ? mine.lo[a] : __ldg(maxs + 3 * (int64_t)obj + a);
        }
    }
    for (int i = tid; i < kHierT + 2; i += kHierT) {
        const int32_t j = B - 1 + i;
        if (j >= 0 && j < nn) s_code[i] = __ldg(codes + j);
    }
    __syncthreads();
    if (p < nn - 1) s_delta[tid + 1] = (uint8_t)delta_of(s_code[tid + 1], s_code[tid + 2], p);
    if (tid == 0 && B > 0) s_delta[0] = (uint8_t)delta_of(s_code[0], s_code[1], B - 1);
    __syncthreads();
    // is_left_child over the CTA's range: l >= B and r <= E, so both prefixes
    // delta(r) and delta(l - 1) are in s_delta
    auto left_child = [&](int32_t l, int32_t r) -> bool {
        if (l == 0) return true;
        if (r == nn - 1) return false;
        return s_delta[r - B + 1] > s_delta[l - B];
    };
    int32_t my_link = 0;
    int32_t l = p, r = p;
    if (active) {
        const uint32_t c30 = code30(s_code[tid + 1]);
        if (leaf_codes) leaf_codes[p] = c30;
        if (leaf_dir) {
            // dir[b] = first leaf whose code >> (30 - bits) >= b: leaf p owns
            // the buckets after its predecessor's, the last leaf the tail = n
            const int sh = 30 - dir_bits;
            const int64_t cb = (int64_t)(c30 >> sh);
            const int64_t pb = p == 0 ? -1 : (int64_t)(code30(s_code[tid]) >> sh);
            dir_run(leaf_dir, pb + 1, cb + 1, (uint32_t)p, runs, run_count);
            if (p == nn - 1)
                dir_run(leaf_dir, cb + 1, ((int64_t)1 << dir_bits) + 1, (uint32_t)n, runs,
                        run_count);
        }
        leaf_obj[p] = (int32_t)gobj;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            node_mins[3 * (int64_t)(internal + p) + a] = mine.lo[a];
            if (leaf_maxs_rows) node_maxs[3 * (int64_t)(internal + p) + a] = mine.hi[a];
        }
        my_link = (int32_t)(gobj | kLeafTag);
        if (nn == 1) {  // leaf-only tree (tree.py:177-209 with n == 1)
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                root_box[a] = mine.lo[a];
                root_box[3 + a] = mine.hi[a];
            }
            active = false;
        }
    }
    // side of the current node; the parent's side is computed with the
    // parent and carried into the next step (one prefix test per level)
    bool left_side = active && left_child(l, r);
    while (active) {
        const int32_t g = left_side ? r : l - 1;
        if (g < B || g >= E) {  // the parent's other child may lie outside the CTA
            const uint32_t at = atomicAdd(frontier_count, 1u);
            frontier[at] = make_uint2((uint32_t)l, (uint32_t)r);
            break;
        }
        const int s = g - B;
        const int side = left_side ? 0 : 1;
        // hand-off slots are accessed only through shared-memory atomics (the
        // fence + exchange below orders them; atomics also keep racecheck exact)
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            atomicExch(reinterpret_cast<unsigned *>(&s_box[side][a][s]), __float_as_uint(mine.lo[a]));
            atomicExch(reinterpret_cast<unsigned *>(&s_box[side][3 + a][s]),
                       __float_as_uint(mine.hi[a]));
        }
        atomicExch(reinterpret_cast<unsigned *>(&s_link[side][s]), (unsigned)my_link);
        __threadfence_block();
        const uint32_t known = (uint32_t)(left_side ? l : r);
        const uint32_t other = atomicExch(&s_slot[s], known + 1u);
        if (other == 0) break;  // first arrival: the sibling continues
        __threadfence_block();
        const int32_t pl = left_side ? l : (int32_t)(other - 1u);
        const int32_t pr = left_side ? (int32_t)(other - 1u) : r;
        const bool root = (pl == 0 && pr == nn - 1);
        const bool parent_left = !root && left_child(pl, pr);
        const int32_t pid = root ? 0 : (parent_left ? pr : pl);
        Box sb;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            sb.lo[a] = __uint_as_float(atomicOr(reinterpret_cast<unsigned *>(&s_box[1 - side][a][s]), 0u));
            sb.hi[a] = __uint_as_float(
                atomicOr(reinterpret_cast<unsigned *>(&s_box[1 - side][3 + a][s]), 0u));
        }
        const Box &L = left_side ? mine : sb;
        const Box &R = left_side ? sb : mine;
        Box P;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            P.lo[a] = min_left(L.lo[a], R.lo[a]);
            P.hi[a] = max_left(L.hi[a], R.hi[a]);
        }
        s_pid[s] = pid;  // its record is s_box / s_link at slot s: written below
        mine = P;
        my_link = (int32_t)pid;
        if (root) {
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                root_box[a] = P.lo[a];
                root_box[3 + a] = P.hi[a];
            }
            break;
        }
        l = pl;
        r = pr;
        left_side = parent_left;
    }
    // Every node completed in this CTA: its record (both child boxes and links
    // as exchanged at its slot g) and its reference left/right entries (a leaf
    // child of slot g is leaf g or g + 1), written by all threads at once --
    // full 32-byte sectors, converged stores.  Round 1 wrote them during the
    // climb, at ~10 active lanes (build 1.19 -> 1.10 ms at 1e7).  A slot with
    // a single arrival keeps its range end in s_slot.
    __syncthreads();
    const int32_t id = s_pid[tid];
    // this CTA's window of the global hand-off slots: a first arrival whose
    // partner never came publishes its range end for the frontier kernel
    // (the partner's subtree crosses the CTA edge); every other slot is 0
    if (p < nn - 1) slots[p] = id >= 0 ? 0u : s_slot[tid];
    if (id >= 0) {
        Box L, R;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            L.lo[a] = s_box[0][a][tid]; L.hi[a] = s_box[0][3 + a][tid];
            R.lo[a] = s_box[1][a][tid]; R.hi[a] = s_box[1][3 + a][tid];
        }
        const int32_t ll = s_link[0][tid], rl = s_link[1][tid];
        store_packed(nodes, id, L, R, ll, rl);
        left[id] = ll < 0 ? internal + p : ll;
        right[id] = rl < 0 ? internal + p + 1 : rl;
    }
}

// Memory-scope helpers of the frontier handshake: GPU scope when climbers
// run in many CTAs, CTA scope for the single-CTA top stage (no L2 round
// trips for fences, records read through L1).
template <bool CTA>
__device__ __forceinline__ uint32_t exch_release(uint32_t *p, uint32_t v) {
    uint32_t old;
    if (CTA)
        asm volatile("atom.release.cta.global.exch.b32 %0, [%1], %2;"
                     : "=r"(old) : "l"(p), "r"(v) : "memory");
    else
        asm volatile("atom.release.gpu.global.exch.b32 %0, [%1], %2;"
                     : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
template <bool CTA>
__device__ __forceinline__ void fence_acq_rel() {
    if (CTA)
        asm volatile("fence.acq_rel.cta;" ::: "memory");
    else
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
template <bool CTA>
__device__ __forceinline__ float ld_rlx(const float *p) {
    float v;
    if (CTA)
        asm volatile("ld.relaxed.cta.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}
template <bool CTA>
__device__ __forceinline__ float4 ld_rlx(const float4 *p) {
    float4 v;
    if (CTA)
        asm volatile("ld.relaxed.cta.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
    return v;
}

// Box of a node the local kernel (or an earlier frontier step) finished:
// a leaf's row, or the union of an internal node's packed child boxes
// (same left-first fold as the refit).  Strong loads: written by other threads.
template <bool CTA>
__device__ __forceinline__ void frontier_box(const PackedNode *nodes, const float *node_mins,
                                             const float *node_maxs, bool leaf_maxs_rows,
                                             int64_t internal, int64_t id, Box &b) {
    if (id < internal) {
        const PackedNode *pn = nodes + id;
        Box L, R;
        unpack_boxes(ld_rlx<CTA>(&pn->a), ld_rlx<CTA>(&pn->b), ld_rlx<CTA>(&pn->c), L, R);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            b.lo[k] = min_left(L.lo[k], R.lo[k]);
            b.hi[k] = max_left(L.hi[k], R.hi[k]);
        }
    } else {
        const float *hi = leaf_maxs_rows ? node_maxs : node_mins;  // point leaves: hi == lo
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            b.lo[a] = ld_rlx<CTA>(node_mins + 3 * id + a);
            b.hi[a] = ld_rlx<CTA>(hi + 3 * id + a);
        }
    }
}

// The frontier climb.  Stage 1 (CTA = false, many CTAs, GPU-scope
// handshakes) climbs until a node spans >= stop_len leaves and defers it to
// stage 2; stage 2 (CTA = true, one CTA, CTA-scope handshakes) finishes the
// top levels -- few nodes, but a chain of dependent handshakes whose GPU-scope
// fences would cost L2 round trips each.  Small trees go to stage 2 directly.
constexpr int kTopThreads = 1024;
#ifndef LBVH_TOP_SPAN_BITS
#define LBVH_TOP_SPAN_BITS 16
#endif
constexpr int64_t kTopSpan = (int64_t)1 << LBVH_TOP_SPAN_BITS;  // stage 1 defers nodes spanning >= this

template <typename CodeT, bool CTA>
__global__ void __launch_bounds__(CTA ? kTopThreads : 256)
hierarchy_frontier_kernel(const CodeT *__restrict__ codes, const int32_t *__restrict__ leaf_obj,
                          int64_t n, uint32_t *slots, const float *node_mins,
                          const float *node_maxs, bool leaf_maxs_rows,
                          int32_t *__restrict__ left, int32_t *__restrict__ right,
                          PackedNode *nodes, float *__restrict__ root_box,
                          const uint2 *__restrict__ frontier, const uint32_t *frontier_count,
                          uint32_t *__restrict__ leaf_dir, const DirRun *__restrict__ runs,
                          const uint32_t *run_count, int64_t stop_len, uint2 *deferred,
                          uint32_t *deferred_count) {
    const int64_t internal = n - 1;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    if (leaf_dir) {  // long leaf-directory runs (> kDirInline buckets): one warp per run
        const uint32_t nr = *run_count;
        const int64_t lane = threadIdx.x & 31;
        for (int64_t k = tid >> 5; k < (int64_t)nr; k += stride >> 5) {
            const DirRun e = runs[k];
            for (int64_t b = e.lo + lane; b < (int64_t)e.hi; b += 32) leaf_dir[b] = e.value;
        }
    }
    const int64_t count = (int64_t)*frontier_count;
    for (int64_t i = tid; i < count; i += stride) {
        const uint2 e = frontier[i];
        int64_t l = e.x, r = e.y;
        Box mine;
        int32_t my_link;
        if (l == r) {  // a leaf (row written by the local kernel)
            frontier_box<CTA>(nodes, node_mins, node_maxs, leaf_maxs_rows, internal,
                              internal + l, mine);
            my_link = (int32_t)((uint32_t)__ldg(leaf_obj + l) | kLeafTag);
        } else {       // an internal node built by the local kernel or stage 1
            const int64_t id = is_left_child(codes, n, l, r) ? r : l;
            frontier_box<CTA>(nodes, node_mins, node_maxs, leaf_maxs_rows, internal, id, mine);
            my_link = (int32_t)id;
        }
        bool left_side = is_left_child(codes, n, l, r);
        while (true) {
            if (!CTA && r - l + 1 >= stop_len) {  // the top levels: stage 2
                deferred[atomicAdd(deferred_count, 1u)] = make_uint2((uint32_t)l, (uint32_t)r);
                break;
            }
            const int64_t g = left_side ? r : l - 1;
            const uint32_t known = (uint32_t)(left_side ? l : r);
            // release: this subtree's record is visible to whoever arrives second
            const uint32_t other = exch_release<CTA>(slots + g, known + 1u);
            if (other == 0) break;  // first arrival: sibling subtree not done
            // second arrival: the exchange read the partner's release; the
            // fence completes the acquire pattern before its record is read
            fence_acq_rel<CTA>();
            const int64_t pl = left_side ? l : (int64_t)(other - 1u);
            const int64_t pr = left_side ? (int64_t)(other - 1u) : r;
            const int64_t lc = (pl == g) ? internal + g : g;
            const int64_t rc = (g + 1 == pr) ? internal + g + 1 : g + 1;
            const bool root = (pl == 0 && pr == n - 1);
            const bool parent_left = root ? false : is_left_child(codes, n, pl, pr);
            const int64_t pid = root ? 0 : (parent_left ? pr : pl);
            left[pid] = (int32_t)lc;
            right[pid] = (int32_t)rc;
            const int64_t sib = left_side ? rc : lc;
            Box sb;
            frontier_box<CTA>(nodes, node_mins, node_maxs, leaf_maxs_rows, internal, sib, sb);
            const int32_t sib_link = sib < internal
                                         ? (int32_t)sib
                                         : (int32_t)((uint32_t)__ldg(leaf_obj + (sib - internal)) |
                                                     kLeafTag);
            const Box &L = left_side ? mine : sb;
            const Box &R = left_side ? sb : mine;
            Box P;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                P.lo[a] = min_left(L.lo[a], R.lo[a]);
                P.hi[a] = max_left(L.hi[a], R.hi[a]);
            }
            store_packed(nodes, pid, L, R, left_side ? my_link : sib_link,
                         left_side ? sib_link : my_link);
            mine = P;
            my_link = (int32_t)pid;
            if (root) {
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    root_box[a] = P.lo[a];
                    root_box[3 + a] = P.hi[a];
                }
                break;
            }
            l = pl;
            r = pr;
            left_side = parent_left;
        }
    }
}

// Reference-layout rows the build defers (LBVH_BUILD_DEFER_ROWS): internal
// row i = union of the two child boxes in packed record i, folded with the
// refit's left-first rule (identical bits to an in-pass write), and for
// point leaves the node_maxs leaf rows (== node_mins rows).  Coalesced.
__global__ void __launch_bounds__(256)
finish_rows_kernel(const PackedNode *__restrict__ nodes, int64_t n, bool copy_leaf_maxs,
                   float *__restrict__ node_mins, float *__restrict__ node_maxs) {
    const int64_t n_internal = n - 1;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_internal; i += stride) {
        const PackedNode *p = nodes + i;
        Box L, R;
        unpack_boxes(__ldcs(&p->a), __ldcs(&p->b), __ldcs(&p->c), L, R);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            node_mins[3 * i + k] = min_left(L.lo[k], R.lo[k]);
            node_maxs[3 * i + k] = max_left(L.hi[k], R.hi[k]);
        }
    }
    if (copy_leaf_maxs)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * n; i += stride)
            node_maxs[3 * n_internal + i] = __ldcs(node_mins + 3 * n_internal + i);
}

// Atomic-flag refit over an arbitrary (left, right, parent) topology --
// refit_bounds (tree.py:108-119): leaf boxes in place, internal boxes filled.
__global__ void __launch_bounds__(256)
refit_kernel(float *node_mins, float *node_maxs, const int32_t *__restrict__ left,
             const int32_t *__restrict__ right, const int32_t *__restrict__ parent, int64_t n,
             uint32_t *visits) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    int64_t node = (n - 1) + p;
    while (true) {
        const int64_t par = __ldg(parent + node);
        if (par < 0) return;
        if (atomic_add_acq_rel(visits + par, 1u) == 0) return;
        const int64_t lc = __ldg(left + par), rc = __ldg(right + par);
        Box L, R, P;
        load_box_cg(node_mins, node_maxs, lc, L);
        load_box_cg(node_mins, node_maxs, rc, R);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            P.lo[a] = min_left(L.lo[a], R.lo[a]);
            P.hi[a] = max_left(L.hi[a], R.hi[a]);
        }
        store_box(node_mins, node_maxs, par, P);
        node = par;
    }
}

__device__ __forceinline__ bool load_child(const lbvh_tree t, int64_t c, Box &b,
                                           int32_t &link) {
    const int64_t internal = t.n - 1;
    if (c < 0 || c >= 2 * t.n - 1) return false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        b.lo[a] = __ldg(t.node_mins + 3 * c + a);
        b.hi[a] = __ldg(t.node_maxs + 3 * c + a);
    }
    if (c >= internal) {
        int32_t obj = __ldg(t.leaf_obj + (c - internal));
        if (obj < 0) return false;
        link = (int32_t)((uint32_t)obj | kLeafTag);
    } else {
        link = (int32_t)c;
    }
    return true;
}

// Reference layout -> traversal layout (user-built or modified trees).
__global__ void __launch_bounds__(256)
pack_kernel(const lbvh_tree t, PackedNode *__restrict__ nodes, float *__restrict__ root_box,
            uint32_t *status) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            root_box[a] = __ldg(t.node_mins + a);
            root_box[3 + a] = __ldg(t.node_maxs + a);
        }
    }
    if (i >= t.n - 1) return;
    Box L, R;
    int32_t ll = 0, rl = 0;
    bool ok = load_child(t, __ldg(t.left + i), L, ll);
    ok = load_child(t, __ldg(t.right + i), R, rl) && ok;
    if (!ok) {
        flag(status, LBVH_FLAG_BAD_TREE);
        L = Box{{0, 0, 0}, {0, 0, 0}};
        R = L;
        ll = rl = (int32_t)kLeafTag;
    }
    store_packed(nodes, i, L, R, ll, rl);
}

__global__ void __launch_bounds__(256)
unpack_kernel(const lbvh_tree t, float *__restrict__ node_mins, float *__restrict__ node_maxs) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            node_mins[a] = t.root_box[a];
            node_maxs[a] = t.root_box[3 + a];
        }
    }
    if (i >= t.n - 1) return;
    const PackedNode *pn = reinterpret_cast<const PackedNode *>(t.nodes) + i;
    Box L, R;
    unpack_boxes(pn->a, pn->b, pn->c, L, R);
    int64_t lc = t.left[i], rc = t.right[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        node_mins[3 * lc + k] = L.lo[k]; node_maxs[3 * lc + k] = L.hi[k];
        node_mins[3 * rc + k] = R.lo[k]; node_maxs[3 * rc + k] = R.hi[k];
    }
}

__global__ void morton_f64_kernel(const double *__restrict__ pts, int64_t n, double lo0,
                                  double lo1, double lo2, double hi0, double hi1, double hi2,
                                  uint32_t *__restrict__ codes) {
    double lo[3] = {lo0, lo1, lo2};
    double ext[3] = {__dsub_rn(hi0, lo0), __dsub_rn(hi1, lo1), __dsub_rn(hi2, lo2)};
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        codes[i] = morton3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], lo, ext);
}

unsigned grid_for(int64_t n, int threads, int per_sm = 8) {
    unsigned g = div_up(n, threads);
    unsigned cap = kNumSMs * per_sm;
    return g < cap ? (g ? g : 1) : cap;
}

}  // namespace

// ----------------------------------------------------------------- host API

constexpr int kDirBitsMax = 24;
constexpr size_t kDirRunsMax = (((size_t)1 << kDirBitsMax) + 1) / (kDirInline + 1) + 2;

size_t build_workspace_bytes(int64_t n) {
    // sized for the wider (63-bit) pipeline so one size serves both
    size_t b = 0;
    b += align_up(sizeof(uint64_t) * (size_t)n) + align_up(sizeof(uint32_t) * (size_t)n);
    b += align_up(sizeof(uint32_t) * (size_t)(n > 1 ? n - 1 : 1));  // handshake slots
    b += align_up(sizeof(uint32_t) * 4);                         // counters
    b += align_up(sizeof(float) * 6 * kNumSMs * 8);              // reduce partials
    b += align_up(sizeof(DirRun) * kDirRunsMax);                 // long directory runs
    size_t s32 = sort_workspace_bytes(n), s64 = sort64_workspace_bytes(n);
    b += s32 > s64 ? s32 : s64;
    return b + 1024;
}

namespace {
int sort_codes(uint32_t *codes, uint32_t *perm, int64_t n, void *ws, cudaStream_t st) {
    return sort_pairs(codes, perm, n, 30, ws, sort_workspace_bytes(n), st);
}
int sort_codes(uint64_t *codes, uint32_t *perm, int64_t n, void *ws, cudaStream_t st) {
    return sort_pairs64(codes, perm, n, 63, ws, sort64_workspace_bytes(n), st);
}

template <typename CodeT>
int build_impl(const float *mins, const float *maxs, int64_t n, void *ws, size_t ws_bytes,
               float *node_mins, float *node_maxs, int32_t *left, int32_t *right,
               int32_t *leaf_obj, float *root_box, void *nodes, uint32_t *sorted_codes,
               uint32_t *leaf_dir, int dir_bits, int flags, const int32_t *leaf_ids,
               uint32_t *status, cudaStream_t stream) {
    Carve c(ws, ws_bytes);
    CodeT *codes = c.take<CodeT>(n);
    uint32_t *perm = c.take<uint32_t>(n);
    uint32_t *slots = c.take<uint32_t>(n > 1 ? n - 1 : 1);  // zeroed by the local kernel
    uint32_t *counter = c.take<uint32_t>(4);  // reduce CTAs, -, frontier, directory runs
    float *partials = c.take<float>(6 * kNumSMs * 8);
    DirRun *runs = c.take<DirRun>(kDirRunsMax);
    void *sort_ws = c.take<char>(sizeof(CodeT) == 4 ? sort_workspace_bytes(n)
                                                    : sort64_workspace_bytes(n));
    if (!c.ok()) return LBVH_ERR_WORKSPACE;
    cudaMemsetAsync(counter, 0, 4 * sizeof(uint32_t), stream);

    unsigned rg = grid_for(n, kReduceThreads, 4);
    scene_reduce_kernel<<<rg, kReduceThreads, 0, stream>>>(mins, maxs, n, partials, counter,
                                                           root_box, status);
    int rc;
    if (sizeof(CodeT) == 4) {
        // the sort's digit histograms come from the Morton pass, its input
        // values are the positions: no histogram pass, no iota array
        uint32_t *hist = sort_prepare(sort_ws, sort_workspace_bytes(n), n, stream);
        morton_kernel<CodeT><<<grid_for(n, 256, LBVH_MORTON_CTAS), 256, 0, stream>>>(
            mins, maxs, n, root_box, codes, nullptr, hist);
        count_launches(2);
        rc = sort_pairs_prepared(reinterpret_cast<uint32_t *>(codes), perm, n, 30, sort_ws,
                                 sort_workspace_bytes(n), stream, 0, false);
    } else {
        morton_kernel<CodeT><<<grid_for(n, 256, 16), 256, 0, stream>>>(mins, maxs, n, root_box,
                                                                       codes, perm);
        count_launches(2);
        rc = sort_codes(codes, perm, n, sort_ws, stream);
    }
    if (rc != LBVH_OK) return rc;
    // point input with deferred rows: node_maxs leaf rows (== node_mins rows)
    // are written by lbvh_finish_rows, the frontier reads node_mins for both
    const bool defer = (flags & LBVH_BUILD_DEFER_ROWS) != 0;
    const bool leaf_maxs_rows = !(defer && mins == maxs);
    // the sort's ping-pong buffers are dead now: the frontier list lives there
    uint2 *frontier = reinterpret_cast<uint2 *>(sort_ws);
    hierarchy_local_kernel<CodeT><<<div_up(n, kHierT), kHierT, 0, stream>>>(
        codes, perm, mins, maxs, n, slots, node_mins, node_maxs, leaf_maxs_rows, left, right,
        leaf_obj, (PackedNode *)nodes, root_box, sorted_codes, leaf_dir, dir_bits, runs,
        counter + 3, frontier, counter + 2, leaf_ids);
    // stage 1 only when the frontier is too large for one CTA; its deferred
    // list lives after the frontier list (at most 2n / kTopSpan + 2 entries)
    uint2 *deferred = frontier + n;
    if (n > 4 * kTopSpan) {
        hierarchy_frontier_kernel<CodeT, false><<<grid_for(n / 64 + 1, 256, 8), 256, 0, stream>>>(
            codes, leaf_obj, n, slots, node_mins, node_maxs, leaf_maxs_rows, left, right,
            (PackedNode *)nodes, root_box, frontier, counter + 2, leaf_dir, runs, counter + 3,
            kTopSpan, deferred, counter + 1);
        hierarchy_frontier_kernel<CodeT, true><<<1, kTopThreads, 0, stream>>>(
            codes, leaf_obj, n, slots, node_mins, node_maxs, leaf_maxs_rows, left, right,
            (PackedNode *)nodes, root_box, deferred, counter + 1, nullptr, runs, counter + 3,
            0, nullptr, nullptr);
        count_launches(1);
    } else {
        hierarchy_frontier_kernel<CodeT, true><<<1, kTopThreads, 0, stream>>>(
            codes, leaf_obj, n, slots, node_mins, node_maxs, leaf_maxs_rows, left, right,
            (PackedNode *)nodes, root_box, frontier, counter + 2, leaf_dir, runs, counter + 3,
            0, nullptr, nullptr);
    }
    count_launches(2);
    if (!defer && n > 1) {
        finish_rows_kernel<<<grid_for(n - 1, 256, 16), 256, 0, stream>>>(
            (const PackedNode *)nodes, n, false, node_mins, node_maxs);
        count_launches(1);
    }
    return check_launch();
}
}  // namespace

int build(const float *mins, const float *maxs, int64_t n, int morton_bits, void *ws,
          size_t ws_bytes, float *node_mins, float *node_maxs, int32_t *left, int32_t *right,
          int32_t *leaf_obj, float *root_box, void *nodes, uint32_t *sorted_codes,
          uint32_t *leaf_dir, int leaf_dir_bits, int flags, const int32_t *leaf_ids,
          uint32_t *status, cudaStream_t stream) {
    if (n == 0) return LBVH_ERR_EMPTY_SCENE;
    if (n < 0 || !mins || !maxs || !node_mins || !node_maxs || !leaf_obj || !root_box ||
        !status || (morton_bits != 30 && morton_bits != 63))
        return LBVH_ERR_INVALID_ARG;
    if (n > 1 && (!left || !right || !nodes)) return LBVH_ERR_INVALID_ARG;
    if (leaf_dir && (leaf_dir_bits < 0 || leaf_dir_bits > kDirBitsMax))
        return LBVH_ERR_INVALID_ARG;
    if (n >= LBVH_MAX_ITEMS) return LBVH_ERR_TOO_LARGE;
    if (ws_bytes < build_workspace_bytes(n)) return LBVH_ERR_WORKSPACE;
    if (morton_bits == 63)
        return build_impl<uint64_t>(mins, maxs, n, ws, ws_bytes, node_mins, node_maxs, left,
                                    right, leaf_obj, root_box, nodes, sorted_codes, leaf_dir,
                                    leaf_dir_bits, flags, leaf_ids, status, stream);
    return build_impl<uint32_t>(mins, maxs, n, ws, ws_bytes, node_mins, node_maxs, left, right,
                                leaf_obj, root_box, nodes, sorted_codes, leaf_dir,
                                leaf_dir_bits, flags, leaf_ids, status, stream);
}

int finish_rows(const lbvh_tree *t, float *node_mins, float *node_maxs, cudaStream_t stream) {
    if (!t || t->n < 1 || !node_mins || !node_maxs) return LBVH_ERR_INVALID_ARG;
    if (t->n > 1 && !t->nodes) return LBVH_ERR_INVALID_ARG;
    const bool leaves = (t->flags & LBVH_TREE_POINT_LEAVES) != 0;
    if (t->n == 1 && !leaves) return LBVH_OK;
    finish_rows_kernel<<<grid_for(3 * t->n, 256, 16), 256, 0, stream>>>(
        (const PackedNode *)t->nodes, t->n, leaves, node_mins, node_maxs);
    count_launches(1);
    return check_launch();
}

size_t topology_workspace_bytes(int64_t n) {
    return align_up(sizeof(uint32_t) * (size_t)(n > 1 ? n : 1)) + 256;
}

int generate_topology(const uint32_t *codes, int64_t n, int32_t *left, int32_t *right,
                      int32_t *parent, void *ws, size_t ws_bytes, cudaStream_t stream) {
    if (n == 0) return LBVH_ERR_EMPTY_SCENE;
    if (n < 0 || !codes || !parent || (n > 1 && (!left || !right))) return LBVH_ERR_INVALID_ARG;
    if (n >= LBVH_MAX_ITEMS) return LBVH_ERR_TOO_LARGE;
    if (ws_bytes < topology_workspace_bytes(n)) return LBVH_ERR_WORKSPACE;
    uint32_t *slots = (uint32_t *)ws;
    cudaMemsetAsync(slots, 0, sizeof(uint32_t) * (size_t)(n > 1 ? n - 1 : 1), stream);
    topology_kernel<<<div_up(n, 256), 256, 0, stream>>>(codes, n, slots, left, right, parent);
    count_launches(1);
    return check_launch();
}

int refit(float *node_mins, float *node_maxs, const int32_t *left, const int32_t *right,
          const int32_t *parent, int64_t n, void *ws, size_t ws_bytes, cudaStream_t stream) {
    if (n < 0 || !node_mins || !node_maxs) return LBVH_ERR_INVALID_ARG;
    if (n <= 1) return LBVH_OK;
    if (!left || !right || !parent) return LBVH_ERR_INVALID_ARG;
    if (ws_bytes < topology_workspace_bytes(n)) return LBVH_ERR_WORKSPACE;
    uint32_t *visits = (uint32_t *)ws;
    cudaMemsetAsync(visits, 0, sizeof(uint32_t) * (size_t)(n - 1), stream);
    refit_kernel<<<div_up(n, 256), 256, 0, stream>>>(node_mins, node_maxs, left, right,
                                                      parent, n, visits); count_launches(1);
    return check_launch();
}

int pack(const lbvh_tree *t, void *nodes, float *root_box, uint32_t *status,
         cudaStream_t stream) {
    if (!t || t->n < 1 || !t->node_mins || !t->node_maxs || !t->leaf_obj || !root_box)
        return LBVH_ERR_INVALID_ARG;
    if (t->n > 1 && (!t->left || !t->right || !nodes)) return LBVH_ERR_INVALID_ARG;
    int64_t work = t->n > 1 ? t->n - 1 : 1;
    pack_kernel<<<div_up(work, 256), 256, 0, stream>>>(*t, (PackedNode *)nodes, root_box,
                                                       status); count_launches(1);
    return check_launch();
}

int unpack_boxes(const lbvh_tree *t, float *node_mins, float *node_maxs, cudaStream_t stream) {
    if (!t || t->n < 1 || !t->root_box || !node_mins || !node_maxs) return LBVH_ERR_INVALID_ARG;
    if (t->n > 1 && (!t->left || !t->right || !t->nodes)) return LBVH_ERR_INVALID_ARG;
    int64_t work = t->n > 1 ? t->n - 1 : 1;
    unpack_kernel<<<div_up(work, 256), 256, 0, stream>>>(*t, node_mins, node_maxs); count_launches(1);
    return check_launch();
}

int morton_codes_f64(const double *pts, int64_t n, const double *lo, const double *hi,
                     uint32_t *codes, cudaStream_t stream) {
    if (n < 0 || (n > 0 && (!pts || !codes)) || !lo || !hi) return LBVH_ERR_INVALID_ARG;
    if (n == 0) return LBVH_OK;
    morton_f64_kernel<<<grid_for(n, 256, 16), 256, 0, stream>>>(pts, n, lo[0], lo[1], lo[2],
                                                               hi[0], hi[1], hi[2], codes); count_launches(1);
    return check_launch();
}

// Query Morton codes on the tree's scene box + stable sort -> order.
size_t query_workspace_bytes(int64_t nq) {
    return align_up(sizeof(uint32_t) * (size_t)nq) + sort_workspace_bytes(nq) + 512;
}

// 30-bit codes of f32 points on a device scene box (6 f32): the f64
// recipe of morton_kernel on exactly-converted coordinates.
int morton_codes_f32(const float *pts, int64_t n, const float *scene, uint32_t *codes,
                     cudaStream_t stream) {
    if (n < 0 || (n > 0 && (!pts || !scene || !codes))) return LBVH_ERR_INVALID_ARG;
    if (n == 0) return LBVH_OK;
    morton_kernel<uint32_t><<<grid_for(n, 256, 16), 256, 0, stream>>>(pts, pts, n, scene, codes,
                                                                       nullptr);
    count_launches(1);
    return check_launch();
}

namespace {
// Query codes for traversal ordering and the kNN seed only: fp32 cell
// arithmetic (may differ from the f64 reference codes on cell boundaries,
// which changes neither results -- query order never does, and any window of
// leaves gives a valid seed -- nor, measurably, coherence).
__global__ void __launch_bounds__(256)
query_morton_kernel(const float *__restrict__ centers, int64_t n, const float *__restrict__ scene,
                    uint32_t *__restrict__ codes, uint32_t *__restrict__ hist, int first_bit,
                    int passes, uint32_t *status = nullptr, int64_t *__restrict__ offsets = nullptr,
                    int64_t span = 0) {
    // the digit histograms of the order's sort (sort_prepare)
    __shared__ uint32_t s_hist[4][kSortDigits];
    for (int i = threadIdx.x; i < 4 * kSortDigits; i += blockDim.x) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    // optional fused batch prologue: the value check of the centers
    // (check_queries_kernel) and uniform CRS offsets (uniform_offsets_kernel)
    uint32_t bad = 0;
    float lo[3], scale[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = __ldg(scene + a);
        const float ext = __ldg(scene + 3 + a) - lo[a];
        scale[a] = ext > 0.0f ? 1024.0f / ext : 0.0f;
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t g[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float c = __ldg(centers + 3 * i + a);
            if (!isfinite(c)) bad |= LBVH_FLAG_NONFINITE;
            float t = (c - lo[a]) * scale[a];
            t = fminf(fmaxf(t, 0.0f), 1023.0f);  // NaN -> 0 (flagged by the value check)
            g[a] = (uint32_t)t;
        }
        const uint32_t code = (spread_bits(g[0]) << 2) | (spread_bits(g[1]) << 1) | spread_bits(g[2]);
        codes[i] = code;
        hist_accumulate(s_hist, code, first_bit, passes);
        if (offsets) offsets[i] = i * span;
    }
    __syncthreads();
    hist_flush(s_hist, passes, hist);
    if (offsets && blockIdx.x == 0 && threadIdx.x == 0) offsets[n] = n * span;
    if (status) {
        bad = __reduce_or_sync(0xFFFFFFFFu, bad);
        if (bad && (threadIdx.x & 31) == 0) atomicOr(status, bad);
    }
}
}  // namespace

int query_order(const float *centers, int64_t nq, const float *scene, int order_bits,
                uint32_t *order, uint32_t *sorted_codes, void *ws, size_t ws_bytes,
                cudaStream_t stream, uint32_t *status, int64_t *offsets, int64_t span) {
    if (nq < 0 || (nq > 0 && (!centers || !order)) || !scene) return LBVH_ERR_INVALID_ARG;
    if (order_bits < 1 || order_bits > 30) return LBVH_ERR_INVALID_ARG;
    if (nq == 0) return LBVH_OK;
    if (nq >= LBVH_MAX_ITEMS) return LBVH_ERR_TOO_LARGE;
    if (ws_bytes < query_workspace_bytes(nq)) return LBVH_ERR_WORKSPACE;
    Carve c(ws, ws_bytes);
    uint32_t *codes = sorted_codes ? sorted_codes : c.take<uint32_t>(nq);
    void *sort_ws = c.take<char>(sort_workspace_bytes(nq));
    // odd pass counts: encode straight into the sort's ping-pong buffers so
    // the last pass writes (codes, order) -- no copy-back
    const int first_bit = 30 - order_bits;
    const int passes = sort_pass_count(30, first_bit);
    const bool odd = (passes & 1) != 0;
    uint32_t *kin = codes, *vin = order;
    if (odd) sort_alt_buffers(sort_ws, sort_workspace_bytes(nq), nq, &kin, &vin);
    uint32_t *hist = sort_prepare(sort_ws, sort_workspace_bytes(nq), nq, stream);
    // fp32 codes on the tree's grid: an ordering choice only (results never
    // depend on it); query_sort_order keeps the exact f64 recipe.  The values
    // sorted along are the positions, implicit in the first pass.
    query_morton_kernel<<<grid_for(nq, 256, 4), 256, 0, stream>>>(centers, nq, scene, kin, hist,
                                                                 first_bit, passes, status,
                                                                 offsets, span);
    count_launches(1);
    int rc = sort_pairs_prepared(codes, order, nq, 30, sort_ws, sort_workspace_bytes(nq), stream,
                                 first_bit, odd);
    if (rc != LBVH_OK) return rc;
    return check_launch();
}

}  // namespace lbvh
