// traverse.cu -- batched radius and k-nearest traversal on sm_100a.
//
//   spatial_kernel<COUNT>   spatial_pass(store=False)   _kernels.py:179-228
//   spatial_kernel<FILL>    spatial_pass(store=True)    _kernels.py:179-228
//   spatial_kernel<BUFFER>  spatial_pass_buffered       _kernels.py:231-282
//   compact_warp_kernel     compact_rows                _kernels.py:285-290
//   knn_kernel<K>           knn_pass, k <= K <= 32      _kernels.py:293-414
//   knn_smem_heap_kernel    knn_pass, 32 < k <= 400 (heap in shared memory)
//   knn_heap_kernel         knn_pass, any k (heap in the output span)
//
// One thread per query slot s; slot s serves query order[s], so Morton-sorted
// queries put spatially close queries in the same warp and the same CTA
// wave, and their node fetches hit in L1/L2.  Each internal node is one
// 64-byte record (both child boxes + links), fetched with two 256-bit
// loads.  Traversal order, stack discipline and the 64-entry stack limit
// are the reference's, so hit order within a span and stack-exhaustion
// behaviour are identical; kNN keeps a register-resident sorted list of
// (dist^2, ordinal) pairs instead of the reference's heap, which yields the
// same unique k smallest under the lexicographic order.

#include <float.h>

#include <atomic>

#include "common.cuh"
#include "internal.cuh"
#include "topk.cuh"
#include "seed.cuh"

namespace lbvh {
namespace {

__device__ __forceinline__ float bx_of(const lbvh_tree &t, int i) { return __ldg(t.root_box + i); }


enum SpatialMode {
    kCount = 0,     // count only                        (spatial_pass store=False)
    kFill = 1,      // write at offsets[q]               (spatial_pass store=True)
    kBuffer = 2,    // 1P: row of `cap`, abort on overflow (spatial_pass_buffered)
    kCountBuf = 3,  // count all, keep the first `cap` hits in the row (and, with
                    // a spill pool, the rest in pool chunks)
};

// Hits of a kCountBuf query beyond its row go to chunks of a caller-owned
// pool: kSpillChunk - 1 hits, then the index of the query's next chunk.
// Chunk 0 is reserved: its first word counts the chunks handed out.  So the
// count pass keeps EVERY hit, in fill order, and heavy queries (C3: 3.6 % of
// the queries hold 99 % of the hits) need no second traversal; only queries
// that find the pool exhausted are traversed again by the fill pass.
constexpr int kSpillChunk = LBVH_SPILL_CHUNK;
struct SpillPool {
    int32_t *heads;   // per query, written when its count exceeds the row:
                      // first chunk, or -1 = pool exhausted (fill pass)
    int32_t *pool;    // chunks of kSpillChunk ints
    uint32_t chunks;  // pool capacity in chunks, the reserved chunk included
    // Optional lists built as queries finish (warp-aggregated appends):
    // queries whose hits overflowed the row and are not all in the pool (the
    // fill pass revisits them), and queries whose overflow is all in the pool
    // (spill_copy).  Counters zeroed by the caller.
    uint32_t *over_list, *over_n, *spill_list, *spill_n;
};

// Append q to list if `take`, one atomic per converged group of lanes.
__device__ __forceinline__ void append_active(bool take, uint32_t q, uint32_t *list,
                                              uint32_t *count) {
    const unsigned am = __activemask();
    const unsigned m = __ballot_sync(am, take);
    if (!m) return;
    const int lane = (int)lane_id();
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(m));
    base = __shfl_sync(am, base, leader);
    if (take) list[base + __popc(m & ((1u << lane) - 1u))] = q;
}

// The 64-byte record in two 256-bit loads (sm_100 LDG.E.ENL2.256): kNN 8.30 vs
// 8.48 ms and radius 2P 6.09 vs 7.01 ms against four 128-bit loads (C2).
__device__ __forceinline__ void load_node(const PackedNode *__restrict__ nodes, int32_t id,
                                          float4 &a, float4 &b, float4 &c, int4 &d) {
    const PackedNode *p = nodes + id;
    float4 dd;
    ldg256(&p->a, a, b);
    ldg256(&p->c, c, dd);
    d = make_int4(__float_as_int(dd.x), __float_as_int(dd.y), __float_as_int(dd.z),
                  __float_as_int(dd.w));
}

// One hit (leaf ordinal `obj`); returns false when the 1P row overflows.
// `dst` is the query's span / row (out + its base), `cap` its width: 32-bit
// compares and addressing on the per-hit path.
template <int MODE>
__device__ __forceinline__ bool emit(int32_t *__restrict__ dst, int32_t &cnt, int32_t cap,
                                     int32_t obj) {
    if (MODE == kBuffer && cnt >= cap) return false;
    if (MODE == kFill || MODE == kBuffer) dst[cnt] = obj;
    if (MODE == kCountBuf && cnt < cap) dst[cnt] = obj;
    ++cnt;
    return true;
}

// `skip` (kFill only, optional): counts of a kCountBuf pass; queries whose
// hits all fit in its rows (count <= cap) are skipped -- the compaction
// kernel copies those.
#ifndef LBVH_SPATIAL_BLOCK
#define LBVH_SPATIAL_BLOCK 256
#endif
// One query q of a radius batch (spatial_pass for a single query).
template <int MODE>
__device__ __forceinline__ void spatial_query(const lbvh_tree &t,
                                              const float *__restrict__ centers,
                                              const float *__restrict__ radii, float radius,
                                              int64_t q, int32_t *__restrict__ counts,
                                              const int64_t *__restrict__ offsets,
                                              int32_t *__restrict__ out, int64_t cap,
                                              uint32_t *status, const SpillPool pool = {}) {
    const float px = __ldg(centers + 3 * q), py = __ldg(centers + 3 * q + 1),
                pz = __ldg(centers + 3 * q + 2);
    const float r = radii ? __ldg(radii + q) : radius;
    const float r2 = __fmul_rn(r, r);
    int64_t base = 0;
    if (MODE == kFill) base = __ldg(offsets + q);
    if (MODE == kBuffer || MODE == kCountBuf) base = q * cap;
    int32_t cnt = 0;
    int32_t *const dst = out + base;
    const int32_t cap32 = (int32_t)cap;  // row widths and 1P buffers are < 2^31
    int32_t spill_cur = 0, spill_slot = 0;  // current pool chunk (0: none yet, -1: failed)
    auto hit = [&](int32_t obj) -> bool {
        if (MODE == kCountBuf && cnt >= cap32) {
            if (pool.pool && spill_cur >= 0) {
                if (spill_cur == 0 || spill_slot == kSpillChunk - 1) {
                    const uint32_t c = atomicAdd(reinterpret_cast<uint32_t *>(pool.pool), 1u) + 1u;
                    if (c >= pool.chunks) {
                        spill_cur = -1;
                        pool.heads[q] = -1;
                    } else {
                        if (spill_cur == 0)
                            pool.heads[q] = (int32_t)c;
                        else
                            pool.pool[(int64_t)spill_cur * kSpillChunk + kSpillChunk - 1] =
                                (int32_t)c;
                        spill_cur = (int32_t)c;
                        spill_slot = 0;
                    }
                }
                if (spill_cur > 0) pool.pool[(int64_t)spill_cur * kSpillChunk + spill_slot++] = obj;
            }
            ++cnt;
            return true;
        }
        return emit<MODE>(dst, cnt, cap32, obj);
    };
    if (t.n == 1) {
        const float *bx = t.root_box;
        if (box_dist_sq(px, py, pz, bx[0], bx[1], bx[2], bx[3], bx[4], bx[5]) <= r2)
            hit(__ldg(t.leaf_obj));
        if (MODE != kFill) counts[q] = cnt;
        return;
    }
    const PackedNode *__restrict__ nodes = reinterpret_cast<const PackedNode *>(t.nodes);
    // The reference pushes the passing children left, right and pops the
    // right one next.  The node about to be popped is kept in a register
    // instead (`node`), and only the left child goes to the stack; the
    // overflow test still counts it as a stack entry, so the node sequence,
    // hit order and stack-exhaustion behaviour are the reference's.
    // The top entry lives in a register; a pop never waits on memory (the
    // next top is reloaded while the node is fetched): 6.95 vs 7.05 ms per
    // 1e7-query 2P batch (C2), 32 registers.  mem[i] holds entry i - 1 and
    // mem[0] is a dummy, so a pop reloads the next top from mem[sp] without
    // testing for an empty stack (C3 4.23 -> 4.13 ms; an unconditional push
    // as well cost C2 1 %).
    int32_t mem[kStack];
    mem[0] = 0;  // the dummy: defined, never used
    int32_t stop = 0;
    int sp = 0;
    int32_t node = 0;
    uint32_t fail = 0;
    while (true) {
        float4 a, b, c;
        int4 d;
        load_node(nodes, node, a, b, c, d);
        float dl, dr;
        child_dists(px, py, pz, a, b, c, dl, dr);
        int32_t next = -1;
        // left child, then right child (_kernels.py:212-225)
        if (dl <= r2) {
            if (d.x < 0) {
                if (!hit(d.x & 0x7FFFFFFF)) {
                    fail = LBVH_FLAG_BUFFER_OVERFLOW;
                    break;
                }
            } else {
                if (sp >= kStack) {
                    fail = LBVH_FLAG_STACK_EXHAUSTED;
                    break;
                }
                if (sp > 0) mem[sp] = stop;  // the previous top goes to memory
                stop = d.x;
                ++sp;
            }
        }
        if (dr <= r2) {
            if (d.y < 0) {
                if (!hit(d.y & 0x7FFFFFFF)) {
                    fail = LBVH_FLAG_BUFFER_OVERFLOW;
                    break;
                }
            } else {
                if (sp >= kStack) {
                    fail = LBVH_FLAG_STACK_EXHAUSTED;
                    break;
                }
                next = d.y;  // pushed and immediately popped
            }
        }
        if (next >= 0) {
            node = next;
        } else if (sp > 0) {
            --sp;
            node = stop;  // no memory round trip on the critical path
            stop = mem[sp];  // sp = 0: the dummy (unused)
        } else {
            break;
        }
    }
    if (fail) atomicOr(status, fail);
    if (MODE != kFill) counts[q] = cnt;
    if (MODE == kCountBuf && pool.over_list) {
        const bool over = cnt > cap32;
        const bool spilled = over && pool.pool && spill_cur > 0;
        append_active(over && !spilled, (uint32_t)q, pool.over_list, pool.over_n);
        if (pool.spill_list) append_active(spilled, (uint32_t)q, pool.spill_list, pool.spill_n);
    }
}

template <int MODE>
__global__ void __launch_bounds__(LBVH_SPATIAL_BLOCK, 2048 / LBVH_SPATIAL_BLOCK)
spatial_kernel(const lbvh_tree t, const float *__restrict__ centers,
               const float *__restrict__ radii, float radius, const uint32_t *__restrict__ order,
               int64_t nq, int32_t *__restrict__ counts, const int64_t *__restrict__ offsets,
               int32_t *__restrict__ out, int64_t cap, const int32_t *__restrict__ skip,
               uint32_t *status, const SpillPool sp) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nq) return;
    const int64_t q = order ? (int64_t)__ldg(order + s) : s;
    if (MODE == kFill && skip && __ldg(skip + q) <= cap) return;
    spatial_query<MODE>(t, centers, radii, radius, q, counts, offsets, out, cap, status, sp);
}

// The listed (heavy) queries of a 2P batch, in list (= traversal) order:
// a persistent grid whose warps stride over 32-query chunks of the list, so
// the queries in flight at any time are a contiguous stretch of it and
// their node records stay in L2 (a one-wave launch over a long list keeps
// every region of the cloud hot at once and re-reads the tree from HBM).
#ifndef LBVH_LIST_CTAS_PER_SM
#define LBVH_LIST_CTAS_PER_SM 4
#endif
template <int MODE>
__global__ void __launch_bounds__(LBVH_SPATIAL_BLOCK, 2048 / LBVH_SPATIAL_BLOCK)
spatial_list_kernel(const lbvh_tree t, const float *__restrict__ centers,
                    const float *__restrict__ radii, float radius,
                    const uint32_t *__restrict__ list, const uint32_t *__restrict__ list_len,
                    int32_t *__restrict__ counts, const int64_t *__restrict__ offsets,
                    int32_t *__restrict__ out, uint32_t *status) {
    const int64_t n = (int64_t)*list_len;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i - (threadIdx.x & 31) < n;
         i += stride) {
        if (i < n)
            spatial_query<MODE>(t, centers, radii, radius, (int64_t)__ldg(list + i), counts,
                                offsets, out, 0, status);
    }
}

// 5 resident CTAs per SM (<= 48 registers, no spills) with the 12-entry
// shared-memory stack measured fastest at K=10 (8.75 vs 8.89 ms for 6 CTAs
// and a local-memory stack, C2); K=32 keeps the compiler's choice.
#ifndef LBVH_KNN_MINBLOCKS
#define LBVH_KNN_MINBLOCKS 5
#endif
#ifndef LBVH_KNN_SPLIT
#define LBVH_KNN_SPLIT 1  // k-best list as split 32-bit fields (TopKSplit)
#endif
#ifndef LBVH_KNN_SMEMSTACK
#define LBVH_KNN_SMEMSTACK 8  // with the block seed: C2 5.71-5.75 vs 5.77 ms (12), 5.72 (6), 5.74 (4), 5.78 (10)
#endif
// Threads per CTA of knn_kernel (resident threads per SM stay
// LBVH_KNN_MINBLOCKS * 256 for K <= 16).
#ifndef LBVH_KNN_BLOCK
#define LBVH_KNN_BLOCK 64  // 7.69 vs 7.79 ms (256) at C2: finer CTA retirement
#endif
#ifndef LBVH_KNN16_MINBLOCKS
#define LBVH_KNN16_MINBLOCKS 3  // k=16: 14.3 ms vs 14.6 (4) and 15.7 (5, spills)
#endif
#ifndef LBVH_KNN_HEAP_MIN
#define LBVH_KNN_HEAP_MIN 33  // smallest k on the shared-memory heap (below: register lists)
#endif
#ifndef LBVH_KNN_K24
#define LBVH_KNN_K24 1  // a 24-slot register list between the 16- and 32-slot ones
#endif
#ifndef LBVH_KNN32_MINBLOCKS
#define LBVH_KNN32_MINBLOCKS 2
#endif
// Resident CTAs per SM by list size: the k-best keys take 2K registers, so
// larger lists get fewer CTAs instead of spilling.
__host__ __device__ constexpr int knn_min_blocks(int K) {
    return (K <= 10 ? LBVH_KNN_MINBLOCKS : K <= 16 ? LBVH_KNN16_MINBLOCKS : LBVH_KNN32_MINBLOCKS) *
           256 / LBVH_KNN_BLOCK;
}

// One query slot s of a kNN batch (s < nq).
template <int K>
__device__ __forceinline__ void knn_query(const lbvh_tree &t, const float *__restrict__ centers,
                                          const uint32_t *__restrict__ order,
                                          const uint32_t *__restrict__ qcodes, int64_t s,
                                          const int64_t *__restrict__ offsets,
                                          int32_t *__restrict__ out_idx,
                                          float *__restrict__ out_dist, bool squared,
                                          uint32_t *status, float *__restrict__ kth = nullptr,
                                          int uniform = 0) {
    const int64_t q = order ? (int64_t)__ldg(order + s) : s;
    // uniform spans (LBVH_KNN_UNIFORM_SPANS): offsets[q] = q * span, computed
    const int64_t base = uniform ? q * uniform : __ldg(offsets + q);
    const int kk = uniform ? uniform : (int)(__ldg(offsets + q + 1) - base);
    if (kk <= 0) return;
    const float px = __ldg(centers + 3 * q), py = __ldg(centers + 3 * q + 1),
                pz = __ldg(centers + 3 * q + 2);
    if (t.n == 1) {
        const float *bx = t.root_box;
        const float d2 = box_dist_sq(px, py, pz, bx[0], bx[1], bx[2], bx[3], bx[4], bx[5]);
        out_dist[base] = squared ? d2 : __fsqrt_rn(d2);
        out_idx[base] = __ldg(t.leaf_obj);
        if (kth) kth[q] = d2;  // the only candidate is the k-th (forwarding bound)
        return;
    }
    const PackedNode *__restrict__ nodes = reinterpret_cast<const PackedNode *>(t.nodes);
#if LBVH_KNN_SPLIT
    TopKSplit<K> top;
#else
    TopK<K> top;
#endif
#ifdef LBVH_KNN_BOUND_FROM_KTH  // instrumentation: start from a given bound (e.g. the exact k-th)
    const float bound = kth ? __ldg(kth + q) : __int_as_float(0x7FFFFFFF);
    kth = nullptr;
#else
    const float bound = (qcodes && t.leaf_codes)
                            ? seed_bound<K>(t, __ldg(qcodes + s), kk, px, py, pz)
                            : __int_as_float(0x7FFFFFFF);
#endif
    top.init(kk, bound);
    // Reference node order: push farther, push nearer, pop (_kernels.py:363-403).
    // The nearer child stays in a register (`next`) instead of a push/pop
    // pair: its pop-time prune test cannot fire (nothing is offered between
    // its push and pop) and the capacity test still counts it, so node order
    // and stack exhaustion are the reference's.  The first LBVH_KNN_SMEMSTACK
    // entries live in shared memory as bare node ids (lane-interleaved,
    // conflict-free), deeper ones in local memory.  Popped entries are not
    // re-tested (a pruned entry costs one node visit whose children are then
    // pruned), so pushes -- and the capacity test -- are exactly as above.
    constexpr int SMS = LBVH_KNN_SMEMSTACK;
    static_assert(SMS > 0 && SMS <= kStack, "shared-memory stack depth");
    int32_t lstack[kStack];
    __shared__ int32_t sst[SMS * LBVH_KNN_BLOCK];
    // 32-bit shared-window address of this lane's column, formed once: through
    // a generic pointer every push re-derived it (S2UR/ULEA, ~10 instructions)
    uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sst + (threadIdx.x % LBVH_KNN_BLOCK));
    asm volatile("" : "+r"(sbase));  // opaque: kept in a register, not re-derived per push
    uint32_t fail = 0;
    int sp = 0;
    int32_t node = 0;  // the root; never pruned (the list is empty)
#ifdef LBVH_KNN_COUNT_VISITS  // instrumentation builds (tools/knn_visits.py)
    int visits = 0;
#endif
    while (true) {
        float4 a, b, c;
        int4 dd;
#ifdef LBVH_KNN_COUNT_VISITS
        ++visits;
#endif
        load_node(nodes, node, a, b, c, dd);
        float dl, dr;
        child_dists(px, py, pz, a, b, c, dl, dr);
        // farther child first so the nearer one is on top (_kernels.py:373-379)
        const bool left_near = dl <= dr;
        const int32_t fl = left_near ? dd.y : dd.x, nl = left_near ? dd.x : dd.y;
        const float fd = left_near ? dr : dl, ndist = left_near ? dl : dr;
        int32_t next = -1;
        if (!(fd > top.worst())) {  // NaN worst = list not full yet
            if (fl < 0) {
                top.offer(fd, fl & 0x7FFFFFFF);
            } else {
                if (sp >= kStack) {
                    fail = LBVH_FLAG_STACK_EXHAUSTED;
                    break;
                }
                if (sp < SMS)
                    st_shared_s32(sbase + sp * (4 * LBVH_KNN_BLOCK), fl);
                else
                    lstack[sp] = fl;
                ++sp;
            }
        }
        if (!(ndist > top.worst())) {
            if (nl < 0) {
                top.offer(ndist, nl & 0x7FFFFFFF);
            } else {
                if (sp >= kStack) {
                    fail = LBVH_FLAG_STACK_EXHAUSTED;
                    break;
                }
                next = nl;
            }
        }
        if (next < 0) {
            if (sp == 0) break;
            --sp;
            next = sp < SMS ? ld_shared_s32(sbase + sp * (4 * LBVH_KNN_BLOCK)) : lstack[sp];
        }
        node = next;
    }
    if (fail) atomicOr(status, fail);
#ifdef LBVH_KNN_COUNT_VISITS  // node visits / kept offers in place of the two nearest distances
#if LBVH_KNN_SPLIT
    top.d[0] = __float_as_uint((float)visits * (float)visits);
    top.d[1] = __float_as_uint((float)top.kept * (float)top.kept);
#else
    top.key[0] = ((uint64_t)__float_as_uint((float)visits * (float)visits) << 32) |
                 (top.key[0] & 0xFFFFFFFFull);
    top.key[1] = ((uint64_t)__float_as_uint((float)top.kept * (float)top.kept) << 32) |
                 (top.key[1] & 0xFFFFFFFFull);
#endif
#endif
    // the k-th squared distance (exact; the sharded search's forwarding bound)
    if (kth) kth[q] = top.dist(K - 1);
    // Spans are written even after a failure; the driver raises anyway.
    if ((K & 1) == 0 && kk == K && (base & 1) == 0) {
        // full span at an even offset: 64-bit stores (half the store requests)
#pragma unroll
        for (int j = 0; j < K; j += 2) {
            const float d0 = squared ? top.dist(j) : __fsqrt_rn(top.dist(j));
            const float d1 = squared ? top.dist(j + 1) : __fsqrt_rn(top.dist(j + 1));
            *reinterpret_cast<int2 *>(out_idx + base + j) =
                make_int2(top.ordinal(j), top.ordinal(j + 1));
            *reinterpret_cast<float2 *>(out_dist + base + j) = make_float2(d0, d1);
        }
        return;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (j >= K - kk) {
            const int64_t o = base + (j - (K - kk));
            out_idx[o] = top.ordinal(j);
            out_dist[o] = squared ? top.dist(j) : __fsqrt_rn(top.dist(j));
        }
    }
}

template <int K>
__global__ void __launch_bounds__(LBVH_KNN_BLOCK,
                                  knn_min_blocks(K))
knn_kernel(const lbvh_tree t, const float *__restrict__ centers,
           const uint32_t *__restrict__ order, const uint32_t *__restrict__ qcodes, int64_t nq,
           const int64_t *__restrict__ offsets, int32_t *__restrict__ out_idx,
           float *__restrict__ out_dist, bool squared, uint32_t *status, float *kth,
           int uniform) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nq) return;
    knn_query<K>(t, centers, order, qcodes, s, offsets, out_idx, out_dist, squared, status, kth,
                 uniform);
}

// General k: the output span doubles as a bounded max-heap, exactly the
// reference's scheme (_kernels.py:299-325, 385-414).
__device__ __forceinline__ bool worse(float d1, int32_t i1, float d2, int32_t i2) {
    return d1 > d2 || (d1 == d2 && i1 > i2);
}

__device__ void sift_down(float *hd, int32_t *hi, int64_t size, int64_t pos) {
    while (true) {
        int64_t child = 2 * pos + 1;
        if (child >= size) break;
        int64_t sib = child + 1;
        if (sib < size && worse(hd[sib], hi[sib], hd[child], hi[child])) child = sib;
        if (!worse(hd[child], hi[child], hd[pos], hi[pos])) break;
        float td = hd[pos]; hd[pos] = hd[child]; hd[child] = td;
        int32_t ti = hi[pos]; hi[pos] = hi[child]; hi[child] = ti;
        pos = child;
    }
}

__device__ void sift_up(float *hd, int32_t *hi, int64_t pos) {
    while (pos > 0) {
        int64_t up = (pos - 1) >> 1;
        if (!worse(hd[pos], hi[pos], hd[up], hi[up])) break;
        float td = hd[pos]; hd[pos] = hd[up]; hd[up] = td;
        int32_t ti = hi[pos]; hi[pos] = hi[up]; hi[up] = ti;
        pos = up;
    }
}

__global__ void __launch_bounds__(128)
knn_heap_kernel(const lbvh_tree t, const float *__restrict__ centers,
                const uint32_t *__restrict__ order, int64_t nq,
                const int64_t *__restrict__ offsets, int32_t *__restrict__ out_idx,
                float *__restrict__ out_dist, bool squared, uint32_t *status) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nq) return;
    const int64_t q = order ? (int64_t)__ldg(order + s) : s;
    const int64_t base = __ldg(offsets + q);
    const int64_t kk = __ldg(offsets + q + 1) - base;
    if (kk <= 0) return;
    const float px = __ldg(centers + 3 * q), py = __ldg(centers + 3 * q + 1),
                pz = __ldg(centers + 3 * q + 2);
    float *hd = out_dist + base;
    int32_t *hi = out_idx + base;
    if (t.n == 1) {
        const float d2 = box_dist_sq(px, py, pz, bx_of(t, 0), bx_of(t, 1), bx_of(t, 2),
                                     bx_of(t, 3), bx_of(t, 4), bx_of(t, 5));
        hd[0] = squared ? d2 : __fsqrt_rn(d2);
        hi[0] = __ldg(t.leaf_obj);
        return;
    }
    const PackedNode *__restrict__ nodes = reinterpret_cast<const PackedNode *>(t.nodes);
    int32_t stack_node[kStack];
    float stack_dist[kStack];
    int sp = 1;
    stack_node[0] = 0;
    stack_dist[0] = 0.0f;
    int64_t size = 0;
    uint32_t fail = 0;
    while (sp > 0) {
        --sp;
        const int32_t node = stack_node[sp];
        if (size == kk && stack_dist[sp] > hd[0]) continue;
        float4 a, b, c;
        int4 dd;
        load_node(nodes, node, a, b, c, dd);
        float dl, dr;
        child_dists(px, py, pz, a, b, c, dl, dr);
        const bool left_near = dl <= dr;
        const int32_t fl = left_near ? dd.y : dd.x, nl = left_near ? dd.x : dd.y;
        const float fd = left_near ? dr : dl, ndist = left_near ? dl : dr;
        for (int pick = 0; pick < 2; ++pick) {
            const int32_t link = pick == 0 ? fl : nl;
            const float cd = pick == 0 ? fd : ndist;
            if (size == kk && cd > hd[0]) continue;
            if (link < 0) {
                const int32_t obj = link & 0x7FFFFFFF;
                if (size < kk) {
                    hd[size] = cd;
                    hi[size] = obj;
                    ++size;
                    sift_up(hd, hi, size - 1);
                } else if (worse(hd[0], hi[0], cd, obj)) {
                    hd[0] = cd;
                    hi[0] = obj;
                    sift_down(hd, hi, kk, 0);
                }
            } else {
                if (sp >= kStack) {
                    fail = LBVH_FLAG_STACK_EXHAUSTED;
                    goto done;
                }
                stack_node[sp] = link;
                stack_dist[sp] = cd;
                ++sp;
            }
        }
    }
done:
    if (fail) atomicOr(status, fail);
    for (int64_t hs = size; hs > 1;) {
        --hs;
        float td = hd[0]; hd[0] = hd[hs]; hd[hs] = td;
        int32_t ti = hi[0]; hi[0] = hi[hs]; hi[hs] = ti;
        sift_down(hd, hi, hs, 0);
    }
    if (!squared)
        for (int64_t j = 0; j < size; ++j) hd[j] = __fsqrt_rn(hd[j]);
}

// k > 32: the reference's bounded max-heap (_kernels.py:299-325, 385-414),
// kept in shared memory (64-bit keys (dist^2 bits << 32 | ordinal), the
// lexicographic "worse" order in one compare; lane-interleaved slots) instead
// of the output span in global memory.  Traversal and stack discipline are
// knn_pass's (push farther then nearer, pop with the prune test), so results
// and stack exhaustion are the reference's.
constexpr int kHeapThreads = 64;

__device__ __forceinline__ uint64_t &hslot(uint64_t *h, int i) {
    return h[(int64_t)i * kHeapThreads];
}

__global__ void __launch_bounds__(kHeapThreads)
knn_smem_heap_kernel(const lbvh_tree t, const float *__restrict__ centers,
                     const uint32_t *__restrict__ order, int64_t nq,
                     const int64_t *__restrict__ offsets, int32_t *__restrict__ out_idx,
                     float *__restrict__ out_dist, bool squared, uint32_t *status) {
    extern __shared__ uint64_t s_heap[];
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nq) return;
    const int64_t q = order ? (int64_t)__ldg(order + s) : s;
    const int64_t base = __ldg(offsets + q);
    const int kk = (int)(__ldg(offsets + q + 1) - base);
    if (kk <= 0) return;
    const float px = __ldg(centers + 3 * q), py = __ldg(centers + 3 * q + 1),
                pz = __ldg(centers + 3 * q + 2);
    if (t.n == 1) {
        const float d2 = box_dist_sq(px, py, pz, bx_of(t, 0), bx_of(t, 1), bx_of(t, 2),
                                     bx_of(t, 3), bx_of(t, 4), bx_of(t, 5));
        out_dist[base] = squared ? d2 : __fsqrt_rn(d2);
        out_idx[base] = __ldg(t.leaf_obj);
        return;
    }
    uint64_t *h = s_heap + threadIdx.x;
    int size = 0;
    auto worst = [&]() { return __uint_as_float((uint32_t)(hslot(h, 0) >> 32)); };
    auto offer = [&](float d, int32_t obj) {
        const uint64_t c = ((uint64_t)__float_as_uint(d) << 32) | (uint32_t)obj;
        if (size < kk) {  // sift up
            int pos = size++;
            while (pos > 0) {
                const int up = (pos - 1) >> 1;
                const uint64_t u = hslot(h, up);
                if (!(c > u)) break;
                hslot(h, pos) = u;
                pos = up;
            }
            hslot(h, pos) = c;
        } else if (c < hslot(h, 0)) {  // replace the worst, sift down
            int pos = 0;
            while (true) {
                int child = 2 * pos + 1;
                if (child >= kk) break;
                uint64_t cv = hslot(h, child);
                if (child + 1 < kk) {
                    const uint64_t sv = hslot(h, child + 1);
                    if (sv > cv) {
                        cv = sv;
                        ++child;
                    }
                }
                if (!(cv > c)) break;
                hslot(h, pos) = cv;
                pos = child;
            }
            hslot(h, pos) = c;
        }
    };
    const PackedNode *__restrict__ nodes = reinterpret_cast<const PackedNode *>(t.nodes);
    uint64_t stack[kStack];
    int sp = 1;
    stack[0] = 0;  // (dist^2 = 0, root)
    uint32_t fail = 0;
    while (sp > 0) {
        const uint64_t e = stack[--sp];
        if (size == kk && __uint_as_float((uint32_t)(e >> 32)) > worst()) continue;
        float4 a, b, c;
        int4 dd;
        load_node(nodes, (int32_t)(uint32_t)e, a, b, c, dd);
        float dl, dr;
        child_dists(px, py, pz, a, b, c, dl, dr);
        const bool left_near = dl <= dr;
        const int32_t fl = left_near ? dd.y : dd.x, nl = left_near ? dd.x : dd.y;
        const float fd = left_near ? dr : dl, ndist = left_near ? dl : dr;
#pragma unroll
        for (int pick = 0; pick < 2; ++pick) {
            const int32_t link = pick == 0 ? fl : nl;
            const float cd = pick == 0 ? fd : ndist;
            if (size == kk && cd > worst()) continue;
            if (link < 0) {
                offer(cd, link & 0x7FFFFFFF);
            } else {
                if (sp >= kStack) {
                    fail = LBVH_FLAG_STACK_EXHAUSTED;
                    goto done;
                }
                stack[sp++] = ((uint64_t)__float_as_uint(cd) << 32) | (uint32_t)link;
            }
        }
    }
done:
    if (fail) atomicOr(status, fail);
    // heap sort: ascending (dist^2, ordinal) into the span
    for (int hs = size; hs > 0; --hs) {
        const uint64_t top = hslot(h, 0);
        const int64_t o = base + hs - 1;
        out_idx[o] = (int32_t)(uint32_t)top;
        const float d2 = __uint_as_float((uint32_t)(top >> 32));
        out_dist[o] = squared ? d2 : __fsqrt_rn(d2);
        const uint64_t c = hslot(h, hs - 1);
        int pos = 0;
        const int n = hs - 1;
        while (true) {
            int child = 2 * pos + 1;
            if (child >= n) break;
            uint64_t cv = hslot(h, child);
            if (child + 1 < n) {
                const uint64_t sv = hslot(h, child + 1);
                if (sv > cv) {
                    cv = sv;
                    ++child;
                }
            }
            if (!(cv > c)) break;
            hslot(h, pos) = cv;
            pos = child;
        }
        if (n > 0) hslot(h, pos) = c;
    }
}

__global__ void __launch_bounds__(256)
check_queries_kernel(const float *__restrict__ centers, int64_t nq,
                     const float *__restrict__ radii, uint32_t *status) {
    uint32_t bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 3 * nq;
         i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(__ldcs(centers + i))) bad |= LBVH_FLAG_NONFINITE;
    if (radii)
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nq;
             i += (int64_t)gridDim.x * blockDim.x) {
            float r = __ldcs(radii + i);
            if (!isfinite(r) || r < 0.0f) bad |= LBVH_FLAG_BAD_RADIUS;
        }
    bad = __reduce_or_sync(0xFFFFFFFFu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicOr(status, bad);
}

bool tree_ok(const lbvh_tree *t) {
    return t && t->n >= 1 && t->leaf_obj && t->root_box && (t->n == 1 || t->nodes);
}

template <int MODE>
int launch_spatial(const lbvh_tree *t, const float *centers, const float *radii, float radius,
                   const uint32_t *order, int64_t nq, int32_t *counts, const int64_t *offsets,
                   int32_t *out, int64_t cap, const int32_t *skip, uint32_t *status,
                   cudaStream_t stream, const SpillPool sp = {}) {
    if (!tree_ok(t) || nq < 0 || !status) return LBVH_ERR_INVALID_ARG;
    if (nq == 0) return LBVH_OK;
    if (!centers) return LBVH_ERR_INVALID_ARG;
    if (MODE != kFill && !counts) return LBVH_ERR_INVALID_ARG;
    if (MODE == kFill && !offsets) return LBVH_ERR_INVALID_ARG;
    if (nq >= LBVH_MAX_ITEMS) return LBVH_ERR_TOO_LARGE;
    spatial_kernel<MODE><<<div_up(nq, LBVH_SPATIAL_BLOCK), LBVH_SPATIAL_BLOCK, 0, stream>>>(
        *t, centers, radii, radius, order, nq, counts, offsets, out, cap, skip, status, sp);
    count_launches(1);
    return check_launch();
}

}  // namespace

int spatial_count(const lbvh_tree *t, const float *centers, const float *radii, float radius,
                  const uint32_t *order, int64_t nq, int32_t *counts, int32_t *buf, int64_t cap,
                  uint32_t *status, cudaStream_t stream, int32_t *spill_heads,
                  int32_t *spill_pool, int64_t spill_chunks, uint32_t *over_list,
                  uint32_t *over_n, uint32_t *spill_list, uint32_t *spill_n) {
    if (buf) {
        if (cap < 1) return LBVH_ERR_INVALID_ARG;
        SpillPool sp = {};
        if (spill_pool && spill_heads && spill_chunks > 1) {
            sp.heads = spill_heads;
            sp.pool = spill_pool;
            sp.chunks = (uint32_t)(spill_chunks < (int64_t)1 << 31 ? spill_chunks
                                                                   : (int64_t)1 << 31);
            cudaMemsetAsync(spill_pool, 0, sizeof(uint32_t), stream);  // allocation counter
            if (spill_list && spill_n) {
                sp.spill_list = spill_list;
                sp.spill_n = spill_n;
                cudaMemsetAsync(spill_n, 0, sizeof(uint32_t), stream);
            }
        }
        if (over_list && over_n) {
            sp.over_list = over_list;
            sp.over_n = over_n;
            cudaMemsetAsync(over_n, 0, sizeof(uint32_t), stream);
        }
        return launch_spatial<kCountBuf>(t, centers, radii, radius, order, nq, counts, nullptr,
                                         buf, cap, nullptr, status, stream, sp);
    }
    return launch_spatial<kCount>(t, centers, radii, radius, order, nq, counts, nullptr,
                                  nullptr, 0, nullptr, status, stream);
}

int spatial_list(const lbvh_tree *t, const float *centers, const float *radii, float radius,
                 const uint32_t *list, const uint32_t *list_len, int64_t max_list,
                 int32_t *counts, const int64_t *offsets, int32_t *out, bool fill,
                 uint32_t *status, cudaStream_t stream) {
    if (!tree_ok(t) || !centers || !list || !list_len || !status || max_list < 0)
        return LBVH_ERR_INVALID_ARG;
    if (fill ? (!offsets || !out) : !counts) return LBVH_ERR_INVALID_ARG;
    if (max_list == 0) return LBVH_OK;
    int64_t ctas = (max_list + LBVH_SPATIAL_BLOCK - 1) / LBVH_SPATIAL_BLOCK;
    const int64_t cap = (int64_t)kNumSMs * LBVH_LIST_CTAS_PER_SM;
    const unsigned g = (unsigned)(ctas < cap ? ctas : cap);
    if (fill)
        spatial_list_kernel<kFill><<<g, LBVH_SPATIAL_BLOCK, 0, stream>>>(
            *t, centers, radii, radius, list, list_len, counts, offsets, out, status);
    else
        spatial_list_kernel<kCount><<<g, LBVH_SPATIAL_BLOCK, 0, stream>>>(
            *t, centers, radii, radius, list, list_len, counts, offsets, out, status);
    count_launches(1);
    return check_launch();
}

int spatial_fill(const lbvh_tree *t, const float *centers, const float *radii, float radius,
                 const uint32_t *order, int64_t nq, const int64_t *offsets, int32_t *out,
                 const int32_t *skip_counts, int64_t cap, uint32_t *status,
                 cudaStream_t stream) {
    return launch_spatial<kFill>(t, centers, radii, radius, order, nq, nullptr, offsets, out,
                                 skip_counts ? cap : 0, skip_counts, status, stream);
}

int spatial_1p(const lbvh_tree *t, const float *centers, const float *radii, float radius,
               const uint32_t *order, int64_t nq, int32_t *buf, int64_t cap, int32_t *counts,
               uint32_t *status, cudaStream_t stream) {
    if (cap < 1 || (nq > 0 && !buf)) return LBVH_ERR_INVALID_ARG;
    return launch_spatial<kBuffer>(t, centers, radii, radius, order, nq, counts, nullptr, buf,
                                   cap, nullptr, status, stream);
}

// Warp-cooperative compaction: a warp takes 32 rows,
// scans their hit counts and writes the concatenation with consecutive lanes
// on consecutive output words (element e of the warp's run belongs to the row
// found by a 5-step shuffle search of the scan).  Rows that overflowed their
// buffer count 0 here (the fill pass writes them).
// (radius 2P at C2: 5.51 vs 5.88 ms with a thread per row; ~30 hits/query: 10.8 vs 12.1)
__global__ void __launch_bounds__(256)
compact_warp_kernel(const int32_t *__restrict__ buf, int64_t cap,
                    const int32_t *__restrict__ counts, const int64_t *__restrict__ offsets,
                    int64_t nq, int32_t *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w * 32 < nq;
         w += warps) {
        const int64_t q = w * 32 + lane;
        int32_t cnt = 0;
        int64_t dst = 0;
        if (q < nq) {
            cnt = __ldg(counts + q);
            cnt = cnt <= cap ? cnt : 0;
            dst = __ldg(offsets + q);
        }
        int32_t incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        const int32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
        const int32_t excl = incl - cnt;
        for (int32_t base = 0; base < total; base += 32) {
            const int32_t e = base + lane;
            // row r: the last lane whose exclusive prefix is <= e
            int r = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int32_t pre = __shfl_sync(0xFFFFFFFFu, excl, r + step);
                if (pre <= e) r += step;
            }
            const int32_t pre_r = __shfl_sync(0xFFFFFFFFu, excl, r);
            const int64_t dst_r = __shfl_sync(0xFFFFFFFFu, dst, r);
            if (e < total) {
                const int32_t j = e - pre_r;
                out[dst_r + j] = __ldcs(buf + (w * 32 + r) * cap + j);
            }
        }
    }
}

int compact(const int32_t *buf, int64_t cap, const int32_t *counts, const int64_t *offsets,
            int64_t nq, int32_t *out, cudaStream_t stream) {
    if (nq < 0 || cap < 1) return LBVH_ERR_INVALID_ARG;
    if (nq == 0) return LBVH_OK;
    if (!buf || !counts || !offsets) return LBVH_ERR_INVALID_ARG;
    unsigned g = div_up(nq, 256);
    g = g < kNumSMs * 8 ? g : kNumSMs * 8;
    compact_warp_kernel<<<g, 256, 0, stream>>>(buf, cap, counts, offsets, nq, out);
    count_launches(1);
    return check_launch();
}

// Reserved: lbvh_knn takes no workspace today (the argument is accepted and unused).
size_t knn_workspace_bytes(int64_t) { return 0; }

namespace {
__global__ void __launch_bounds__(256)
leaf_directory_kernel(const uint32_t *__restrict__ codes, int64_t n, int bits,
                      uint32_t *__restrict__ dir) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p > ((int64_t)1 << bits)) return;
    const uint64_t target = (uint64_t)p << (30 - bits);
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((uint64_t)__ldg(codes + mid) < target)
            lo = mid + 1;
        else
            hi = mid;
    }
    dir[p] = (uint32_t)lo;
}
}  // namespace

int leaf_directory(const uint32_t *codes, int64_t n, int bits, uint32_t *dir,
                   cudaStream_t stream) {
    if (n < 1 || bits < 0 || bits > 30 || !codes || !dir) return LBVH_ERR_INVALID_ARG;
    if (n >= LBVH_MAX_ITEMS) return LBVH_ERR_TOO_LARGE;
    const int64_t entries = ((int64_t)1 << bits) + 1;
    leaf_directory_kernel<<<div_up(entries, 256), 256, 0, stream>>>(codes, n, bits, dir);
    count_launches(1);
    return check_launch();
}

int knn(const lbvh_tree *t, const float *centers, const uint32_t *order,
        const uint32_t *qcodes, int64_t nq, const int64_t *offsets, int64_t max_span,
        int32_t *out_idx, float *out_dist, int flags, void *ws, size_t ws_bytes,
        uint32_t *status, cudaStream_t stream, float *kth) {
    if (kth && max_span > 32) return LBVH_ERR_INVALID_ARG;  // register-list kernels only
    if (!tree_ok(t) || nq < 0 || !status) return LBVH_ERR_INVALID_ARG;
    if (nq == 0 || max_span <= 0) return LBVH_OK;
    if (!centers || !offsets || !out_idx || !out_dist) return LBVH_ERR_INVALID_ARG;
    if (nq >= LBVH_MAX_ITEMS) return LBVH_ERR_TOO_LARGE;
    const unsigned g = div_up(nq, LBVH_KNN_BLOCK);
#define LBVH_KNN_CASE(KV)                                                                   \
    if (max_span <= KV) {                                                                   \
        knn_kernel<KV><<<g, LBVH_KNN_BLOCK, 0, stream>>>(*t, centers, order, qcodes, nq,     \
                                                        offsets, out_idx, out_dist, squared, \
                                                        status, kth, uniform);              \
        count_launches(1);                                                                  \
        return check_launch();                                                              \
    }
    const bool squared = (flags & LBVH_KNN_SQUARED) != 0;
    const int uniform = (flags & LBVH_KNN_UNIFORM_SPANS) ? (int)max_span : 0;
    LBVH_KNN_CASE(4)
    LBVH_KNN_CASE(8)
    LBVH_KNN_CASE(10)
    // register lists up to k = 32 (split lists + block seed, round 2): C2 k = 20 / 24 / 32
    // 14.3 / 15.9 / 27.9 ms with 24- and 32-slot lists vs 21.1 / 23.7 / 31.5 ms on the
    // shared-memory heap (which round 1 preferred above k = 16: 23.9 vs 33.9 ms at k = 24)
    if (max_span < LBVH_KNN_HEAP_MIN || kth) {
        LBVH_KNN_CASE(16)
#if LBVH_KNN_K24
        LBVH_KNN_CASE(24)
#endif
        LBVH_KNN_CASE(32)
    }
#undef LBVH_KNN_CASE
    // shared-memory heap up to 400 slots per query (64 threads x 8 B x k <= 200 KB)
    const size_t smem = (size_t)kHeapThreads * 8 * (size_t)max_span;
    if (max_span <= 400) {
        // the opt-in is per device context: remember it per device (atomically,
        // host threads may launch concurrently)
        static std::atomic<uint32_t> opted{0};
        int dev = 0;
        cudaGetDevice(&dev);
        const uint32_t bit = 1u << (dev & 31);
        if (smem > 48 * 1024 && !(opted.load() & bit)) {
            cudaFuncSetAttribute(knn_smem_heap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(kHeapThreads * 8 * 400));
            opted.fetch_or(bit);
        }
        knn_smem_heap_kernel<<<div_up(nq, kHeapThreads), kHeapThreads, smem, stream>>>(
            *t, centers, order, nq, offsets, out_idx, out_dist, squared, status);
        count_launches(1);
        return check_launch();
    }
    knn_heap_kernel<<<div_up(nq, 128), 128, 0, stream>>>(*t, centers, order, nq, offsets,
                                                         out_idx, out_dist, squared, status);
    count_launches(1);
    return check_launch();
}

namespace {
__global__ void __launch_bounds__(256)
unpack_knn_keys_kernel(const uint64_t *__restrict__ keys, int64_t n, int64_t *__restrict__ gid,
                       float *__restrict__ dist) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t k = __ldg(keys + i);
        gid[i] = (int64_t)(k & 0xFFFFFFFFull);
        dist[i] = __fsqrt_rn(__uint_as_float((uint32_t)(k >> 32)));
    }
}
}  // namespace

namespace {
// Queries whose hits overflowed their row, listed (in traversal order within
// each warp) so the fill pass runs on full warps of them only.
// With spill heads: queries whose overflow hits all went to the pool go to
// the spill list (copied by spill_copy_kernel), the others to `list`.
__device__ __forceinline__ void append_warp(bool take, uint32_t q, uint32_t *list,
                                            uint32_t *count) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, take);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(m));
    base = __shfl_sync(0xFFFFFFFFu, base, leader);
    if (take) list[base + __popc(m & ((1u << lane) - 1u))] = q;
}

__global__ void __launch_bounds__(256)
select_overflow_kernel(const uint32_t *__restrict__ order, const int32_t *__restrict__ counts,
                       int64_t nq, int64_t cap, uint32_t *__restrict__ list, uint32_t *count,
                       const int32_t *__restrict__ heads, uint32_t *__restrict__ spill_list,
                       uint32_t *spill_count) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t q = 0;
    bool over = false, spilled = false;
    if (s < nq) {
        q = order ? __ldg(order + s) : (uint32_t)s;
        over = __ldg(counts + q) > cap;
        if (over && heads) spilled = __ldg(heads + q) > 0;
    }
    append_warp(over && !spilled, q, list, count);
    if (heads) append_warp(spilled, q, spill_list, spill_count);
}

// Spilled queries' spans: the row (first `cap` hits) then the pool chunks,
// one half-warp per query (two queries' chunk chains in flight per warp),
// consecutive lanes on consecutive output words; each lane has all of its
// loads of a chunk in flight before it stores, the next chunk's index among them.
__global__ void __launch_bounds__(256)
spill_copy_kernel(const int32_t *__restrict__ buf, int64_t cap,
                  const int32_t *__restrict__ counts, const int64_t *__restrict__ offsets,
                  const int32_t *__restrict__ heads, const int32_t *__restrict__ pool,
                  const uint32_t *__restrict__ list, const uint32_t *__restrict__ list_len,
                  int32_t *__restrict__ out) {
    constexpr int kG = 16;                           // lanes per query
    constexpr int kPer = (kSpillChunk + kG - 1) / kG;  // words per lane per chunk
    const int g = threadIdx.x & (kG - 1);
    const unsigned gmask = 0xFFFFu << (threadIdx.x & 16);  // this half-warp
    const int64_t n = (int64_t)*list_len;
    const int64_t groups = ((int64_t)gridDim.x * blockDim.x) / kG;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kG; w < n; w += groups) {
        const int64_t q = __ldg(list + w);
        const int64_t cnt = __ldg(counts + q);
        int32_t *dst = out + __ldg(offsets + q);
        int64_t c = __ldg(heads + q);
        const int32_t *row = buf + q * cap;
        for (int64_t j = g; j < cap; j += kG) dst[j] = __ldcs(row + j);
        int64_t done = cap;
        while (done < cnt) {
            const int64_t take = cnt - done < kSpillChunk - 1 ? cnt - done : kSpillChunk - 1;
            const int32_t *ch = pool + c * kSpillChunk;
            int32_t v[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) v[u] = __ldcs(ch + u * kG + g);  // slot 127: the link
            const int64_t next = __shfl_sync(gmask, v[kPer - 1], kG - 1, kG);
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const int j = u * kG + g;
                if (j < take) dst[done + j] = v[u];
            }
            done += take;
            c = next;
        }
    }
}
}  // namespace

int select_overflow(const uint32_t *order, const int32_t *counts, int64_t nq, int64_t cap,
                    uint32_t *list, uint32_t *count, cudaStream_t stream,
                    const int32_t *spill_heads, uint32_t *spill_list, uint32_t *spill_count) {
    if (nq < 0 || (nq > 0 && (!counts || !list || !count))) return LBVH_ERR_INVALID_ARG;
    if (!count || (spill_heads && (!spill_list || !spill_count))) return LBVH_ERR_INVALID_ARG;
    cudaMemsetAsync(count, 0, sizeof(uint32_t), stream);
    if (spill_heads) cudaMemsetAsync(spill_count, 0, sizeof(uint32_t), stream);
    if (nq == 0) return check_launch();
    select_overflow_kernel<<<div_up(nq, 256), 256, 0, stream>>>(
        order, counts, nq, cap, list, count, spill_heads, spill_list, spill_count);
    count_launches(1);
    return check_launch();
}

int spill_copy(const int32_t *buf, int64_t cap, const int32_t *counts, const int64_t *offsets,
               const int32_t *heads, const int32_t *pool, const uint32_t *list,
               const uint32_t *list_len, int64_t max_list, int32_t *out, cudaStream_t stream) {
    if (max_list < 0 || cap < 1) return LBVH_ERR_INVALID_ARG;
    if (max_list == 0) return LBVH_OK;
    if (!buf || !counts || !offsets || !heads || !pool || !list || !list_len || !out)
        return LBVH_ERR_INVALID_ARG;
    int64_t ctas = (max_list + 15) / 16;  // 16 queries per 256-thread CTA
    const int64_t lim = (int64_t)kNumSMs * 8;
    spill_copy_kernel<<<(unsigned)(ctas < lim ? ctas : lim), 256, 0, stream>>>(
        buf, cap, counts, offsets, heads, pool, list, list_len, out);
    count_launches(1);
    return check_launch();
}

int unpack_knn_keys(const uint64_t *keys, int64_t n, int64_t *gid, float *dist,
                    cudaStream_t stream) {
    if (n < 0 || (n > 0 && (!keys || !gid || !dist))) return LBVH_ERR_INVALID_ARG;
    if (n == 0) return LBVH_OK;
    unsigned g = div_up(n, 256);
    g = g < kNumSMs * 16 ? g : kNumSMs * 16;
    unpack_knn_keys_kernel<<<g, 256, 0, stream>>>(keys, n, gid, dist);
    count_launches(1);
    return check_launch();
}

int check_queries(const float *centers, int64_t nq, const float *radii, uint32_t *status,
                  cudaStream_t stream) {
    if (nq < 0 || !status) return LBVH_ERR_INVALID_ARG;
    if (nq == 0) return LBVH_OK;
    if (!centers) return LBVH_ERR_INVALID_ARG;
    unsigned g = div_up(3 * nq, 256);
    g = g < kNumSMs * 8 ? g : kNumSMs * 8;
    check_queries_kernel<<<g, 256, 0, stream>>>(centers, nq, radii, status); count_launches(1);
    return check_launch();
}

}  // namespace lbvh
