// wide.cu -- 4-wide traversal records for kNN (no reference counterpart; a
// layout of the same tree, results unchanged).
//
// wide record of internal node X (128 B, one L2 line): the up-to-four
// "grandchild" entries of X -- for each child C of X, C itself if it is a
// leaf, else C's two children -- as SoA boxes + links.  A traversal that
// starts at the root and descends through entries only ever enters internal
// nodes two binary levels apart, so one dependent 128-byte fetch replaces two
// 64-byte ones, and the four box tests are independent.
//
//   lox, loy, loz, hix, hiy, hiz : float4 (entry i in lane i of each)
//   link : int4   leaf = obj | 1<<31, internal = Karras id, empty = -1
//   pad  : int4
//
// knn_wide_kernel<K> returns exactly knn_kernel<K>'s results (the k smallest
// (dist^2, ordinal) pairs; order of visits never matters).  It visits a
// different node sequence than the reference's binary DFS, so it is used only
// on trees built by lbvh_build with 30-bit codes: their depth is <= 60 (30
// code bits + at most 30 index bits), so the reference's 64-entry stack never
// overflows on them, and this kernel's stack (at most 3 pushes per wide
// level, <= 30 levels) is sized to never overflow either.

#include <float.h>

#include "common.cuh"
#include "internal.cuh"
#include "topk.cuh"
#include "seed.cuh"

namespace lbvh {

struct __align__(128) WideNode {
    float4 lox, loy, loz, hix, hiy, hiz;
    int4 link;
    int4 pad;
};
static_assert(sizeof(WideNode) == 128, "wide record must be 128 B");

namespace {

constexpr int kWideStack = 96;
constexpr int kEmpty = -1;

__device__ __forceinline__ void put(WideNode &w, int i, float lx, float ly, float lz, float hx,
                                    float hy, float hz, int32_t link) {
    reinterpret_cast<float *>(&w.lox)[i] = lx;
    reinterpret_cast<float *>(&w.loy)[i] = ly;
    reinterpret_cast<float *>(&w.loz)[i] = lz;
    reinterpret_cast<float *>(&w.hix)[i] = hx;
    reinterpret_cast<float *>(&w.hiy)[i] = hy;
    reinterpret_cast<float *>(&w.hiz)[i] = hz;
    reinterpret_cast<int32_t *>(&w.link)[i] = link;
}

__global__ void __launch_bounds__(256)
wide_records_kernel(const PackedNode *__restrict__ nodes, int64_t n_internal,
                    WideNode *__restrict__ wide) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n_internal;
         x += (int64_t)gridDim.x * blockDim.x) {
        const PackedNode *p = nodes + x;
        const float4 a = __ldg(&p->a), b = __ldg(&p->b), c = __ldg(&p->c);
        const int4 d = __ldg(&p->d);
        WideNode w;
        int cnt = 0;
        // left child box a.x a.y a.z | a.w b.x b.y ; right child b.z b.w c.x | c.y c.z c.w
        const float cb[2][6] = {{a.x, a.y, a.z, a.w, b.x, b.y}, {b.z, b.w, c.x, c.y, c.z, c.w}};
        const int32_t cl[2] = {d.x, d.y};
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            if (cl[s] < 0) {
                put(w, cnt++, cb[s][0], cb[s][1], cb[s][2], cb[s][3], cb[s][4], cb[s][5], cl[s]);
            } else {
                const PackedNode *q = nodes + cl[s];
                const float4 qa = __ldg(&q->a), qb = __ldg(&q->b), qc = __ldg(&q->c);
                const int4 qd = __ldg(&q->d);
                put(w, cnt++, qa.x, qa.y, qa.z, qa.w, qb.x, qb.y, qd.x);
                put(w, cnt++, qb.z, qb.w, qc.x, qc.y, qc.z, qc.w, qd.y);
            }
        }
        for (int i = cnt; i < 4; ++i)
            put(w, i, INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY, kEmpty);
        w.pad = make_int4(0, 0, 0, 0);
        WideNode *o = wide + x;
        __stcs(&o->lox, w.lox);
        __stcs(&o->loy, w.loy);
        __stcs(&o->loz, w.loz);
        __stcs(&o->hix, w.hix);
        __stcs(&o->hiy, w.hiy);
        __stcs(&o->hiz, w.hiz);
        __stcs(&o->link, w.link);
        __stcs(&o->pad, w.pad);
    }
}

__device__ __forceinline__ void cswap(float &da, int32_t &la, float &db, int32_t &lb) {
    const bool s = db < da;
    const float td = s ? db : da;
    const int32_t tl = s ? lb : la;
    db = s ? da : db;
    lb = s ? la : lb;
    da = td;
    la = tl;
}

}  // namespace

#ifndef LBVH_WIDE_SMEMSTACK
#define LBVH_WIDE_SMEMSTACK 12
#endif
#ifndef LBVH_WIDE_MINBLOCKS
#define LBVH_WIDE_MINBLOCKS 5
#endif

namespace {

template <int K>
__global__ void __launch_bounds__(256, (K <= 16 ? LBVH_WIDE_MINBLOCKS : 1))
knn_wide_kernel(const lbvh_tree t, const float *__restrict__ centers,
                const uint32_t *__restrict__ order, const uint32_t *__restrict__ qcodes,
                int64_t nq, const int64_t *__restrict__ offsets, int32_t *__restrict__ out_idx,
                float *__restrict__ out_dist, bool squared, uint32_t *status) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nq) return;
    const int64_t q = order ? (int64_t)__ldg(order + s) : s;
    const int64_t base = __ldg(offsets + q);
    const int kk = (int)(__ldg(offsets + q + 1) - base);
    if (kk <= 0) return;
    const float px = __ldg(centers + 3 * q), py = __ldg(centers + 3 * q + 1),
                pz = __ldg(centers + 3 * q + 2);
    const WideNode *__restrict__ wide = reinterpret_cast<const WideNode *>(t.nodes4);
    TopK<K> top;
    const float bound = (qcodes && t.leaf_codes) ? seed_bound<K>(t, __ldg(qcodes + s), kk, px, py, pz)
                                                 : __int_as_float(0x7FFFFFFF);
    top.init(kk, bound);
    constexpr int SMS = LBVH_WIDE_SMEMSTACK;
    __shared__ int32_t sst[(SMS > 0 ? SMS : 1) * 256];
    int32_t *const sbase = sst + threadIdx.x;
    int32_t lstack[kWideStack];
    int sp = 0;
    uint32_t fail = 0;
    auto push = [&](int32_t v) {
        if (sp < SMS)
            sbase[sp * 256] = v;
        else
            lstack[sp] = v;
        ++sp;
    };
    int32_t node = 0;
    while (true) {
        const WideNode *w = wide + node;
        float4 lx, ly, lz, hx, hy, hz, lkf, pad;
        ldg256(&w->lox, lx, ly);
        ldg256(&w->loz, lz, hx);
        ldg256(&w->hiy, hy, hz);
        ldg256(&w->link, lkf, pad);
        const int4 lk = make_int4(__float_as_int(lkf.x), __float_as_int(lkf.y),
                                  __float_as_int(lkf.z), __float_as_int(lkf.w));
        float d0 = box_dist_sq(px, py, pz, lx.x, ly.x, lz.x, hx.x, hy.x, hz.x);
        float d1 = box_dist_sq(px, py, pz, lx.y, ly.y, lz.y, hx.y, hy.y, hz.y);
        float d2 = box_dist_sq(px, py, pz, lx.z, ly.z, lz.z, hx.z, hy.z, hz.z);
        float d3 = box_dist_sq(px, py, pz, lx.w, ly.w, lz.w, hx.w, hy.w, hz.w);
        int32_t l0 = lk.x, l1 = lk.y, l2 = lk.z, l3 = lk.w;
        // nearest first: leaves are offered and internal entries descended /
        // pushed in ascending distance (empty slots sort last: +inf)
        if (l0 == kEmpty) d0 = INFINITY;
        if (l1 == kEmpty) d1 = INFINITY;
        if (l2 == kEmpty) d2 = INFINITY;
        if (l3 == kEmpty) d3 = INFINITY;
        cswap(d0, l0, d1, l1);
        cswap(d2, l2, d3, l3);
        cswap(d0, l0, d2, l2);
        cswap(d1, l1, d3, l3);
        cswap(d1, l1, d2, l2);
        // leaves (empty slots have l == -1: skipped as "leaf" with d = inf)
        if (l0 < 0 && l0 != kEmpty && !(d0 > top.worst())) top.offer(d0, l0 & 0x7FFFFFFF);
        if (l1 < 0 && l1 != kEmpty && !(d1 > top.worst())) top.offer(d1, l1 & 0x7FFFFFFF);
        if (l2 < 0 && l2 != kEmpty && !(d2 > top.worst())) top.offer(d2, l2 & 0x7FFFFFFF);
        if (l3 < 0 && l3 != kEmpty && !(d3 > top.worst())) top.offer(d3, l3 & 0x7FFFFFFF);
        const float wv = top.worst();
        const bool c0 = l0 >= 0 && !(d0 > wv), c1 = l1 >= 0 && !(d1 > wv);
        const bool c2 = l2 >= 0 && !(d2 > wv), c3 = l3 >= 0 && !(d3 > wv);
        const int nc = (int)c0 + (int)c1 + (int)c2 + (int)c3;
        if (sp + (nc > 0 ? nc - 1 : 0) > kWideStack) {
            fail = LBVH_FLAG_STACK_EXHAUSTED;
            break;
        }
        // push the farther candidates (farthest first), descend the nearest
        const int first = c0 ? 0 : c1 ? 1 : c2 ? 2 : c3 ? 3 : -1;
        if (c3 && first != 3) push(l3);
        if (c2 && first != 2) push(l2);
        if (c1 && first != 1) push(l1);
        int32_t next = first == 0 ? l0 : first == 1 ? l1 : first == 2 ? l2 : first == 3 ? l3 : -1;
        if (next < 0) {
            if (sp == 0) break;
            --sp;
            next = sp < SMS ? sbase[sp * 256] : lstack[sp];
        }
        node = next;
    }
    if (fail) atomicOr(status, fail);
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (j >= K - kk) {
            const int64_t o = base + (j - (K - kk));
            out_idx[o] = top.ordinal(j);
            out_dist[o] = squared ? top.dist(j) : __fsqrt_rn(top.dist(j));
        }
    }
}

}  // namespace

int wide_records(const lbvh_tree *t, void *nodes4, cudaStream_t stream) {
    if (!t || t->n < 2 || !t->nodes || !nodes4) return LBVH_ERR_INVALID_ARG;
    const int64_t ni = t->n - 1;
    unsigned g = div_up(ni, 256);
    g = g < kNumSMs * 16 ? g : kNumSMs * 16;
    wide_records_kernel<<<g, 256, 0, stream>>>((const PackedNode *)t->nodes, ni,
                                               (WideNode *)nodes4);
    count_launches(1);
    return check_launch();
}

// Launch the wide kNN for span <= K; returns -1 when not applicable.
int knn_wide(const lbvh_tree *t, const float *centers, const uint32_t *order,
             const uint32_t *qcodes, int64_t nq, const int64_t *offsets, int64_t max_span,
             int32_t *out_idx, float *out_dist, bool squared, uint32_t *status,
             cudaStream_t stream) {
    const unsigned g = div_up(nq, 256);
#define LBVH_WIDE_CASE(KV)                                                                  \
    if (max_span <= KV) {                                                                   \
        knn_wide_kernel<KV><<<g, 256, 0, stream>>>(*t, centers, order, qcodes, nq, offsets, \
                                                   out_idx, out_dist, squared, status);     \
        count_launches(1);                                                                  \
        return check_launch();                                                              \
    }
    LBVH_WIDE_CASE(4)
    LBVH_WIDE_CASE(8)
    LBVH_WIDE_CASE(10)
    LBVH_WIDE_CASE(16)
    LBVH_WIDE_CASE(32)
#undef LBVH_WIDE_CASE
    return -1;
}

}  // namespace lbvh
