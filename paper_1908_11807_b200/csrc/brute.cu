// brute.cu -- brute-force neighbour search on the GPU (the reference's
// verification helpers, pkg/src/lbvh/oracle.py:18-70), O(n) per query.
//
// Same fp32 arithmetic as the reference: d = p - c per axis, then
// d0*d0 + d1*d1 + d2*d2 accumulated x -> y -> z, unfused (oracle.py:18-21);
// radius hit iff d^2 <= r*r; kNN keeps the k smallest (d^2, ordinal) pairs
// (oracle.py:35-45) and reports sqrt.  Points are streamed through shared
// memory in tiles shared by the CTA's queries.

#include "common.cuh"
#include "internal.cuh"
#include "topk.cuh"

namespace lbvh {
namespace {

constexpr int kBruteThreads = 128;
constexpr int kTilePts = 1024;

__device__ __forceinline__ float point_dist_sq(float px, float py, float pz, float cx, float cy,
                                               float cz) {
    const float dx = __fsub_rn(px, cx), dy = __fsub_rn(py, cy), dz = __fsub_rn(pz, cz);
    float d = __fmul_rn(dx, dx);
    d = __fadd_rn(d, __fmul_rn(dy, dy));
    return __fadd_rn(d, __fmul_rn(dz, dz));
}

__device__ __forceinline__ void load_tile(float *s, const float *__restrict__ pts, int64_t base,
                                          int64_t n) {
    const int64_t cnt = (n - base) < kTilePts ? (n - base) : kTilePts;
    for (int i = threadIdx.x; i < 3 * cnt; i += blockDim.x) s[i] = __ldg(pts + 3 * base + i);
}

template <int K>
__global__ void __launch_bounds__(kBruteThreads)
brute_knn_kernel(const float *__restrict__ pts, int64_t n, const float *__restrict__ centers,
                 int64_t nq, int kk, int32_t *__restrict__ out_idx, float *__restrict__ out_dist) {
    __shared__ float s_pts[3 * kTilePts];
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = q < nq;
    float cx = 0, cy = 0, cz = 0;
    if (live) {
        cx = __ldg(centers + 3 * q);
        cy = __ldg(centers + 3 * q + 1);
        cz = __ldg(centers + 3 * q + 2);
    }
    TopK<K> top;
    top.init(kk, __int_as_float(0x7FFFFFFF));
    for (int64_t base = 0; base < n; base += kTilePts) {
        __syncthreads();
        load_tile(s_pts, pts, base, n);
        __syncthreads();
        const int cnt = (int)((n - base) < kTilePts ? (n - base) : kTilePts);
        if (live)
            for (int i = 0; i < cnt; ++i) {
                const float d = point_dist_sq(s_pts[3 * i], s_pts[3 * i + 1], s_pts[3 * i + 2],
                                              cx, cy, cz);
                if (!(d > top.worst())) top.offer(d, (int32_t)(base + i));
            }
    }
    if (!live) return;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (j >= K - kk) {
            const int64_t o = q * kk + (j - (K - kk));
            out_idx[o] = top.ordinal(j);
            out_dist[o] = __fsqrt_rn(top.dist(j));
        }
    }
}

// any k: bounded max-heap in the output row (oracle semantics via the
// reference kernel's heap, _kernels.py:299-325)
__device__ __forceinline__ bool worse(float d1, int32_t i1, float d2, int32_t i2) {
    return d1 > d2 || (d1 == d2 && i1 > i2);
}

__global__ void __launch_bounds__(kBruteThreads)
brute_knn_heap_kernel(const float *__restrict__ pts, int64_t n, const float *__restrict__ centers,
                      int64_t nq, int64_t kk, int32_t *__restrict__ out_idx,
                      float *__restrict__ out_dist) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const float cx = __ldg(centers + 3 * q), cy = __ldg(centers + 3 * q + 1),
                cz = __ldg(centers + 3 * q + 2);
    float *hd = out_dist + q * kk;
    int32_t *hi = out_idx + q * kk;
    int64_t size = 0;
    for (int64_t i = 0; i < n; ++i) {
        const float d = point_dist_sq(__ldg(pts + 3 * i), __ldg(pts + 3 * i + 1),
                                      __ldg(pts + 3 * i + 2), cx, cy, cz);
        const int32_t id = (int32_t)i;
        int64_t pos;
        if (size < kk) {
            pos = size++;
            hd[pos] = d;
            hi[pos] = id;
            while (pos > 0) {  // sift up
                const int64_t up = (pos - 1) >> 1;
                if (!worse(hd[pos], hi[pos], hd[up], hi[up])) break;
                float td = hd[pos]; hd[pos] = hd[up]; hd[up] = td;
                int32_t ti = hi[pos]; hi[pos] = hi[up]; hi[up] = ti;
                pos = up;
            }
        } else if (worse(hd[0], hi[0], d, id)) {
            hd[0] = d;
            hi[0] = id;
            pos = 0;
            while (true) {  // sift down
                int64_t c = 2 * pos + 1;
                if (c >= kk) break;
                if (c + 1 < kk && worse(hd[c + 1], hi[c + 1], hd[c], hi[c])) ++c;
                if (!worse(hd[c], hi[c], hd[pos], hi[pos])) break;
                float td = hd[pos]; hd[pos] = hd[c]; hd[c] = td;
                int32_t ti = hi[pos]; hi[pos] = hi[c]; hi[c] = ti;
                pos = c;
            }
        }
    }
    for (int64_t hs = size; hs > 1;) {  // heap-sort ascending
        --hs;
        float td = hd[0]; hd[0] = hd[hs]; hd[hs] = td;
        int32_t ti = hi[0]; hi[0] = hi[hs]; hi[hs] = ti;
        int64_t pos = 0;
        while (true) {
            int64_t c = 2 * pos + 1;
            if (c >= hs) break;
            if (c + 1 < hs && worse(hd[c + 1], hi[c + 1], hd[c], hi[c])) ++c;
            if (!worse(hd[c], hi[c], hd[pos], hi[pos])) break;
            float t2 = hd[pos]; hd[pos] = hd[c]; hd[c] = t2;
            int32_t t3 = hi[pos]; hi[pos] = hi[c]; hi[c] = t3;
            pos = c;
        }
    }
    for (int64_t j = 0; j < size; ++j) hd[j] = __fsqrt_rn(hd[j]);
}

template <bool FILL>
__global__ void __launch_bounds__(kBruteThreads)
brute_radius_kernel(const float *__restrict__ pts, int64_t n, const float *__restrict__ centers,
                    const float *__restrict__ radii, float radius, int64_t nq,
                    int32_t *__restrict__ counts, const int64_t *__restrict__ offsets,
                    int32_t *__restrict__ out) {
    __shared__ float s_pts[3 * kTilePts];
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool live = q < nq;
    float cx = 0, cy = 0, cz = 0, r2 = 0;
    int64_t base_out = 0;
    if (live) {
        cx = __ldg(centers + 3 * q);
        cy = __ldg(centers + 3 * q + 1);
        cz = __ldg(centers + 3 * q + 2);
        const float r = radii ? __ldg(radii + q) : radius;
        r2 = __fmul_rn(r, r);
        if (FILL) base_out = __ldg(offsets + q);
    }
    int32_t cnt_hits = 0;
    for (int64_t base = 0; base < n; base += kTilePts) {
        __syncthreads();
        load_tile(s_pts, pts, base, n);
        __syncthreads();
        const int cnt = (int)((n - base) < kTilePts ? (n - base) : kTilePts);
        if (live)
            for (int i = 0; i < cnt; ++i) {
                const float d = point_dist_sq(s_pts[3 * i], s_pts[3 * i + 1], s_pts[3 * i + 2],
                                              cx, cy, cz);
                if (d <= r2) {
                    if (FILL) out[base_out + cnt_hits] = (int32_t)(base + i);
                    ++cnt_hits;
                }
            }
    }
    if (live && !FILL) counts[q] = cnt_hits;
}

}  // namespace

int brute_knn(const float *pts, int64_t n, const float *centers, int64_t nq, int64_t k,
              int32_t *out_idx, float *out_dist, cudaStream_t stream) {
    if (n < 1 || nq < 0 || k < 1) return LBVH_ERR_INVALID_ARG;
    if (nq == 0) return LBVH_OK;
    if (!pts || !centers || !out_idx || !out_dist) return LBVH_ERR_INVALID_ARG;
    if (n >= LBVH_MAX_ITEMS || nq >= LBVH_MAX_ITEMS) return LBVH_ERR_TOO_LARGE;
    const int64_t kk = k < n ? k : n;
    const unsigned g = div_up(nq, kBruteThreads);
#define LBVH_BRUTE_CASE(KV)                                                                  \
    if (kk <= KV) {                                                                          \
        brute_knn_kernel<KV><<<g, kBruteThreads, 0, stream>>>(pts, n, centers, nq, (int)kk, \
                                                              out_idx, out_dist);           \
        count_launches(1);                                                                   \
        return check_launch();                                                               \
    }
    LBVH_BRUTE_CASE(4)
    LBVH_BRUTE_CASE(16)
    LBVH_BRUTE_CASE(32)
#undef LBVH_BRUTE_CASE
    brute_knn_heap_kernel<<<g, kBruteThreads, 0, stream>>>(pts, n, centers, nq, kk, out_idx,
                                                           out_dist);
    count_launches(1);
    return check_launch();
}

int brute_radius(const float *pts, int64_t n, const float *centers, const float *radii,
                 float radius, int64_t nq, int32_t *counts, const int64_t *offsets, int32_t *out,
                 cudaStream_t stream) {
    if (n < 0 || nq < 0) return LBVH_ERR_INVALID_ARG;
    if (nq == 0) return LBVH_OK;
    if ((n > 0 && !pts) || !centers) return LBVH_ERR_INVALID_ARG;
    if (n >= LBVH_MAX_ITEMS || nq >= LBVH_MAX_ITEMS) return LBVH_ERR_TOO_LARGE;
    const unsigned g = div_up(nq, kBruteThreads);
    if (offsets) {
        if (!out) return LBVH_ERR_INVALID_ARG;
        brute_radius_kernel<true><<<g, kBruteThreads, 0, stream>>>(pts, n, centers, radii, radius,
                                                                   nq, nullptr, offsets, out);
    } else {
        if (!counts) return LBVH_ERR_INVALID_ARG;
        brute_radius_kernel<false><<<g, kBruteThreads, 0, stream>>>(
            pts, n, centers, radii, radius, nq, counts, nullptr, nullptr);
    }
    count_launches(1);
    return check_launch();
}

}  // namespace lbvh
