/*
 * lbvh_oracle.c -- CPU restatement of the reference LBVH hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker and the CPU
 * baseline; it is never linked into, loaded by, or called from the product
 * path (paper_1908_11807_b200/). Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may use it.
 *
 * Every function restates one reference routine (paths relative to the
 * reference checkout, pkg/src/lbvh/):
 *   orc_morton_codes      morton.py:52-58 (_spread_bits), morton.py:68-91
 *   orc_sort_perm         tree.py:194 / traversal.py:159 (stable argsort)
 *   orc_generate_topology tree.py:40-44, tree.py:85-105,
 *                         _kernels.py:23-115 (_prefix, find_split, node_range,
 *                         build_topology)
 *   orc_refit             tree.py:108-119, _kernels.py:118-138
 *   orc_build             tree.py:177-209
 *   orc_spatial_pass      _kernels.py:146-228
 *   orc_spatial_buffered  _kernels.py:231-282
 *   orc_compact_rows      _kernels.py:285-290
 *   orc_knn_pass          _kernels.py:293-414
 *
 * Arithmetic follows the reference exactly: Morton normalisation in double,
 * box distances in float, unfused, accumulated x -> y -> z, skipping axes
 * with no gap.  Build with -O2 -ffp-contract=off so gcc never fuses.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_STACK_CAPACITY 64 /* _kernels.py:15 */

/* ------------------------------------------------------------------ */
/* Morton codes (morton.py:28-91)                                      */
/* ------------------------------------------------------------------ */

static inline uint32_t spread_bits(uint32_t v) {
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

static inline uint32_t grid_cell(double c, double lo, double ext) {
    double t = 0.0;
    if (ext > 0.0) t = (c - lo) / ext;  /* np.divide(..., where=extent > 0) */
    if (t < 0.0) t = 0.0;                /* np.clip(t, 0, 1) */
    if (t > 1.0) t = 1.0;
    uint32_t g = (uint32_t)(t * 1024.0); /* astype(uint32) truncates */
    return g < 1023u ? g : 1023u;        /* np.minimum(..., 1023) */
}

static inline uint32_t morton3(double x, double y, double z, const double smin[3],
                               const double ext[3]) {
    return (spread_bits(grid_cell(x, smin[0], ext[0])) << 2) |
           (spread_bits(grid_cell(y, smin[1], ext[1])) << 1) |
           spread_bits(grid_cell(z, smin[2], ext[2]));
}

void orc_morton_codes(const double *pts, int64_t n, const double *smin,
                      const double *smax, uint32_t *codes, int threads) {
    double ext[3] = {smax[0] - smin[0], smax[1] - smin[1], smax[2] - smin[2]};
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n; ++i)
        codes[i] = morton3(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], smin, ext);
}

/* ------------------------------------------------------------------ */
/* Stable argsort of 30-bit codes == sort of (code << 32 | index)      */
/* (tree.py:194, morton.py:102-119).  LSD radix, 3 x 11-bit digits.    */
/* ------------------------------------------------------------------ */

void orc_sort_perm(const uint32_t *codes, int64_t n, int64_t *perm) {
    uint32_t *k0 = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n ? n : 1));
    uint32_t *k1 = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)(n ? n : 1));
    int64_t *v1 = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    int64_t *v0 = perm;
    for (int64_t i = 0; i < n; ++i) { k0[i] = codes[i]; v0[i] = i; }
    uint32_t *ks = k0, *kd = k1;
    int64_t *vs = v0, *vd = v1;
    for (int shift = 0; shift < 32; shift += 11) {
        int64_t hist[2048];
        memset(hist, 0, sizeof(hist));
        for (int64_t i = 0; i < n; ++i) hist[(ks[i] >> shift) & 2047u]++;
        int64_t run = 0;
        for (int d = 0; d < 2048; ++d) { int64_t c = hist[d]; hist[d] = run; run += c; }
        for (int64_t i = 0; i < n; ++i) {
            int64_t p = hist[(ks[i] >> shift) & 2047u]++;
            kd[p] = ks[i];
            vd[p] = vs[i];
        }
        uint32_t *tk = ks; ks = kd; kd = tk;
        int64_t *tv = vs; vs = vd; vd = tv;
    }
    /* 3 passes: the result lives in (ks, vs) == (k1, v1) */
    if (vs != perm) memcpy(perm, vs, sizeof(int64_t) * (size_t)n);
    free(k0); free(k1); free(v1);
}

/* ------------------------------------------------------------------ */
/* Karras topology (_kernels.py:23-115, tree.py:40-44, 85-105)         */
/* ------------------------------------------------------------------ */

static inline int prefix(const int64_t *ak, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    uint64_t x = (uint64_t)(ak[i] ^ ak[j]);
    if (x == 0) return 64;
    return __builtin_clzll(x); /* 64 - bit_length(x) */
}

int64_t orc_find_split(const int64_t *ak, int64_t n, int64_t first, int64_t last) {
    int common = prefix(ak, n, first, last);
    int64_t split = first;
    int64_t step = last - first;
    for (;;) {
        step = (step + 1) >> 1;
        int64_t cand = split + step;
        if (cand < last && prefix(ak, n, first, cand) > common) split = cand;
        if (step <= 1) break;
    }
    return split;
}

void orc_node_range(const int64_t *ak, int64_t n, int64_t i, int64_t *first,
                    int64_t *last) {
    int64_t d = prefix(ak, n, i, i + 1) > prefix(ak, n, i, i - 1) ? 1 : -1;
    int floor_ = prefix(ak, n, i, i - d);
    int64_t span_max = 2;
    while (prefix(ak, n, i, i + span_max * d) > floor_) span_max <<= 1;
    int64_t span = 0;
    for (int64_t t = span_max >> 1; t >= 1; t >>= 1)
        if (prefix(ak, n, i, i + (span + t) * d) > floor_) span += t;
    int64_t j = i + span * d;
    if (i < j) { *first = i; *last = j; } else { *first = j; *last = i; }
}

void orc_augmented_keys(const uint32_t *sorted_codes, int64_t n, int64_t *ak) {
    for (int64_t i = 0; i < n; ++i) ak[i] = ((int64_t)sorted_codes[i] << 32) | i;
}

void orc_generate_topology(const uint32_t *sorted_codes, int64_t n, int32_t *left,
                           int32_t *right, int32_t *parent, int threads) {
    for (int64_t i = 0; i < n - 1; ++i) left[i] = right[i] = -1;
    for (int64_t i = 0; i < 2 * n - 1; ++i) parent[i] = -1;
    if (n < 2) return;
    int64_t *ak = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    orc_augmented_keys(sorted_codes, n, ak);
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n - 1; ++i) {
        int64_t first, last;
        orc_node_range(ak, n, i, &first, &last);
        int64_t g = orc_find_split(ak, n, first, last);
        int64_t lc = (g == first) ? (n - 1) + g : g;
        int64_t rc = (g + 1 == last) ? (n - 1) + (g + 1) : g + 1;
        left[i] = (int32_t)lc;
        right[i] = (int32_t)rc;
        parent[lc] = (int32_t)i;
        parent[rc] = (int32_t)i;
    }
    free(ak);
}

/* _kernels.py:118-138: serial walk, second arrival proceeds; numba min/max
 * keep the first argument on ties. */
void orc_refit(float *node_mins, float *node_maxs, const int32_t *left,
               const int32_t *right, const int32_t *parent, int64_t n) {
    if (n < 2) return;
    int32_t *visits = (int32_t *)calloc((size_t)(n - 1), sizeof(int32_t));
    for (int64_t leaf = n - 1; leaf < 2 * n - 1; ++leaf) {
        int64_t node = leaf;
        for (;;) {
            int64_t p = parent[node];
            if (p < 0) break;
            visits[p] += 1;
            if (visits[p] < 2) break;
            int64_t lc = left[p], rc = right[p];
            for (int a = 0; a < 3; ++a) {
                float l = node_mins[3 * lc + a], r = node_mins[3 * rc + a];
                node_mins[3 * p + a] = (r < l) ? r : l;
                l = node_maxs[3 * lc + a]; r = node_maxs[3 * rc + a];
                node_maxs[3 * p + a] = (r > l) ? r : l;
            }
            node = p;
        }
    }
    free(visits);
}

/* tree.py:177-209 for validated (n,3) mins/maxs. */
int orc_build(const float *mins, const float *maxs, int64_t n, float *node_mins,
              float *node_maxs, int32_t *left, int32_t *right, int32_t *leaf_obj,
              float *scene_min, float *scene_max, int threads) {
    if (n < 1) return 1; /* "empty scene" */
    for (int a = 0; a < 3; ++a) { scene_min[a] = mins[a]; scene_max[a] = maxs[a]; }
    for (int64_t i = 1; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            if (mins[3 * i + a] < scene_min[a]) scene_min[a] = mins[3 * i + a];
            if (maxs[3 * i + a] > scene_max[a]) scene_max[a] = maxs[3 * i + a];
        }
    double *cent = (double *)malloc(sizeof(double) * 3 * (size_t)n);
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < 3 * n; ++i) cent[i] = ((double)mins[i] + (double)maxs[i]) * 0.5;
    double smin[3] = {scene_min[0], scene_min[1], scene_min[2]};
    double smax[3] = {scene_max[0], scene_max[1], scene_max[2]};
    uint32_t *codes = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
    orc_morton_codes(cent, n, smin, smax, codes, threads);
    free(cent);
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    orc_sort_perm(codes, n, perm);
    uint32_t *sorted = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t p = 0; p < n; ++p) {
        int64_t o = perm[p];
        sorted[p] = codes[o];
        leaf_obj[p] = (int32_t)o;
        for (int a = 0; a < 3; ++a) {
            node_mins[3 * ((n - 1) + p) + a] = mins[3 * o + a];
            node_maxs[3 * ((n - 1) + p) + a] = maxs[3 * o + a];
        }
    }
    free(codes);
    free(perm);
    int32_t *parent = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * n - 1));
    orc_generate_topology(sorted, n, left, right, parent, threads);
    orc_refit(node_mins, node_maxs, left, right, parent, n);
    free(parent);
    free(sorted);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Traversal (_kernels.py:146-414)                                     */
/* ------------------------------------------------------------------ */

static inline float box_dist_sq(const float *mn, const float *mx, int64_t node,
                                float px, float py, float pz) {
    float d = 0.0f, t;
    float v = px, lo = mn[3 * node], hi = mx[3 * node];
    if (v < lo) { t = lo - v; d += t * t; } else if (v > hi) { t = v - hi; d += t * t; }
    v = py; lo = mn[3 * node + 1]; hi = mx[3 * node + 1];
    if (v < lo) { t = lo - v; d += t * t; } else if (v > hi) { t = v - hi; d += t * t; }
    v = pz; lo = mn[3 * node + 2]; hi = mx[3 * node + 2];
    if (v < lo) { t = lo - v; d += t * t; } else if (v > hi) { t = v - hi; d += t * t; }
    return d;
}

typedef struct {
    const float *node_mins, *node_maxs;
    const int32_t *left, *right, *leaf_obj;
    int64_t n;
} orc_tree;

/* _kernels.py:179-228.  counts int64 per query; store==0 counts, else fills
 * out[offsets[q] + j].  err[q] = 1 on stack exhaustion. */
void orc_spatial_pass(const orc_tree *tr, const float *centers, const float *radii,
                      const int64_t *order, int64_t nq, int64_t *counts,
                      const int64_t *offsets, int32_t *out, int store, uint8_t *err,
                      int threads) {
    const int64_t n = tr->n, internal = n - 1;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 256)
    for (int64_t s = 0; s < nq; ++s) {
        int64_t stack[ORC_STACK_CAPACITY];
        int64_t q = order[s];
        float px = centers[3 * q], py = centers[3 * q + 1], pz = centers[3 * q + 2];
        float r = radii[q];
        float r2 = r * r;
        int64_t base = store ? offsets[q] : 0;
        int64_t cnt = 0;
        if (n == 1) {
            if (box_dist_sq(tr->node_mins, tr->node_maxs, 0, px, py, pz) <= r2) {
                if (store) out[base] = tr->leaf_obj[0];
                cnt = 1;
            }
            counts[q] = cnt;
            continue;
        }
        int sp = 1;
        stack[0] = 0;
        int failed = 0;
        while (sp > 0 && !failed) {
            int64_t node = stack[--sp];
            for (int side = 0; side < 2; ++side) {
                int64_t child = side == 0 ? tr->left[node] : tr->right[node];
                if (box_dist_sq(tr->node_mins, tr->node_maxs, child, px, py, pz) <= r2) {
                    if (child >= internal) {
                        if (store) out[base + cnt] = tr->leaf_obj[child - internal];
                        cnt++;
                    } else {
                        if (sp >= ORC_STACK_CAPACITY) { err[q] = 1; failed = 1; break; }
                        stack[sp++] = child;
                    }
                }
            }
        }
        counts[q] = cnt;
    }
}

/* _kernels.py:231-282 */
void orc_spatial_buffered(const orc_tree *tr, const float *centers, const float *radii,
                          const int64_t *order, int64_t nq, int32_t *buf, int64_t cap,
                          int64_t *counts, uint8_t *overflow, uint8_t *err, int threads) {
    const int64_t n = tr->n, internal = n - 1;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 256)
    for (int64_t s = 0; s < nq; ++s) {
        int64_t stack[ORC_STACK_CAPACITY];
        int64_t q = order[s];
        float px = centers[3 * q], py = centers[3 * q + 1], pz = centers[3 * q + 2];
        float r = radii[q];
        float r2 = r * r;
        int64_t cnt = 0;
        if (n == 1) {
            if (box_dist_sq(tr->node_mins, tr->node_maxs, 0, px, py, pz) <= r2) {
                buf[q * cap] = tr->leaf_obj[0];
                cnt = 1;
            }
            counts[q] = cnt;
            continue;
        }
        int sp = 1;
        stack[0] = 0;
        int failed = 0;
        while (sp > 0 && !failed) {
            int64_t node = stack[--sp];
            for (int side = 0; side < 2; ++side) {
                int64_t child = side == 0 ? tr->left[node] : tr->right[node];
                if (box_dist_sq(tr->node_mins, tr->node_maxs, child, px, py, pz) <= r2) {
                    if (child >= internal) {
                        if (cnt >= cap) { overflow[q] = 1; failed = 1; break; }
                        buf[q * cap + cnt] = tr->leaf_obj[child - internal];
                        cnt++;
                    } else {
                        if (sp >= ORC_STACK_CAPACITY) { err[q] = 1; failed = 1; break; }
                        stack[sp++] = child;
                    }
                }
            }
        }
        counts[q] = cnt;
    }
}

/* _kernels.py:285-290 */
void orc_compact_rows(const int32_t *buf, int64_t cap, const int64_t *counts,
                      const int64_t *offsets, int32_t *out, int64_t nq, int threads) {
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t q = 0; q < nq; ++q)
        for (int64_t j = 0; j < counts[q]; ++j) out[offsets[q] + j] = buf[q * cap + j];
}

/* _kernels.py:293-325 */
static inline int worse(float d1, int32_t i1, float d2, int32_t i2) {
    return d1 > d2 || (d1 == d2 && i1 > i2);
}

static inline void sift_down(float *hd, int32_t *hi, int64_t size, int64_t pos) {
    for (;;) {
        int64_t child = 2 * pos + 1;
        if (child >= size) break;
        int64_t sib = child + 1;
        if (sib < size && worse(hd[sib], hi[sib], hd[child], hi[child])) child = sib;
        if (worse(hd[child], hi[child], hd[pos], hi[pos])) {
            float td = hd[pos]; hd[pos] = hd[child]; hd[child] = td;
            int32_t ti = hi[pos]; hi[pos] = hi[child]; hi[child] = ti;
            pos = child;
        } else break;
    }
}

static inline void sift_up(float *hd, int32_t *hi, int64_t pos) {
    while (pos > 0) {
        int64_t up = (pos - 1) >> 1;
        if (worse(hd[pos], hi[pos], hd[up], hi[up])) {
            float td = hd[pos]; hd[pos] = hd[up]; hd[up] = td;
            int32_t ti = hi[pos]; hi[pos] = hi[up]; hi[up] = ti;
            pos = up;
        } else break;
    }
}

/* _kernels.py:328-414 */
void orc_knn_pass(const orc_tree *tr, const float *centers, const int64_t *order,
                  int64_t nq, const int64_t *offsets, int32_t *out_idx, float *out_dist,
                  uint8_t *err, int threads) {
    const int64_t n = tr->n, internal = n - 1;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 256)
    for (int64_t s = 0; s < nq; ++s) {
        int64_t stack_node[ORC_STACK_CAPACITY];
        float stack_dist[ORC_STACK_CAPACITY];
        int64_t q = order[s];
        float px = centers[3 * q], py = centers[3 * q + 1], pz = centers[3 * q + 2];
        int64_t base = offsets[q];
        int64_t kk = offsets[q + 1] - base;
        float *hd = out_dist + base;
        int32_t *hi = out_idx + base;
        if (kk <= 0) continue;
        int64_t size = 0;
        if (n == 1) {
            hd[0] = sqrtf(box_dist_sq(tr->node_mins, tr->node_maxs, 0, px, py, pz));
            hi[0] = tr->leaf_obj[0];
            continue;
        }
        int sp = 1;
        stack_node[0] = 0;
        stack_dist[0] = box_dist_sq(tr->node_mins, tr->node_maxs, 0, px, py, pz);
        int failed = 0;
        while (sp > 0 && !failed) {
            --sp;
            int64_t node = stack_node[sp];
            float nd = stack_dist[sp];
            if (size == kk && nd > hd[0]) continue;
            int64_t cl = tr->left[node], cr = tr->right[node];
            float dl = box_dist_sq(tr->node_mins, tr->node_maxs, cl, px, py, pz);
            float dr = box_dist_sq(tr->node_mins, tr->node_maxs, cr, px, py, pz);
            int64_t fc, sc;
            float fd, sd;
            if (dl <= dr) { fc = cr; fd = dr; sc = cl; sd = dl; }
            else { fc = cl; fd = dl; sc = cr; sd = dr; }
            for (int pick = 0; pick < 2; ++pick) {
                int64_t child = pick == 0 ? fc : sc;
                float cd = pick == 0 ? fd : sd;
                if (size == kk && cd > hd[0]) continue;
                if (child >= internal) {
                    int32_t obj = tr->leaf_obj[child - internal];
                    if (size < kk) {
                        hd[size] = cd; hi[size] = obj; size++;
                        sift_up(hd, hi, size - 1);
                    } else if (worse(hd[0], hi[0], cd, obj)) {
                        hd[0] = cd; hi[0] = obj;
                        sift_down(hd, hi, kk, 0);
                    }
                } else {
                    if (sp >= ORC_STACK_CAPACITY) { err[q] = 1; failed = 1; break; }
                    stack_node[sp] = child;
                    stack_dist[sp] = cd;
                    sp++;
                }
            }
        }
        int64_t hs = size;
        while (hs > 1) {
            hs--;
            float td = hd[0]; hd[0] = hd[hs]; hd[hs] = td;
            int32_t ti = hi[0]; hi[0] = hi[hs]; hi[hs] = ti;
            sift_down(hd, hi, hs, 0);
        }
        for (int64_t j = 0; j < size; ++j) hd[j] = sqrtf(hd[j]);
    }
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------ */
/* 63-bit Morton build (north_star "30/63-bit"; NOT in the reference,  */
/* which is 30-bit only).  Same recipe at 21 bits/axis:   */
/* f64 normalise, clip, floor(t * 2^21) clamped to 2^21 - 1, x-major   */
/* interleave; Karras topology over (code, position) keys.  Parity of  */
/* this path is pinned only by this restatement (no reference output). */
/* ------------------------------------------------------------------ */

static inline uint64_t spread21(uint64_t v) {
    v &= 0x1FFFFFull;
    v = (v | (v << 32)) & 0x1F00000000FFFFull;
    v = (v | (v << 16)) & 0x1F0000FF0000FFull;
    v = (v | (v << 8)) & 0x100F00F00F00F00Full;
    v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

static inline uint64_t grid21(double c, double lo, double ext) {
    double t = 0.0;
    if (ext > 0.0) t = (c - lo) / ext;
    if (t < 0.0) t = 0.0;
    if (t > 1.0) t = 1.0;
    uint64_t g = (uint64_t)(t * 2097152.0);
    return g < 2097151ull ? g : 2097151ull;
}

void orc_morton63_codes(const double *pts, int64_t n, const double *smin, const double *smax,
                        uint64_t *codes, int threads) {
    double ext[3] = {smax[0] - smin[0], smax[1] - smin[1], smax[2] - smin[2]};
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n; ++i)
        codes[i] = (spread21(grid21(pts[3 * i], smin[0], ext[0])) << 2) |
                   (spread21(grid21(pts[3 * i + 1], smin[1], ext[1])) << 1) |
                   spread21(grid21(pts[3 * i + 2], smin[2], ext[2]));
}

static int cmp_code64(const void *a, const void *b) {
    const uint64_t *x = (const uint64_t *)a, *y = (const uint64_t *)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return x[1] < y[1] ? -1 : (x[1] > y[1]);
}

/* stable argsort of 64-bit codes == sort of (code, index) pairs */
void orc_sort_perm64(const uint64_t *codes, int64_t n, int64_t *perm) {
    uint64_t *kv = (uint64_t *)malloc(sizeof(uint64_t) * 2 * (size_t)(n ? n : 1));
    for (int64_t i = 0; i < n; ++i) { kv[2 * i] = codes[i]; kv[2 * i + 1] = (uint64_t)i; }
    qsort(kv, (size_t)n, 2 * sizeof(uint64_t), cmp_code64);
    for (int64_t i = 0; i < n; ++i) perm[i] = (int64_t)kv[2 * i + 1];
    free(kv);
}

static inline int prefix64(const uint64_t *c, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    if (c[i] != c[j]) return __builtin_clzll(c[i] ^ c[j]);
    return 64 + __builtin_clz((uint32_t)(i ^ j));
}

static int64_t find_split64(const uint64_t *c, int64_t n, int64_t first, int64_t last) {
    int common = prefix64(c, n, first, last);
    int64_t split = first, step = last - first;
    for (;;) {
        step = (step + 1) >> 1;
        int64_t cand = split + step;
        if (cand < last && prefix64(c, n, first, cand) > common) split = cand;
        if (step <= 1) break;
    }
    return split;
}

void orc_generate_topology64(const uint64_t *c, int64_t n, int32_t *left, int32_t *right,
                             int32_t *parent, int threads) {
    for (int64_t i = 0; i < n - 1; ++i) left[i] = right[i] = -1;
    for (int64_t i = 0; i < 2 * n - 1; ++i) parent[i] = -1;
    if (n < 2) return;
#pragma omp parallel for num_threads(threads) schedule(static)
    for (int64_t i = 0; i < n - 1; ++i) {
        int64_t d = prefix64(c, n, i, i + 1) > prefix64(c, n, i, i - 1) ? 1 : -1;
        int floor_ = prefix64(c, n, i, i - d);
        int64_t span_max = 2;
        while (prefix64(c, n, i, i + span_max * d) > floor_) span_max <<= 1;
        int64_t span = 0;
        for (int64_t t = span_max >> 1; t >= 1; t >>= 1)
            if (prefix64(c, n, i, i + (span + t) * d) > floor_) span += t;
        int64_t j = i + span * d;
        int64_t first = i < j ? i : j, last = i < j ? j : i;
        int64_t g = find_split64(c, n, first, last);
        int64_t lc = (g == first) ? (n - 1) + g : g;
        int64_t rc = (g + 1 == last) ? (n - 1) + (g + 1) : g + 1;
        left[i] = (int32_t)lc;
        right[i] = (int32_t)rc;
        parent[lc] = (int32_t)i;
        parent[rc] = (int32_t)i;
    }
}

int orc_build63(const float *mins, const float *maxs, int64_t n, float *node_mins,
                float *node_maxs, int32_t *left, int32_t *right, int32_t *leaf_obj,
                float *scene_min, float *scene_max, int threads) {
    if (n < 1) return 1;
    for (int a = 0; a < 3; ++a) { scene_min[a] = mins[a]; scene_max[a] = maxs[a]; }
    for (int64_t i = 1; i < n; ++i)
        for (int a = 0; a < 3; ++a) {
            if (mins[3 * i + a] < scene_min[a]) scene_min[a] = mins[3 * i + a];
            if (maxs[3 * i + a] > scene_max[a]) scene_max[a] = maxs[3 * i + a];
        }
    double *cent = (double *)malloc(sizeof(double) * 3 * (size_t)n);
    for (int64_t i = 0; i < 3 * n; ++i) cent[i] = ((double)mins[i] + (double)maxs[i]) * 0.5;
    double smin[3] = {scene_min[0], scene_min[1], scene_min[2]};
    double smax[3] = {scene_max[0], scene_max[1], scene_max[2]};
    uint64_t *codes = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    orc_morton63_codes(cent, n, smin, smax, codes, threads);
    free(cent);
    int64_t *perm = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
    orc_sort_perm64(codes, n, perm);
    uint64_t *sorted = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)n);
    for (int64_t p = 0; p < n; ++p) {
        int64_t o = perm[p];
        sorted[p] = codes[o];
        leaf_obj[p] = (int32_t)o;
        for (int a = 0; a < 3; ++a) {
            node_mins[3 * ((n - 1) + p) + a] = mins[3 * o + a];
            node_maxs[3 * ((n - 1) + p) + a] = maxs[3 * o + a];
        }
    }
    free(codes);
    free(perm);
    int32_t *parent = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * n - 1));
    orc_generate_topology64(sorted, n, left, right, parent, threads);
    orc_refit(node_mins, node_maxs, left, right, parent, n);
    free(parent);
    free(sorted);
    return 0;
}
