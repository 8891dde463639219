// common.cuh -- shared device helpers for the sm_100a LBVH kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/lbvh_b200.h"

namespace lbvh {

constexpr int kStack = LBVH_STACK_CAPACITY;
constexpr uint32_t kLeafTag = 0x80000000u;
constexpr int kNumSMs = 148;  // B200

// Traversal layout of one internal node: both child boxes, interleaved per
// coordinate (left, right) so the two children's box distances run as packed
// f32x2 operations (child_dists), + both links.  64 bytes, 64-byte aligned
// (half an L2 line), read as two 256-bit loads.
//   a = {L.min.x, R.min.x, L.min.y, R.min.y}
//   b = {L.min.z, R.min.z, L.max.x, R.max.x}
//   c = {L.max.y, R.max.y, L.max.z, R.max.z}
//   d = {left link, right link, 0, 0}; a leaf link is obj | kLeafTag.
struct __align__(64) PackedNode {
    float4 a, b, c;
    int4 d;
};
static_assert(sizeof(PackedNode) == LBVH_NODE_BYTES, "packed node must be 64 B");

struct Box {
    float lo[3], hi[3];
};

// Reference box distance (_kernels.py:146-176): per axis the clamp gap,
// squared and accumulated x -> y -> z in fp32, every op round-to-nearest and
// unfused.  max(lo - v, v - hi, 0) equals the reference's branch: when v < lo
// the first term is the (positive, exactly rounded) gap, when v > hi the
// second is, otherwise both are <= 0; adding a +0 gap term is the identity,
// matching the reference's "skip axis".
__device__ __forceinline__ float gap(float v, float lo, float hi) {
    return fmaxf(fmaxf(__fsub_rn(lo, v), __fsub_rn(v, hi)), 0.0f);
}

__device__ __forceinline__ float box_dist_sq(float px, float py, float pz, float lx,
                                             float ly, float lz, float hx, float hy,
                                             float hz) {
    float tx = gap(px, lx, hx), ty = gap(py, ly, hy), tz = gap(pz, lz, hz);
    float d = __fmul_rn(tx, tx);
    d = __fadd_rn(d, __fmul_rn(ty, ty));
    d = __fadd_rn(d, __fmul_rn(tz, tz));
    return d;
}

__device__ __forceinline__ void pack_boxes(const Box &L, const Box &R, float4 &a, float4 &b,
                                           float4 &c) {
    a = make_float4(L.lo[0], R.lo[0], L.lo[1], R.lo[1]);
    b = make_float4(L.lo[2], R.lo[2], L.hi[0], R.hi[0]);
    c = make_float4(L.hi[1], R.hi[1], L.hi[2], R.hi[2]);
}

__device__ __forceinline__ void unpack_boxes(const float4 &a, const float4 &b, const float4 &c,
                                             Box &L, Box &R) {
    L.lo[0] = a.x; R.lo[0] = a.y; L.lo[1] = a.z; R.lo[1] = a.w;
    L.lo[2] = b.x; R.lo[2] = b.y; L.hi[0] = b.z; R.hi[0] = b.w;
    L.hi[1] = c.x; R.hi[1] = c.y; L.hi[2] = c.z; R.hi[2] = c.w;
}

// Packed fp32 pairs (sm_100 FADD2 / FMUL2): each lane rounds to nearest on
// its own, so a pair op is bit-identical to the two scalar ops.
__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(uint64_t v, float &lo, float &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t f2_sub(uint64_t x, uint64_t y) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
    return r;
}
__device__ __forceinline__ uint64_t f2_mul(uint64_t x, uint64_t y) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
    return r;
}

// box_dist_sq of both children of a packed record, as pair operations: the
// same roundings in the same order (per axis lo - v and v - hi, the clamp,
// then x^2, + y^2, + z^2), so dl / dr equal box_dist_sq bit for bit.
__device__ __forceinline__ void child_dists(float px, float py, float pz, const float4 &a,
                                            const float4 &b, const float4 &c, float &dl,
                                            float &dr) {
    const uint64_t vx = f2_pack(px, px), vy = f2_pack(py, py), vz = f2_pack(pz, pz);
    float l0, r0, l1, r1;
    f2_unpack(f2_sub(f2_pack(a.x, a.y), vx), l0, r0);
    f2_unpack(f2_sub(vx, f2_pack(b.z, b.w)), l1, r1);
    const uint64_t gx = f2_pack(fmaxf(fmaxf(l0, l1), 0.0f), fmaxf(fmaxf(r0, r1), 0.0f));
    f2_unpack(f2_sub(f2_pack(a.z, a.w), vy), l0, r0);
    f2_unpack(f2_sub(vy, f2_pack(c.x, c.y)), l1, r1);
    const uint64_t gy = f2_pack(fmaxf(fmaxf(l0, l1), 0.0f), fmaxf(fmaxf(r0, r1), 0.0f));
    f2_unpack(f2_sub(f2_pack(b.x, b.y), vz), l0, r0);
    f2_unpack(f2_sub(vz, f2_pack(c.z, c.w)), l1, r1);
    const uint64_t gz = f2_pack(fmaxf(fmaxf(l0, l1), 0.0f), fmaxf(fmaxf(r0, r1), 0.0f));
    // Squares as pairs, sums as scalar add.rn: ptxas 12.9 contracts
    // mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (even with --fmad=false), which
    // would round once instead of twice; a scalar add.rn is never contracted.
    float xl, xr, yl, yr, zl, zr;
    f2_unpack(f2_mul(gx, gx), xl, xr);
    f2_unpack(f2_mul(gy, gy), yl, yr);
    f2_unpack(f2_mul(gz, gz), zl, zr);
    dl = __fadd_rn(__fadd_rn(xl, yl), zl);
    dr = __fadd_rn(__fadd_rn(xr, yr), zr);
}

// Refit tie rules of numba's min/max (first argument wins ties,
// _kernels.py:136-137): matters only for signed zeros.
__device__ __forceinline__ float min_left(float l, float r) { return (r < l) ? r : l; }
__device__ __forceinline__ float max_left(float l, float r) { return (r > l) ? r : l; }

__device__ __forceinline__ void flag(uint32_t *status, uint32_t bits) {
    if (status) atomicOr(status, bits);
}

// Morton (morton.py:52-58, 68-91): f64 normalisation, correctly rounded.
__device__ __forceinline__ uint32_t spread_bits(uint32_t v) {
    v = (v | (v << 16)) & 0x030000FFu;
    v = (v | (v << 8)) & 0x0300F00Fu;
    v = (v | (v << 4)) & 0x030C30C3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__device__ __forceinline__ uint32_t grid_cell(double c, double lo, double ext) {
    double t = 0.0;
    if (ext > 0.0) t = __ddiv_rn(__dsub_rn(c, lo), ext);
    t = t < 0.0 ? 0.0 : t;
    t = t > 1.0 ? 1.0 : t;
    uint32_t g = (uint32_t)__double2uint_rz(__dmul_rn(t, 1024.0));
    return g < 1023u ? g : 1023u;
}

__device__ __forceinline__ uint32_t morton3(double x, double y, double z, const double *lo,
                                            const double *ext) {
    return (spread_bits(grid_cell(x, lo[0], ext[0])) << 2) |
           (spread_bits(grid_cell(y, lo[1], ext[1])) << 1) |
           spread_bits(grid_cell(z, lo[2], ext[2]));
}

// 63-bit codes (north_star "30/63-bit"; not in the reference):
// the same recipe at 21 bits per axis, so code63 >> 33 == the 30-bit code.
__device__ __forceinline__ uint64_t spread21(uint64_t v) {
    v &= 0x1FFFFFull;
    v = (v | (v << 32)) & 0x1F00000000FFFFull;
    v = (v | (v << 16)) & 0x1F0000FF0000FFull;
    v = (v | (v << 8)) & 0x100F00F00F00F00Full;
    v = (v | (v << 4)) & 0x10C30C30C30C30C3ull;
    v = (v | (v << 2)) & 0x1249249249249249ull;
    return v;
}

__device__ __forceinline__ uint64_t grid21(double c, double lo, double ext) {
    double t = 0.0;
    if (ext > 0.0) t = __ddiv_rn(__dsub_rn(c, lo), ext);
    t = t < 0.0 ? 0.0 : t;
    t = t > 1.0 ? 1.0 : t;
    uint64_t g = __double2ull_rz(__dmul_rn(t, 2097152.0));
    return g < 2097151ull ? g : 2097151ull;
}

__device__ __forceinline__ uint64_t morton63(double x, double y, double z, const double *lo,
                                             const double *ext) {
    return (spread21(grid21(x, lo[0], ext[0])) << 2) | (spread21(grid21(y, lo[1], ext[1])) << 1) |
           spread21(grid21(z, lo[2], ext[2]));
}

// 32 bytes in one read-only 256-bit load (sm_100: LDG.E.ENL2.256); p must
// be 32-byte aligned.
__device__ __forceinline__ void ldg256(const void *p, float4 &x, float4 &y) {
    asm("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w), "=f"(y.x), "=f"(y.y), "=f"(y.z), "=f"(y.w)
        : "l"(p));
}

// 32-byte store (sm_100 STG.E.ENL2.256): one full L2 sector per store.
__device__ __forceinline__ void stg256(void *p, float4 x, float4 y) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                 :: "l"(p), "f"(x.x), "f"(x.y), "f"(x.z), "f"(x.w), "f"(y.x), "f"(y.y),
                    "f"(y.z), "f"(y.w)
                 : "memory");
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// 16-byte shared-memory store / load the compiler may not move across fences
// or atomics (the hierarchy's in-CTA sibling hand-off).
__device__ __forceinline__ void st_shared_v4(void *p, float4 v) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("st.volatile.shared.v4.f32 [%0], {%1, %2, %3, %4};"
                 :: "r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 ld_shared_v4(const void *p) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    float4 v;
    asm volatile("ld.volatile.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
    return v;
}

// Plain 32-bit shared-memory accesses through a shared-window address (the
// kNN stack): volatile so they stay ordered with each other like the array
// accesses they replace.
__device__ __forceinline__ void st_shared_s32(uint32_t addr, int32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" :: "r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_shared_s32(uint32_t addr) {
    int32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}

// GPU-scope release+acquire read-modify-writes (no full membar).
__device__ __forceinline__ uint32_t atomic_exch_acq_rel(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.exch.b32 %0, [%1], %2;"
                 : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ uint32_t atomic_exch_release(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.release.gpu.global.exch.b32 %0, [%1], %2;"
                 : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

// Strong (relaxed, gpu-scope) loads: read at the point of coherence, never a
// stale L1 line.
__device__ __forceinline__ float ld_relaxed(const float *p) {
    float v;
    asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ float4 ld_relaxed(const float4 *p) {
    float4 v;
    asm volatile("ld.relaxed.gpu.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t atomic_add_acq_rel(uint32_t *p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;"
                 : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}

template <typename T>
__device__ __forceinline__ T ld_volatile(const T *p) {
    return *reinterpret_cast<const volatile T *>(p);
}

// Digit histograms of the sort's passes (8-bit digits from first_bit) built
// by the kernel that produces the keys: shared-memory counts per CTA, one
// global add per non-empty bin (sort_prepare / sort_pairs_prepared).
constexpr int kSortDigits = 256;
__device__ __forceinline__ void hist_accumulate(uint32_t (*s)[kSortDigits], uint32_t key,
                                                int first_bit, int passes) {
#pragma unroll
    for (int p = 0; p < 4; ++p)
        if (p < passes) atomicAdd(&s[p][(key >> (first_bit + 8 * p)) & (kSortDigits - 1)], 1u);
}
__device__ __forceinline__ void hist_flush(const uint32_t (*s)[kSortDigits], int passes,
                                           uint32_t *hist) {
    for (int i = threadIdx.x; i < passes * kSortDigits; i += blockDim.x) {
        const uint32_t c = s[i / kSortDigits][i % kSortDigits];
        if (c) atomicAdd(hist + i, c);
    }
}

inline unsigned int div_up(int64_t a, int64_t b) { return (unsigned int)((a + b - 1) / b); }

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-owned workspace.
struct Carve {
    char *base;
    size_t off, cap;
    __host__ Carve(void *p, size_t c) : base((char *)p), off(0), cap(c) {}
    template <typename T>
    __host__ T *take(size_t count) {
        size_t o = align_up(off);
        off = o + sizeof(T) * count;
        return (T *)(base + o);
    }
    __host__ bool ok() const { return off <= cap; }
};

}  // namespace lbvh
