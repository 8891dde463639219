// datagen.cu -- the benchmark point clouds generated on the device, bit for
// bit the reference's numpy streams (pkg/src/lbvh/datasets.py:95-153; host
// restatement in paper_1908_11807_b200/datasets.py).  Harness only: clouds
// are never generated inside a timed region.
//
// numpy's PCG64 is the 128-bit LCG  s <- s*M + inc  with the XSL-RR output
// rotr64(hi(s) ^ lo(s), s >> 122) taken after the step; Generator.uniform(lo,
// hi) returns lo + (hi - lo) * ((x >> 11) * 2^-53).  Each thread jumps the LCG
// to its first draw (O(log i) advance, pcg_advance_lcg_128) and steps through
// its points; the initial (state, inc) come from numpy's SeedSequence on the
// host.

#include "common.cuh"
#include "internal.cuh"

namespace lbvh {
namespace {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 mk(uint64_t hi, uint64_t lo) { return ((u128)hi << 64) | lo; }

__device__ __forceinline__ u128 pcg_mult() {
    return mk(0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull);
}

__device__ u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

__device__ __forceinline__ double next_double(u128 &s, u128 inc) {
    s = s * pcg_mult() + inc;
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    const uint64_t r = (x >> rot) | (x << ((64u - rot) & 63u));
    return (double)(r >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ float clipf(float v, float lim) {
    return v < -lim ? -lim : (v > lim ? lim : v);
}

constexpr int kGenPts = 64;  // points per thread

// kind 0: cube filled (3 draws/pt), 1: cube hollow (2), 2: sphere hollow (3)
__global__ void __launch_bounds__(256)
cloud_kernel(int kind, int64_t p, double a, float lim, uint64_t st_hi, uint64_t st_lo,
             uint64_t inc_hi, uint64_t inc_lo, float *__restrict__ out, uint32_t *status) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i0 = t * kGenPts;
    if (i0 >= p) return;
    const int64_t i1 = (i0 + kGenPts < p) ? i0 + kGenPts : p;
    const int per = kind == 1 ? 2 : 3;
    const u128 inc = mk(inc_hi, inc_lo);
    u128 s = pcg_advance(mk(st_hi, st_lo), inc, (uint64_t)(i0 * per));
    const double lo = kind == 2 ? -1.0 : -a;
    const double range = kind == 2 ? 2.0 : __dsub_rn(a, -a);
    for (int64_t i = i0; i < i1; ++i) {
        if (kind == 0) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double v = __dadd_rn(lo, __dmul_rn(range, next_double(s, inc)));
                out[3 * i + c] = clipf(__double2float_rn(v), lim);
            }
        } else if (kind == 1) {
            const float u = __double2float_rn(__dadd_rn(lo, __dmul_rn(range, next_double(s, inc))));
            const float v = __double2float_rn(__dadd_rn(lo, __dmul_rn(range, next_double(s, inc))));
            const int f = (int)(i % 6);  // faces -x, +x, -y, +y, -z, +z
            const int axis = f >> 1;
            const float side = (f & 1) ? lim : -lim;
            float xyz[3];
            xyz[axis] = side;
            xyz[axis == 0 ? 1 : 0] = u;
            xyz[axis == 2 ? 1 : 2] = v;
#pragma unroll
            for (int c = 0; c < 3; ++c) out[3 * i + c] = clipf(xyz[c], lim);
        } else {
            double u[3];
#pragma unroll
            for (int c = 0; c < 3; ++c)
                u[c] = __dadd_rn(lo, __dmul_rn(range, next_double(s, inc)));
            const double ss = __dadd_rn(__dadd_rn(__dmul_rn(u[0], u[0]), __dmul_rn(u[1], u[1])),
                                        __dmul_rn(u[2], u[2]));
            const double nrm = __dsqrt_rn(ss);
            if (nrm < 1e-6) atomicOr(status, LBVH_FLAG_NONFINITE);  // numpy redraws: host path
#pragma unroll
            for (int c = 0; c < 3; ++c)
                out[3 * i + c] = __double2float_rn(__ddiv_rn(__dmul_rn(a, u[c]), nrm));
        }
    }
}

}  // namespace
}  // namespace lbvh

using namespace lbvh;

extern "C" int lbvh_generate_cloud(int kind, int64_t p, double a, float lim, uint64_t st_hi,
                                   uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, float *out,
                                   uint32_t *status, void *stream) {
    if (kind < 0 || kind > 2 || p < 0 || (p > 0 && (!out || !status)))
        return LBVH_ERR_INVALID_ARG;
    if (p == 0) return LBVH_OK;
    const int64_t threads = (p + kGenPts - 1) / kGenPts;
    cloud_kernel<<<div_up(threads, 256), 256, 0, (cudaStream_t)stream>>>(
        kind, p, a, lim, st_hi, st_lo, inc_hi, inc_lo, out, status);
    count_launches(1);
    return check_launch();
}
