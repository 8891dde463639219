// scan.cu -- single-pass exclusive scan producing CRS offsets.
//
// Replaces _exclusive_scan (reference traversal.py:173-176) for the spatial
// counts, and the kNN span computation spans = min(k_q, n) + scan
// (traversal.py:261-262).  Decoupled look-back: each 2048-element tile
// publishes its aggregate, then its inclusive prefix, in one 64-bit word
// (2 flag bits + 62-bit value).  Traffic: 4 B (or 8 B for ks) read + 8 B
// written per query.

#include "common.cuh"
#include "internal.cuh"

namespace lbvh {
namespace {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanThreads * kScanItems;
constexpr uint64_t kAgg = 1ull << 62;
constexpr uint64_t kPrefix = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

struct CountsIn {
    const int32_t *counts;
    __device__ __forceinline__ int64_t operator()(int64_t i, uint32_t &) const {
        return (int64_t)__ldcs(counts + i);
    }
};

struct KnnSpanIn {
    const int64_t *ks;
    int64_t k, n;
    __device__ __forceinline__ int64_t operator()(int64_t i, uint32_t &bad) const {
        int64_t kq = ks ? __ldcs(ks + i) : k;
        if (kq < 1) {
            bad = LBVH_FLAG_BAD_K;
            return 0;
        }
        return kq < n ? kq : n;
    }
};

template <class In>
__global__ void __launch_bounds__(kScanThreads)
scan_kernel(In in, int64_t n, int64_t *__restrict__ offsets, uint64_t *lookback,
            uint32_t *counter, int32_t *max_out, uint32_t *status) {
    __shared__ int64_t s_v[kScanTile + kScanTile / 32];
    __shared__ int64_t s_warp[kScanThreads / 32];
    __shared__ int64_t s_prefix;
    __shared__ uint32_t s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const int64_t base = tile * kScanTile;
    uint32_t bad = 0;
    int64_t vmax = 0;
    // Striped (coalesced) load into padded shared memory.
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int idx = j * kScanThreads + tid;
        int64_t i = base + idx;
        int64_t v = i < n ? in(i, bad) : 0;
        vmax = v > vmax ? v : vmax;
        s_v[idx + (idx >> 5)] = v;
    }
    __syncthreads();
    // Blocked: thread tid owns tile elements tid*kItems .. +kItems-1.
    int64_t x[kScanItems];
    int64_t sum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int idx = tid * kScanItems + j;
        x[j] = s_v[idx + (idx >> 5)];
        sum += x[j];
    }
    int64_t incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int64_t warp_off = 0, tile_total = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
        int64_t t = s_warp[w];
        warp_off += (w < warp) ? t : 0;
        tile_total += t;
    }
    // Publish the aggregate, then warp 0 walks back 32 predecessors per round
    // trip: the nearest lane holding an inclusive prefix ends the walk, the
    // lanes before it add their aggregates (tiles before 0 read as prefix 0).
    if (warp == 0) {
        uint64_t *slot = lookback + tile;
        int64_t excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch((unsigned long long *)slot, kPrefix | (uint64_t)tile_total);
        } else {
            if (lane == 0) atomicExch((unsigned long long *)slot, kAgg | (uint64_t)tile_total);
            int64_t t = tile - 1 - lane;
            while (true) {
                const uint64_t v = t >= 0 ? ld_volatile(lookback + t) : kPrefix;
                if (!__all_sync(0xFFFFFFFFu, (v & ~kValMask) != 0)) continue;  // not all published
                const uint32_t pm = __ballot_sync(0xFFFFFFFFu, (v & kPrefix) != 0);
                const int stop = pm ? __ffs(pm) - 1 : 31;
                int64_t part = lane <= stop ? (int64_t)(v & kValMask) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xFFFFFFFFu, part, o);
                excl += part;
                if (pm) break;
                t -= 32;
            }
            if (lane == 0)
                atomicExch((unsigned long long *)slot, kPrefix | (uint64_t)(excl + tile_total));
        }
        if (lane == 0) {
            s_prefix = excl;
            if (tile == 0) offsets[0] = 0;
        }
    }
    __syncthreads();
    // Inclusive results back through shared memory, then coalesced stores
    // to offsets[i + 1].
    int64_t run = s_prefix + warp_off + incl - sum;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        run += x[j];
        int idx = tid * kScanItems + j;
        s_v[idx + (idx >> 5)] = run;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        int idx = j * kScanThreads + tid;
        int64_t i = base + idx;
        if (i < n) offsets[i + 1] = s_v[idx + (idx >> 5)];
    }
    if (max_out || status) {
        bad = __reduce_or_sync(0xFFFFFFFFu, bad);
        int32_t m = (int32_t)vmax;
        m = __reduce_max_sync(0xFFFFFFFFu, m);
        if (lane == 0) {
            if (bad && status) atomicOr(status, bad);
            if (max_out) atomicMax(max_out, m);
        }
    }
}

__global__ void __launch_bounds__(256)
uniform_offsets_kernel(int64_t *__restrict__ offsets, int64_t nq, int64_t span,
                       int32_t *max_out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= nq;
         i += (int64_t)gridDim.x * blockDim.x)
        offsets[i] = i * span;
    if (max_out && blockIdx.x == 0 && threadIdx.x == 0) *max_out = (int32_t)span;
}

template <class In>
int launch_scan(In in, int64_t n, int64_t *offsets, int32_t *max_out, uint32_t *status,
                void *ws, size_t ws_bytes, cudaStream_t stream) {
    if (n < 0 || !offsets) return LBVH_ERR_INVALID_ARG;
    if (ws_bytes < scan_workspace_bytes(n)) return LBVH_ERR_WORKSPACE;
    if (n == 0) {
        cudaMemsetAsync(offsets, 0, sizeof(int64_t), stream);
        return check_launch();
    }
    int64_t tiles = (n + kScanTile - 1) / kScanTile;
    Carve c(ws, ws_bytes);
    uint64_t *lookback = c.take<uint64_t>(tiles);
    uint32_t *counter = c.take<uint32_t>(1);
    cudaMemsetAsync(c.base, 0, c.off, stream);
    if (max_out) cudaMemsetAsync(max_out, 0, sizeof(int32_t), stream);
    scan_kernel<In><<<(unsigned)tiles, kScanThreads, 0, stream>>>(in, n, offsets, lookback,
                                                                 counter, max_out, status); count_launches(1);
    return check_launch();
}

}  // namespace

size_t scan_workspace_bytes(int64_t n) {
    int64_t tiles = (n + kScanTile - 1) / kScanTile;
    return align_up(sizeof(uint64_t) * (size_t)(tiles > 0 ? tiles : 1)) + 512;
}

int scan_counts(const int32_t *counts, int64_t n, int64_t *offsets, void *ws, size_t ws_bytes,
                cudaStream_t stream) {
    if (n > 0 && !counts) return LBVH_ERR_INVALID_ARG;
    return launch_scan(CountsIn{counts}, n, offsets, nullptr, nullptr, ws, ws_bytes, stream);
}

int knn_offsets(const int64_t *ks, int64_t k, int64_t n_leaves, int64_t nq, int64_t *offsets,
                int32_t *max_span, uint32_t *status, void *ws, size_t ws_bytes,
                cudaStream_t stream) {
    if (n_leaves < 1) return LBVH_ERR_INVALID_ARG;
    if (!ks) {
        // uniform k: offsets[i] = i * min(k, n), no scan needed
        if (!offsets || nq < 0 || k < 1) return LBVH_ERR_INVALID_ARG;
        const int64_t span = k < n_leaves ? k : n_leaves;
        unsigned g = div_up(nq + 1, 256);
        g = g < kNumSMs * 16 ? g : kNumSMs * 16;
        uniform_offsets_kernel<<<g, 256, 0, stream>>>(offsets, nq, span, max_span); count_launches(1);
        return check_launch();
    }
    return launch_scan(KnnSpanIn{ks, k, n_leaves}, nq, offsets, max_span, status, ws, ws_bytes,
                       stream);
}

}  // namespace lbvh
