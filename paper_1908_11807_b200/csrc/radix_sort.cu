// radix_sort.cu -- stable LSD radix sort of (key, u32 value) pairs.
//
// Replaces np.argsort(codes, kind="stable") (reference tree.py:194,
// traversal.py:159): sorting (code, index) pairs with a stable LSD sort gives
// exactly the stable argsort.  One-sweep design (Adinets & Merrill): one
// upfront pass builds the digit histograms of every digit position, then each
// digit pass is a single kernel that ranks a tile in shared memory, resolves
// its global offsets with a decoupled look-back over preceding tiles and
// scatters.  8-bit digits: 30-bit Morton keys take 4 passes (u32 keys,
// 4096-key tiles), 63-bit keys 8 passes (u64 keys, 2048-key tiles).
//
// HBM traffic per pass: (sizeof key + 4) B read + the same written per pair.

#include "common.cuh"
#include "internal.cuh"

namespace lbvh {
namespace {

constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
#ifndef LBVH_SORT_ITEMS
#define LBVH_SORT_ITEMS 16
#endif
// Measured at 1e7: ballot ranking + 4 CTAs/SM (64
// registers) 9.5 % faster builds than MATCH.ANY ranking at 3 CTAs/SM; the
// look-back reads W = 8 predecessors per round trip (0.339 ms vs 0.382 at
// W = 1, 0.353 at 16, 0.40 at 32); a tile publishes its digit counts right
// after its loads, before ranking (0.339 vs 0.398 ms); the histogram pass is a
// grid-stride loop at 2 CTAs/SM (21.7 vs 33 us for one CTA per 8192 keys).
#ifndef LBVH_SORT_MINBLOCKS
#define LBVH_SORT_MINBLOCKS 4
#endif
#ifndef LBVH_SORT_LOOKBACK_W
#define LBVH_SORT_LOOKBACK_W 8
#endif
constexpr int kHistCtasPerSm = 2;

template <typename KeyT>
struct SortCfg {
    static constexpr int kItems = sizeof(KeyT) == 4 ? LBVH_SORT_ITEMS : 8;
    static constexpr int kTile = kSortThreads * kItems;
    static constexpr int kMaxPasses = sizeof(KeyT) == 4 ? 4 : 8;
};

constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPrefix = 2u << 30;
constexpr uint32_t kCountMask = (1u << 30) - 1;

constexpr int kHistThreads = 512;
constexpr int kHistItems = 16;

// Digit histograms of every pass in one read of the keys.
template <typename KeyT>
__global__ void __launch_bounds__(kHistThreads)
histogram_kernel(const KeyT *__restrict__ keys, int64_t n, int passes, int first_bit,
                 uint32_t *__restrict__ hist) {
    constexpr int P = SortCfg<KeyT>::kMaxPasses;
    __shared__ uint32_t s_hist[P][kRadix];
    for (int i = threadIdx.x; i < P * kRadix; i += blockDim.x) (&s_hist[0][0])[i] = 0;
    __syncthreads();
    // grid-stride over 8192-key chunks, the chunk's loads issued together;
    // a grid of a few CTAs per SM keeps the final global atomics few
    for (int64_t base = (int64_t)blockIdx.x * kHistThreads * kHistItems; base < n;
         base += (int64_t)gridDim.x * kHistThreads * kHistItems) {
        KeyT k[kHistItems];
#pragma unroll
        for (int j = 0; j < kHistItems; ++j) {
            const int64_t i = base + (int64_t)j * kHistThreads + threadIdx.x;
            k[j] = i < n ? __ldcs(keys + i) : (KeyT)0;
        }
#pragma unroll
        for (int j = 0; j < kHistItems; ++j) {
            if (base + (int64_t)j * kHistThreads + threadIdx.x >= n) break;
#pragma unroll
            for (int p = 0; p < P; ++p)
                if (p < passes)
                    atomicAdd(&s_hist[p][(uint32_t)(k[j] >> (first_bit + p * kRadixBits)) &
                                         (kRadix - 1)],
                              1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
        uint32_t c = (&s_hist[0][0])[i];
        if (c) atomicAdd(hist + i, c);
    }
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// One digit pass.  Tiles are claimed in order through `tile_counter`, so a
// tile only ever waits on tiles already owned by running CTAs.
template <typename KeyT, bool IOTA>
__global__ void __launch_bounds__(kSortThreads, sizeof(KeyT) == 4 ? LBVH_SORT_MINBLOCKS : 1)
onesweep_kernel(const KeyT *__restrict__ keys_in, const uint32_t *__restrict__ vals_in,
                KeyT *__restrict__ keys_out, uint32_t *__restrict__ vals_out, int64_t n,
                int shift, const uint32_t *__restrict__ hist, uint32_t *lookback,
                uint32_t *tile_counter) {
    constexpr int kItems = SortCfg<KeyT>::kItems;
    constexpr int kTile = SortCfg<KeyT>::kTile;
    __shared__ KeyT s_keys[kTile];
    __shared__ uint32_t s_vals[kTile];
    __shared__ uint32_t s_warp[kSortWarps][kRadix];  // counts -> warp exclusive offsets
    __shared__ uint32_t s_local[kRadix];             // digit start within the tile
    __shared__ uint32_t s_global[kRadix];            // global dest of tile position 0 of digit
    __shared__ uint32_t s_scan[kSortWarps];
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_cnt[kRadix];

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;

    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    for (int i = tid; i < kSortWarps * kRadix; i += kSortThreads) (&s_warp[0][0])[i] = 0;
    s_cnt[tid] = 0;
    __syncthreads();
    const uint32_t tile = s_tile;
    // 32-bit positions (sorts hold < 2^30 pairs): single-instruction index math
    const uint32_t nn = (uint32_t)n;
    const uint32_t tile_base = tile * kTile;
    const uint32_t warp_base = tile_base + warp * 32 * kItems;

    // Warp-striped load: item j of a lane sits at warp_base + j*32 + lane, so
    // (j, lane) order is position order and the ranking below is stable.
    KeyT key[kItems];
    uint32_t val[kItems], rank[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const uint32_t i = warp_base + j * 32 + lane;
        const bool ok = i < nn;
        key[j] = ok ? __ldcs(keys_in + i) : ~(KeyT)0;  // pads sort last
        // IOTA: no value array, the input values are the positions (argsort)
        val[j] = ok ? (IOTA ? (uint32_t)i : __ldcs(vals_in + i)) : 0u;
    }
#pragma unroll
    for (int j = 0; j < kItems; ++j) atomicAdd(&s_cnt[(uint32_t)(key[j] >> shift) & (kRadix - 1)], 1u);
    __syncthreads();
    atomicExch(lookback + (size_t)tile * kRadix + tid,
               (tile == 0 ? kFlagPrefix : kFlagAgg) | s_cnt[tid]);
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        uint32_t d = (uint32_t)(key[j] >> shift) & (kRadix - 1);
        // lanes holding the same digit: AND of one ballot per digit bit
        // (independent votes, no MATCH.ANY latency chain)
        uint32_t peers = 0xFFFFFFFFu;
#pragma unroll
        for (int b = 0; b < kRadixBits; ++b) {
            const uint32_t bb = __ballot_sync(0xFFFFFFFFu, (d >> b) & 1u);
            peers &= ((d >> b) & 1u) ? bb : ~bb;
        }
        // every peer reads the running count; the highest peer bumps it
        const uint32_t before = s_warp[warp][d];
        __syncwarp();
        if ((peers >> lane) == 1u) s_warp[warp][d] = before + __popc(peers);
        rank[j] = before + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();

    // Thread tid owns digit tid: exclusive scan over warps, tile total.
    const uint32_t d = tid;
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) {
        uint32_t c = s_warp[w][d];
        s_warp[w][d] = total;
        total += c;
    }
    // (the tile aggregate was published right after the loads)
    uint32_t *my_slot = lookback + (size_t)tile * kRadix + d;

    // Block-wide exclusive scan of digit totals -> tile-local digit starts.
    uint32_t incl = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_scan[warp] = incl;
    __syncthreads();
    uint32_t warp_prefix = 0;
#pragma unroll
    for (int w = 0; w < kSortWarps; ++w) warp_prefix += (w < warp) ? s_scan[w] : 0u;
    const uint32_t local_start = warp_prefix + incl - total;
    s_local[d] = local_start;

    // Decoupled look-back for digit d.
    uint32_t excl = 0;
    if (tile > 0) {
        int64_t t = (int64_t)tile - 1;
        // W predecessors per round trip: the loads are independent, so a walk
        // over aggregates costs one L2 latency per W tiles instead of per tile
        constexpr int W = LBVH_SORT_LOOKBACK_W;
        bool done = false;
        while (!done) {
            uint32_t v[W];
#pragma unroll
            for (int i = 0; i < W; ++i)
                v[i] = (t - i >= 0) ? ld_volatile(lookback + (size_t)(t - i) * kRadix + d)
                                    : kFlagPrefix;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                if (done) break;
                if ((v[i] & ~kCountMask) == 0) break;  // not yet published: re-poll from t
                excl += v[i] & kCountMask;
                --t;
                if (v[i] & kFlagPrefix) done = true;
            }
        }
        atomicExch(my_slot, kFlagPrefix | (excl + total));
    }
    s_global[d] = hist[d] + excl - local_start;  // wraps back into range at use
    __syncthreads();

    // Scatter into shared memory in tile-sorted order.
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        uint32_t dj = (uint32_t)(key[j] >> shift) & (kRadix - 1);
        uint32_t pos = s_local[dj] + s_warp[warp][dj] + rank[j];
        s_keys[pos] = key[j];
        s_vals[pos] = val[j];
    }
    __syncthreads();

    // Pads (all-ones keys, positions >= n) are last in tile order.
    const uint32_t valid = (nn - tile_base) < (uint32_t)kTile ? (nn - tile_base) : (uint32_t)kTile;
#pragma unroll 4
    for (int i = tid; i < kTile; i += kSortThreads) {
        if ((uint32_t)i < valid) {
            const KeyT k = s_keys[i];
            const uint32_t dst = s_global[(uint32_t)(k >> shift) & (kRadix - 1)] + (uint32_t)i;
            keys_out[dst] = k;
            vals_out[dst] = s_vals[i];
        }
    }
}

__global__ void exclusive_hist_kernel(uint32_t *hist, int passes) {
    // One warp per pass: exclusive scan of 256 digit counts in place.
    int p = blockIdx.x;
    if (p >= passes) return;
    uint32_t *h = hist + p * kRadix;
    int lane = threadIdx.x;
    uint32_t c[8];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        c[j] = h[lane * 8 + j];
        s += c[j];
    }
    uint32_t incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
    }
    uint32_t run = incl - s;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        h[lane * 8 + j] = run;
        run += c[j];
    }
}

template <typename KeyT>
size_t sort_ws_bytes(int64_t n) {
    using C = SortCfg<KeyT>;
    int64_t tiles = (n + C::kTile - 1) / C::kTile;
    size_t b = 0;
    b += align_up(sizeof(KeyT) * (size_t)n) + align_up(sizeof(uint32_t) * (size_t)n);
    b += align_up(sizeof(uint32_t) * C::kMaxPasses * kRadix);                // hist
    b += align_up(sizeof(uint32_t) * C::kMaxPasses * (size_t)tiles * kRadix);  // look-back
    b += align_up(sizeof(uint32_t) * C::kMaxPasses);                         // counters
    return b + 256;
}

// from_alt: the input pairs were written to the workspace's ping-pong buffers
// (sort_alt_buffers) -- with an odd pass count the result then lands in
// (keys, vals) without the final device copies.
// hist_given: sort_prepare() zeroed the state and a producer kernel filled the
// digit histograms; iota: the input values are the positions 0..n-1 (not read).
template <typename KeyT>
int sort_impl(KeyT *keys, uint32_t *vals, int64_t n, int key_bits, void *ws, size_t ws_bytes,
              cudaStream_t stream, int first_bit, bool from_alt = false, bool hist_given = false,
              bool iota = false) {
    using C = SortCfg<KeyT>;
    if (n <= 1) {  // nothing to order; the pair may still have to land in place
        if (n == 1 && from_alt) {
            Carve c(ws, ws_bytes);
            KeyT *k_alt = c.take<KeyT>(n);
            uint32_t *v_alt = c.take<uint32_t>(n);
            cudaMemcpyAsync(keys, k_alt, sizeof(KeyT), cudaMemcpyDeviceToDevice, stream);
            if (!iota) cudaMemcpyAsync(vals, v_alt, 4, cudaMemcpyDeviceToDevice, stream);
        }
        if (n == 1 && iota) cudaMemsetAsync(vals, 0, 4, stream);
        return check_launch();
    }
    if (n >= LBVH_MAX_ITEMS) return LBVH_ERR_TOO_LARGE;
    if (key_bits < 1 || key_bits > (int)(8 * sizeof(KeyT)) || first_bit < 0 ||
        first_bit >= key_bits)
        return LBVH_ERR_INVALID_ARG;
    if (ws_bytes < sort_ws_bytes<KeyT>(n)) return LBVH_ERR_WORKSPACE;
    const int passes = (key_bits - first_bit + kRadixBits - 1) / kRadixBits;
    const int64_t tiles = (n + C::kTile - 1) / C::kTile;
    Carve c(ws, ws_bytes);
    KeyT *k_alt = c.take<KeyT>(n);
    uint32_t *v_alt = c.take<uint32_t>(n);
    // hist, look-back and counters are contiguous so one memset clears them.
    size_t zero_begin = align_up(c.off);
    uint32_t *hist = c.take<uint32_t>(C::kMaxPasses * kRadix);
    uint32_t *lookback = c.take<uint32_t>((size_t)C::kMaxPasses * tiles * kRadix);
    uint32_t *counters = c.take<uint32_t>(C::kMaxPasses);
    size_t zero_end = c.off;
    if (!hist_given) cudaMemsetAsync(c.base + zero_begin, 0, zero_end - zero_begin, stream);

    unsigned hist_blocks = div_up(n, (int64_t)kHistThreads * kHistItems);
    if (hist_blocks > (unsigned)(kNumSMs * kHistCtasPerSm)) hist_blocks = kNumSMs * kHistCtasPerSm;
    KeyT *ks = keys, *kd = k_alt;
    uint32_t *vs = vals, *vd = v_alt;
    if (from_alt) {
        ks = k_alt; kd = keys;
        vs = v_alt; vd = vals;
    }
    if (!hist_given) {
        histogram_kernel<KeyT><<<hist_blocks, kHistThreads, 0, stream>>>(ks, n, passes, first_bit,
                                                                          hist);
        count_launches(1);
    }
    exclusive_hist_kernel<<<passes, 32, 0, stream>>>(hist, passes);
    count_launches(1);

    for (int p = 0; p < passes; ++p) {
        if (iota && p == 0)
            onesweep_kernel<KeyT, true><<<(unsigned)tiles, kSortThreads, 0, stream>>>(
                ks, nullptr, kd, vd, n, first_bit, hist, lookback, counters);
        else
            onesweep_kernel<KeyT, false><<<(unsigned)tiles, kSortThreads, 0, stream>>>(
                ks, vs, kd, vd, n, first_bit + p * kRadixBits, hist + p * kRadix,
                lookback + (size_t)p * tiles * kRadix, counters + p);
        count_launches(1);
        KeyT *tk = ks; ks = kd; kd = tk;
        uint32_t *tv = vs; vs = vd; vd = tv;
    }
    if (ks != keys) {
        cudaMemcpyAsync(keys, ks, sizeof(KeyT) * n, cudaMemcpyDeviceToDevice, stream);
        cudaMemcpyAsync(vals, vs, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, stream);
    }
    return check_launch();
}

}  // namespace

size_t sort_workspace_bytes(int64_t n) { return sort_ws_bytes<uint32_t>(n); }
size_t sort64_workspace_bytes(int64_t n) { return sort_ws_bytes<uint64_t>(n); }

int sort_pairs(uint32_t *keys, uint32_t *vals, int64_t n, int key_bits, void *ws,
               size_t ws_bytes, cudaStream_t stream, int first_bit) {
    return sort_impl<uint32_t>(keys, vals, n, key_bits, ws, ws_bytes, stream, first_bit);
}

void sort_alt_buffers(void *ws, size_t ws_bytes, int64_t n, uint32_t **k_alt, uint32_t **v_alt) {
    Carve c(ws, ws_bytes);
    *k_alt = c.take<uint32_t>(n);
    *v_alt = c.take<uint32_t>(n);
}

int sort_pass_count(int key_bits, int first_bit) {
    return (key_bits - first_bit + kRadixBits - 1) / kRadixBits;
}

int sort_pairs_from_alt(uint32_t *keys, uint32_t *vals, int64_t n, int key_bits, void *ws,
                        size_t ws_bytes, cudaStream_t stream, int first_bit) {
    return sort_impl<uint32_t>(keys, vals, n, key_bits, ws, ws_bytes, stream, first_bit, true);
}

uint32_t *sort_prepare(void *ws, size_t ws_bytes, int64_t n, cudaStream_t stream) {
    using C = SortCfg<uint32_t>;
    const int64_t tiles = (n + C::kTile - 1) / C::kTile;
    Carve c(ws, ws_bytes);
    c.take<uint32_t>(n);
    c.take<uint32_t>(n);
    const size_t zero_begin = align_up(c.off);
    uint32_t *hist = c.take<uint32_t>(C::kMaxPasses * kRadix);
    c.take<uint32_t>((size_t)C::kMaxPasses * tiles * kRadix);
    c.take<uint32_t>(C::kMaxPasses);
    cudaMemsetAsync(c.base + zero_begin, 0, c.off - zero_begin, stream);
    return hist;
}

int sort_pairs_prepared(uint32_t *keys, uint32_t *vals, int64_t n, int key_bits, void *ws,
                        size_t ws_bytes, cudaStream_t stream, int first_bit, bool from_alt) {
    return sort_impl<uint32_t>(keys, vals, n, key_bits, ws, ws_bytes, stream, first_bit, from_alt,
                               true, true);
}

int sort_pairs64(uint64_t *keys, uint32_t *vals, int64_t n, int key_bits, void *ws,
                 size_t ws_bytes, cudaStream_t stream) {
    return sort_impl<uint64_t>(keys, vals, n, key_bits, ws, ws_bytes, stream, 0);
}

}  // namespace lbvh
