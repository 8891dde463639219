// EXPERIMENT (not compiled into the library): warp-cooperative pass for heavy
// 2P radius queries that keeps the reference's fill order (ordered atom
// sequence expanded level by level, one query per warp), fed by a count pass
// that stops a query at its first hit beyond the row.  Exact and
// sanitizer-clean, but at C3 the heavy pass took 9.5 ms (12.0 ms with four
// atoms per lane per step) against ~2.4 ms for the serial traversal it
// replaces (the count pass itself fell 3.37 -> 1.00 ms): each tree level is a
// dependent round for the whole warp and only ~1,800 such warps run at once,
// against ~300,000 per-lane queries.

// Heavy radius queries (more hits than the 2P row): one warp per query.
// The reference's DFS (_kernels.py:212-225) emits, at each node, the left
// leaf hit, the right leaf hit, then the whole right subtree, then the whole
// left subtree.  So the hit sequence is an ordered sequence of atoms -- a
// leaf hit or a subtree still to expand -- and expanding every subtree atom
// in place by [L hit][R hit][R subtree][L subtree] keeps it in the
// reference's order.  The warp expands all subtree atoms of the sequence at
// once, one level per round (a warp scan places each atom's products), until
// only hits remain: the count, and the hits in fill order, with 32 node
// fetches in flight and no per-lane divergence.  Hits beyond the row go to
// the spill pool as one run of linked chunks (spill_copy reads them as
// before).  A sequence that outgrows shared memory is recounted without its
// hits and filled by the fill pass.  Trees from lbvh_build with 30-bit codes
// only: their depth (< 63) keeps the reference's 64-entry stack from ever
// overflowing, which the level-by-level order does not track.
constexpr int kHeavyWarps = 4;
constexpr int kAtomCap = 2048;
constexpr int kHeavyU = 4;  // atoms per lane per step

__device__ __forceinline__ int warp_excl_scan(int v, int &total) {
    const int lane = threadIdx.x & 31;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xFFFFFFFFu, x, 31);
    return x - v;
}

__global__ void __launch_bounds__(32 * kHeavyWarps)
spatial_heavy_kernel(const lbvh_tree t, const float *__restrict__ centers,
                     const float *__restrict__ radii, float radius,
                     const uint32_t *__restrict__ list, const uint32_t *__restrict__ list_len,
                     int32_t *__restrict__ counts, int64_t cap, int32_t *__restrict__ heads,
                     int32_t *__restrict__ pool, uint32_t pool_chunks) {
    extern __shared__ int32_t heavy_atoms[];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    int32_t *const bufA = heavy_atoms + wib * 2 * kAtomCap;
    int32_t *const bufB = bufA + kAtomCap;
    const PackedNode *__restrict__ nodes = reinterpret_cast<const PackedNode *>(t.nodes);
    const int64_t n = (int64_t)*list_len;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n; w += warps) {
        const int64_t q = __ldg(list + w);
        const float px = __ldg(centers + 3 * q), py = __ldg(centers + 3 * q + 1),
                    pz = __ldg(centers + 3 * q + 2);
        const float r = radii ? __ldg(radii + q) : radius;
        const float r2 = __fmul_rn(r, r);
        int32_t *A = bufA;
        int ma = 0;
        int64_t dropped = 0;  // count-only attempt: leaf hits counted, not kept
        bool ordered = true, overflow = false;
        for (int attempt = 0; attempt < 2; ++attempt) {
            ordered = attempt == 0;
            A = bufA;
            int32_t *B = bufB;
            if (lane == 0) A[0] = 0;  // the root (a heavy query's tree has >= 2 leaves)
            __syncwarp();
            ma = 1;
            dropped = 0;
            overflow = false;
            bool inner = true;
            while (inner && !overflow) {
                int mo = 0;
                bool any_inner = false;
                // each lane takes kHeavyU consecutive atoms: their node loads
                // are in flight together, and a scan of the lane totals keeps
                // the products in sequence order
                for (int base = 0; base < ma; base += 32 * kHeavyU) {
                    int32_t lk[kHeavyU], rk[kHeavyU];
                    uint32_t pass = 0;  // bit 2u: left child passes, 2u + 1: right
                    uint32_t carried = 0;  // bit u: atom u is a hit, carried as is
                    int c = 0, lc = 0;
#pragma unroll
                    for (int u = 0; u < kHeavyU; ++u) {
                        const int i = base + lane * kHeavyU + u;
                        const int32_t at = i < ma ? A[i] : 0x7FFFFFFF;  // 0x7FFFFFFF: none
                        lk[u] = at;
                        rk[u] = 0;
                        if (at >= 0 && at != 0x7FFFFFFF) {
                            float4 a, b, cc;
                            int4 d;
                            load_node(nodes, at, a, b, cc, d);
                            const bool pl =
                                box_dist_sq(px, py, pz, a.x, a.y, a.z, a.w, b.x, b.y) <= r2;
                            const bool pr =
                                box_dist_sq(px, py, pz, b.z, b.w, cc.x, cc.y, cc.z, cc.w) <= r2;
                            lk[u] = d.x;
                            rk[u] = d.y;
                            pass |= (pl ? 1u : 0u) << (2 * u);
                            pass |= (pr ? 2u : 0u) << (2 * u);
                            // products: [L hit][R hit][R subtree][L subtree]
                            if (ordered) c += (int)pl + (int)pr;
                            else lc += (int)(pl && d.x < 0) + (int)(pr && d.y < 0),
                                 c += (int)(pl && d.x >= 0) + (int)(pr && d.y >= 0);
                        } else if (at < 0) {
                            c += 1;  // a hit: carried
                            carried |= 1u << u;
                        }
                    }
                    int tot = 0;
                    const int ex = warp_excl_scan(c, tot);
                    bool inner_here = false;
                    if (mo + tot > kAtomCap) {
                        overflow = true;  // warp-uniform
                    } else if (!overflow) {
                        int32_t *o = B + mo + ex;
#pragma unroll
                        for (int u = 0; u < kHeavyU; ++u) {
                            const int32_t at = lk[u];
                            const uint32_t pb = pass >> (2 * u);
                            if (base + lane * kHeavyU + u >= ma) continue;
                            if (carried & (1u << u)) {
                                *o++ = at;
                                continue;
                            }
                            const int32_t L = lk[u], R = rk[u];
                            const bool pl = pb & 1u, pr = pb & 2u;
                            if (pl && L < 0 && ordered) *o++ = L;
                            if (pr && R < 0 && ordered) *o++ = R;
                            if (pr && R >= 0) { *o++ = R; inner_here = true; }
                            if (pl && L >= 0) { *o++ = L; inner_here = true; }
                        }
                    }
                    any_inner |= __any_sync(0xFFFFFFFFu, inner_here);
                    int lsum = lc;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(0xFFFFFFFFu, lsum, o);
                    dropped += lsum;
                    mo += tot;
                }
                __syncwarp();
                int32_t *tmp = A; A = B; B = tmp;
                ma = mo;
                inner = any_inner;
            }
            if (!overflow) break;
            // too many atoms for shared memory: count again without the hits
        }
        int64_t total = ordered ? ma : dropped;
        if (overflow) {  // even the subtree frontier outgrew it: one lane counts serially
            int64_t cnt = 0;
            if (lane == 0) {
                int32_t stack[kStack];
                int sp = 0;
                int32_t node = 0;
                while (true) {
                    float4 a, b, cc;
                    int4 d;
                    load_node(nodes, node, a, b, cc, d);
                    int32_t next = -1;
                    if (box_dist_sq(px, py, pz, a.x, a.y, a.z, a.w, b.x, b.y) <= r2) {
                        if (d.x < 0) ++cnt; else stack[sp++] = d.x;
                    }
                    if (box_dist_sq(px, py, pz, b.z, b.w, cc.x, cc.y, cc.z, cc.w) <= r2) {
                        if (d.y < 0) ++cnt; else next = d.y;
                    }
                    if (next < 0) {
                        if (sp == 0) break;
                        next = stack[--sp];
                    }
                    node = next;
                }
            }
            total = __shfl_sync(0xFFFFFFFFu, cnt, 0);
        }
        if (lane == 0) counts[q] = (int32_t)total;
        int32_t c0 = -1;
        if (ordered && total > cap) {
            const int64_t nsp = total - cap;
            const int64_t nch = (nsp + kSpillChunk - 2) / (kSpillChunk - 1);
            if (lane == 0) {
                const uint64_t at = atomicAdd(reinterpret_cast<uint32_t *>(pool), (uint32_t)nch);
                c0 = (at + 1 + nch <= pool_chunks) ? (int32_t)(at + 1) : -1;
            }
            c0 = __shfl_sync(0xFFFFFFFFu, c0, 0);
            if (c0 > 0) {
                for (int64_t j = lane; j < nsp; j += 32)
                    pool[(int64_t)(c0 + j / (kSpillChunk - 1)) * kSpillChunk +
                         j % (kSpillChunk - 1)] = A[cap + j] & 0x7FFFFFFF;
                for (int64_t k = lane; k + 1 < nch; k += 32)
                    pool[(int64_t)(c0 + k) * kSpillChunk + kSpillChunk - 1] = (int32_t)(c0 + k + 1);
            }
        }
        if (lane == 0) heads[q] = c0;  // -1: the fill pass writes this query
        __syncwarp();
    }
}

int spatial_heavy(const lbvh_tree *t, const float *centers, const float *radii, float radius,
                  const uint32_t *list, const uint32_t *list_len, int32_t *counts, int64_t cap,
                  int32_t *heads, int32_t *pool, int64_t pool_chunks, cudaStream_t stream);

