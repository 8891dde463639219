// EXPERIMENT (not compiled into the library): warp-packet kNN for queries
// with large search balls (hollow-sphere sources), routed per warp by the
// seed radius, optionally after a per-lane nearest-first dive.  Exact
// results, but slower ("Explored and rejected"): at C3
// sources / 1e7 filled queries the per-warp union of visited nodes is 9,634
// vs 3,608 for the per-thread path's slowest lane (tools/knn_visits.py),
// 1,190 vs 785 ms.  Drop-in for knn_kernel in csrc/traverse.cu (needs
// knn_write_span and knn_query's pre_bound parameter from the same commit).

// Warp packets for queries with a large search ball (a query inside a hollow
// sphere has a k-th distance comparable to the sphere's radius and its ball
// overlaps thousands of node boxes): the 32 queries of a warp descend one
// shared node sequence, every record fetched once for the warp (a broadcast
// load) and tested by every lane against its own k-th distance; a child is
// visited if any lane's test passes, the nearer one (by lane vote) first.
// Each lane's k-best list, seed and pruning rule are the per-query path's,
// and the result -- the unique k smallest (dist^2, ordinal) pairs -- does not
// depend on the visiting order.  Only trees built from 30-bit codes take it:
// their depth is below 63 (each level strictly lengthens the common prefix
// of the 62-bit augmented keys), so neither path can exhaust the 64-entry
// stack and the reference's stack limit never applies.
#ifndef LBVH_KNN_PACKET_DIVE
#define LBVH_KNN_PACKET_DIVE 0
#endif
#ifndef LBVH_KNN_PACKET_MIN_LANES
#define LBVH_KNN_PACKET_MIN_LANES 4
#endif
// A lane asks for the packet path when its seed radius exceeds this many
// times the k-neighbour radius of a uniform cloud filling the scene box.
#ifndef LBVH_KNN_PACKET_RADIUS_X
#define LBVH_KNN_PACKET_RADIUS_X 8.0f
#endif

__device__ __forceinline__ float packet_threshold_sq(const lbvh_tree &t, int kk) {
    float ext[3], emax = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        ext[a] = __ldg(t.root_box + 3 + a) - __ldg(t.root_box + a);
        emax = fmaxf(emax, ext[a]);
    }
    // flat or degenerate scenes: no axis thinner than 1e-3 of the widest
    const float v = fmaxf(ext[0], 1e-3f * emax) * fmaxf(ext[1], 1e-3f * emax) *
                    fmaxf(ext[2], 1e-3f * emax);
    const float rk = cbrtf((float)kk * v / (float)t.n * 0.2387324f);  // 3 / (4 pi)
    const float r = LBVH_KNN_PACKET_RADIUS_X * rk;
    return r * r;
}

template <int K>
__device__ __forceinline__ int knn_packet(const lbvh_tree &t, bool active, float px, float py,
                                           float pz, TopK<K> &top, int32_t *wstack) {
    const PackedNode *__restrict__ nodes = reinterpret_cast<const PackedNode *>(t.nodes);
    const uint32_t amask = __ballot_sync(0xFFFFFFFFu, active);
    const int half = __popc(amask) >> 1;
    int sp = 0;
    int32_t node = 0;
#ifdef LBVH_KNN_COUNT_VISITS
    int visits = 0;
#endif
    while (true) {
        float4 a, b, c;
        int4 dd;
#ifdef LBVH_KNN_COUNT_VISITS
        ++visits;
#endif
        load_node(nodes, node, a, b, c, dd);  // one address for the whole warp
        const float dl = box_dist_sq(px, py, pz, a.x, a.y, a.z, a.w, b.x, b.y);
        const float dr = box_dist_sq(px, py, pz, b.z, b.w, c.x, c.y, c.z, c.w);
        const bool wl = active && !(dl > top.worst());
        const bool wr = active && !(dr > top.worst());
        const bool lleaf = dd.x < 0, rleaf = dd.y < 0;  // warp-uniform
        if (lleaf && wl) top.offer(dl, dd.x & 0x7FFFFFFF);
        if (rleaf && wr) top.offer(dr, dd.y & 0x7FFFFFFF);
        const bool gl = __any_sync(0xFFFFFFFFu, wl && !lleaf);
        const bool gr = __any_sync(0xFFFFFFFFu, wr && !rleaf);
        int32_t next = -1;
        if (gl && gr) {
            const bool left_first =
                __popc(__ballot_sync(0xFFFFFFFFu, active && dl <= dr)) >= half;
            next = left_first ? dd.x : dd.y;
            if (lane_id() == 0) wstack[sp] = left_first ? dd.y : dd.x;
            ++sp;
        } else if (gl) {
            next = dd.x;
        } else if (gr) {
            next = dd.y;
        }
        if (next < 0) {
            if (sp == 0) break;
            --sp;
            __syncwarp();
            next = wstack[sp];
        }
        node = next;
    }
#ifdef LBVH_KNN_COUNT_VISITS
    return visits;
#else
    return 0;
#endif
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
    constexpr uint32_t kPacketTree = LBVH_TREE_BUILT | LBVH_TREE_CODES30;
    if ((t.flags & kPacketTree) != kPacketTree || t.n < 2 || !qcodes || !t.leaf_codes) {
        if (s >= nq) return;
        knn_query<K>(t, centers, order, qcodes, s, offsets, out_idx, out_dist, squared, status,
                     kth, uniform);
        return;
    }
    // per lane: its query, span and exact seed; then the warp picks a path
    const bool valid = s < nq;
    int64_t q = 0, base = 0;
    int kk = 0;
    float px = 0.f, py = 0.f, pz = 0.f, bound = __int_as_float(0x7FFFFFFF);
    if (valid) {
        q = order ? (int64_t)__ldg(order + s) : s;
        base = uniform ? q * uniform : __ldg(offsets + q);
        kk = uniform ? uniform : (int)(__ldg(offsets + q + 1) - base);
        if (kk > 0) {
            px = __ldg(centers + 3 * q);
            py = __ldg(centers + 3 * q + 1);
            pz = __ldg(centers + 3 * q + 2);
            bound = seed_bound<K>(t, __ldg(qcodes + s), kk, px, py, pz);
        }
    }
    const bool active = valid && kk > 0;
    const bool want = active && bound > packet_threshold_sq(t, kk);
    if (__popc(__ballot_sync(0xFFFFFFFFu, want)) >= LBVH_KNN_PACKET_MIN_LANES) {
        __shared__ int32_t pstack[(LBVH_KNN_BLOCK / 32) * kStack];
        TopK<K> top;
        top.init(active ? kk : K, bound);
#if LBVH_KNN_PACKET_DIVE > 0
        // each lane first dives nearest-first on its own for a few node
        // visits: its k-th best so far is a tight bound for the packet pass,
        // which then starts over (virtual candidates at that bound, like the seed)
        if (active) {
            const PackedNode *__restrict__ nodes = reinterpret_cast<const PackedNode *>(t.nodes);
            int32_t dstack[16];
            int dsp = 0;
            int32_t node = 0;
            for (int v = 0; v < LBVH_KNN_PACKET_DIVE; ++v) {
                float4 a, b, c;
                int4 dd;
                load_node(nodes, node, a, b, c, dd);
                const float dl = box_dist_sq(px, py, pz, a.x, a.y, a.z, a.w, b.x, b.y);
                const float dr = box_dist_sq(px, py, pz, b.z, b.w, c.x, c.y, c.z, c.w);
                const bool left_near = dl <= dr;
                const int32_t fl = left_near ? dd.y : dd.x, nl = left_near ? dd.x : dd.y;
                const float fd = left_near ? dr : dl, nd = left_near ? dl : dr;
                int32_t next = -1;
                if (!(fd > top.worst())) {
                    if (fl < 0) top.offer(fd, fl & 0x7FFFFFFF);
                    else if (dsp < 16) dstack[dsp++] = fl;
                }
                if (!(nd > top.worst())) {
                    if (nl < 0) top.offer(nd, nl & 0x7FFFFFFF);
                    else next = nl;
                }
                if (next < 0) {
                    if (dsp == 0) break;
                    next = dstack[--dsp];
                }
                node = next;
            }
            const float b2 = top.worst();
            top.init(kk, isnan(b2) ? bound : b2);
        }
#endif
        const int visits =
            knn_packet<K>(t, active, px, py, pz, top, pstack + (threadIdx.x >> 5) * kStack);
        if (!active) return;
        if (kth) kth[q] = top.dist(K - 1);
        knn_write_span<K>(top, base, kk, out_idx, out_dist, squared);
#ifdef LBVH_KNN_COUNT_VISITS  // instrumentation builds only: -visits in place of distance 0
        out_dist[base] = -(float)visits;
#else
        (void)visits;
#endif
        return;
    }
    if (!valid) return;
    knn_query<K>(t, centers, order, qcodes, s, offsets, out_idx, out_dist, squared, status, kth,
                 uniform, &bound);
}

