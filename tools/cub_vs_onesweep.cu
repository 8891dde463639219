// CUB bar for the build's key sort ("beat CUB SortPairs on
// the same box").  Times cub::DeviceRadixSort::SortPairs over key bits
// [0, 30) -- what the build needs for 30-bit Morton codes with iota values --
// against lbvh_sort_pairs (liblbvh_b200.so) on the same keys, at 1e7 and 1e8.
//
//   make -C tools cub_vs_onesweep && tools/cub_vs_onesweep > profiles/r02_cub_vs_onesweep.json
//
// Keys: the 30-bit Morton codes of the C2 cloud are uniform over the grid,
// so uniform random 30-bit keys (splitmix64) have the same digit statistics.
// Both sorts are stable; the outputs are compared element for element.
#include <cub/cub.cuh>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../include/lbvh_b200.h"

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            exit(1);                                                                \
        }                                                                           \
    } while (0)

__global__ void fill_keys(uint32_t *k, uint32_t *v, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + 0x632BE59BD9B4E019ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        k[i] = (uint32_t)(z & ((1u << 30) - 1));
        v[i] = (uint32_t)i;
    }
}

int main(int argc, char **argv) {
    const int reps = argc > 1 ? atoi(argv[1]) : 20;
    const int64_t sizes[2] = {10000000, 100000000};
    printf("{\n \"what\": \"stable (30-bit key, u32 value) sort, keys uniform over [0, 2^30), "
           "values iota; mean of %d reps, CUDA events around the sort call only\",\n", reps);
    printf(" \"results\": [\n");
    for (int si = 0; si < 2; ++si) {
        const int64_t n = sizes[si];
        uint32_t *k0, *v0, *k1, *v1, *kc, *vc;
        CK(cudaMalloc(&k0, n * 4));
        CK(cudaMalloc(&v0, n * 4));
        CK(cudaMalloc(&k1, n * 4));
        CK(cudaMalloc(&v1, n * 4));
        CK(cudaMalloc(&kc, n * 4));
        CK(cudaMalloc(&vc, n * 4));
        fill_keys<<<148 * 8, 256>>>(k0, v0, n);
        CK(cudaDeviceSynchronize());
        // CUB, out of place (input untouched between reps)
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k0, kc, v0, vc, (int)n, 0, 30);
        void *tmp;
        CK(cudaMalloc(&tmp, tmp_bytes));
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        float cub_ms = 0.f;
        for (int r = -2; r < reps; ++r) {
            CK(cudaEventRecord(a));
            cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k0, kc, v0, vc, (int)n, 0, 30);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (r >= 0) cub_ms += ms;
        }
        cub_ms /= reps;
        // lbvh_sort_pairs, in place: reload the keys before every rep (untimed)
        size_t ws_bytes = lbvh_sort_workspace_bytes(n);
        void *ws;
        CK(cudaMalloc(&ws, ws_bytes));
        float lb_ms = 0.f;
        for (int r = -2; r < reps; ++r) {
            CK(cudaMemcpy(k1, k0, n * 4, cudaMemcpyDeviceToDevice));
            CK(cudaMemcpy(v1, v0, n * 4, cudaMemcpyDeviceToDevice));
            CK(cudaEventRecord(a));
            int rc = lbvh_sort_pairs(k1, v1, n, 30, ws, ws_bytes, nullptr);
            CK(cudaEventRecord(b));
            CK(cudaEventSynchronize(b));
            if (rc) {
                fprintf(stderr, "lbvh_sort_pairs: %s\n", lbvh_strerror(rc));
                return 1;
            }
            float ms;
            CK(cudaEventElapsedTime(&ms, a, b));
            if (r >= 0) lb_ms += ms;
        }
        lb_ms /= reps;
        // same output (both stable)
        uint32_t *hk = (uint32_t *)malloc(n * 4), *hkc = (uint32_t *)malloc(n * 4);
        uint32_t *hv = (uint32_t *)malloc(n * 4), *hvc = (uint32_t *)malloc(n * 4);
        CK(cudaMemcpy(hk, k1, n * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hkc, kc, n * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hv, v1, n * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hvc, vc, n * 4, cudaMemcpyDeviceToHost));
        int64_t diff = 0;
        for (int64_t i = 0; i < n; ++i) diff += (hk[i] != hkc[i]) | (hv[i] != hvc[i]);
        const double gb = 16.0 * n / 1e9;  // one read + one write of (key, value) pairs
        printf("  {\"n\": %lld, \"cub_sortpairs_0_30_ms\": %.4f, \"lbvh_sort_pairs_30_ms\": %.4f, "
               "\"lbvh_over_cub\": %.3f, \"cub_gkeys_per_s\": %.3f, \"lbvh_gkeys_per_s\": %.3f, "
               "\"pair_bytes_gb\": %.3f, \"mismatches\": %lld}%s\n",
               (long long)n, cub_ms, lb_ms, lb_ms / cub_ms, n / cub_ms / 1e6, n / lb_ms / 1e6, gb,
               (long long)diff, si == 0 ? "," : "");
        free(hk); free(hkc); free(hv); free(hvc);
        cudaFree(k0); cudaFree(v0); cudaFree(k1); cudaFree(v1); cudaFree(kc); cudaFree(vc);
        cudaFree(tmp); cudaFree(ws);
    }
    printf(" ]\n}\n");
    return 0;
}
