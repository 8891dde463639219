// internal.cuh -- host-side declarations shared between translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lbvh {

// Records the CUDA error string for lbvh_last_cuda_error(); returns
// LBVH_ERR_CUDA on a pending launch error, LBVH_OK otherwise.
int check_launch();
void set_cuda_error(cudaError_t e);
// Kernel-launch accounting for lbvh_launch_count().
void count_launches(int k);
uint64_t launch_count();

size_t sort_workspace_bytes(int64_t n);
// Stable LSD sort on key bits [first_bit, key_bits).
int sort_pairs(uint32_t *keys, uint32_t *vals, int64_t n, int key_bits, void *ws,
               size_t ws_bytes, cudaStream_t stream, int first_bit = 0);
// The workspace's ping-pong buffers, where sort_pairs_from_alt expects its
// input; pass count of a sort of bits [first_bit, key_bits).
void sort_alt_buffers(void *ws, size_t ws_bytes, int64_t n, uint32_t **k_alt, uint32_t **v_alt);
int sort_pass_count(int key_bits, int first_bit);
int sort_pairs_from_alt(uint32_t *keys, uint32_t *vals, int64_t n, int key_bits, void *ws,
                        size_t ws_bytes, cudaStream_t stream, int first_bit);
// Fused producers (u32 keys, 8-bit digits): sort_prepare zeroes the sort
// state and returns the digit-histogram array (4 x 256 counts) that a
// producer kernel fills while it writes the keys (hist_accumulate /
// hist_flush); sort_pairs_prepared then sorts with the values implicitly
// 0..n-1 (argsort: `vals` is written, not read).
uint32_t *sort_prepare(void *ws, size_t ws_bytes, int64_t n, cudaStream_t stream);
int sort_pairs_prepared(uint32_t *keys, uint32_t *vals, int64_t n, int key_bits, void *ws,
                        size_t ws_bytes, cudaStream_t stream, int first_bit, bool from_alt);
size_t sort64_workspace_bytes(int64_t n);
int sort_pairs64(uint64_t *keys, uint32_t *vals, int64_t n, int key_bits, void *ws,
                 size_t ws_bytes, cudaStream_t stream);

size_t scan_workspace_bytes(int64_t n);
// offsets[0] = 0, offsets[i+1] = offsets[i] + f(i); f reads counts (i32) or
// the per-query kNN span min(k_q, n).
int scan_counts(const int32_t *counts, int64_t n, int64_t *offsets, void *ws,
                size_t ws_bytes, cudaStream_t stream);

}  // namespace lbvh
