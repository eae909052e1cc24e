#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace asb {

// Fill dst with offset + amp * U[-1, 1) drawn from splitmix64 state0 (counter-based).  Source
// row r lands on logical row r*row_mult+row_off; packed_kb > 0 selects the tile-packed weight
// layout [N/128][K/64][128][64] with K = 64*packed_kb (0: row-major [..][cols]).
cudaError_t init_weights(__nv_bfloat16* dst, uint64_t state0, int64_t rows, int cols, int row_mult,
                         int row_off, int packed_kb, float offset, float amp, cudaStream_t stream);
cudaError_t pack_weights(const __nv_bfloat16* src, __nv_bfloat16* dst, int64_t rows, int cols,
                         cudaStream_t stream);
// zero_keys (optional): zeroed [n_keys] argmax-key accumulator of the LM head of this forward.
// norm_w (optional): also h[t] = layer 0's pre-norm of the row (rmsnorm_kernel arithmetic).
cudaError_t embed(const int32_t* ids, const __nv_bfloat16* emb, __nv_bfloat16* x, int T, int d,
                  cudaStream_t stream, unsigned long long* zero_keys = nullptr, int n_keys = 0,
                  const __nv_bfloat16* norm_w = nullptr, __nv_bfloat16* h = nullptr, float eps = 0.f);
// zero_keys (optional): zeroed [n_rows] argmax-key accumulator for the LM head that follows.
cudaError_t rmsnorm(const __nv_bfloat16* x, const int32_t* rows_idx, const __nv_bfloat16* w,
                    __nv_bfloat16* y, int n_rows, int d, float eps, cudaStream_t stream,
                    unsigned long long* zero_keys = nullptr);
cudaError_t rope_append(const __nv_bfloat16* qkv, const int32_t* pos, const int32_t* slot,
                        const float* cos_t, const float* sin_t, __nv_bfloat16* q_out,
                        __nv_bfloat16* k_pool, __nv_bfloat16* v_pool, int T, int hq, int hkv, int hd,
                        int layer, int num_blocks, cudaStream_t stream);
// Row argmax as argmax_key (sm100.cuh): idx = argmax_key_index(key).
cudaError_t argmax_rows(const float* logits, int rows, int V, int ld, unsigned long long* out_keys,
                        cudaStream_t stream);

}  // namespace asb
