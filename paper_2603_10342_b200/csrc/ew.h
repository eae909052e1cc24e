#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace asb {

// Fill dst (row-major [rows*row_mult][cols] slab; source row r lands at r*row_mult+row_off)
// with offset + amp * U[-1, 1) drawn from splitmix64 state0 (counter-based).
cudaError_t init_weights(__nv_bfloat16* dst, uint64_t state0, int64_t rows, int cols, int row_mult,
                         int row_off, float offset, float amp, cudaStream_t stream);
cudaError_t embed(const int32_t* ids, const __nv_bfloat16* emb, __nv_bfloat16* x, int T, int d,
                  cudaStream_t stream);
cudaError_t rmsnorm(const __nv_bfloat16* x, const int32_t* rows_idx, const __nv_bfloat16* w,
                    __nv_bfloat16* y, int n_rows, int d, float eps, cudaStream_t stream);
cudaError_t rope_append(const __nv_bfloat16* qkv, const int32_t* pos, const int32_t* slot,
                        const float* cos_t, const float* sin_t, __nv_bfloat16* q_out,
                        __nv_bfloat16* k_pool, __nv_bfloat16* v_pool, int T, int hq, int hkv, int hd,
                        int layer, int num_blocks, cudaStream_t stream);
cudaError_t argmax_rows(const float* logits, int rows, int V, int ld, int32_t* out_ids,
                        float* out_max, cudaStream_t stream);

}  // namespace asb
