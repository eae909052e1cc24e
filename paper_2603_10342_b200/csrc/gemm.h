#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace asb {

enum EpiMode : int {
    EPI_BF16 = 0,    // y = bf16(acc + bias?)
    EPI_RESID = 1,   // y = bf16(acc + resid)       (resid may alias out: in-place residual add)
    EPI_SILU = 2,    // y[:, j] = bf16(silu(acc[2j]) * acc[2j+1])  (interleaved gate/up rows)
    EPI_F32 = 3,     // y = acc (fp32)
    EPI_ATOMIC = 4,  // internal: split-K partial sums into ws
};

struct GemmParams {
    int M, N, K;          // kernel view: D[M][N] = A[M][K] . B[N][K]^T
    int tokens, n_out;    // logical view: Y[tokens][n_out]
    int swap;             // 0: A = X, B = W.  1: A = W, B = X (Y = D^T)
    int splits, kb_per_split;
    int streamk;          // 1: balanced stream-K over (tile, k-block); epilogue via ws atomics
    int epi;
    __nv_bfloat16* out;   // Y (bf16), row stride ldo
    float* out_f32;       // Y (fp32), row stride ldo
    int ldo;
    const __nv_bfloat16* bias;   // [n_out] or null
    const __nv_bfloat16* resid;  // [tokens][ldr]
    int ldr;
    float* ws;            // split-K workspace fp32 [tokens][n_out], must be zero on entry
};

int gemm_pick_bn(int n);
int gemm_smem_bytes(int bn);
cudaError_t gemm_launch(const CUtensorMap& ta, const CUtensorMap& tb, GemmParams p, int bn,
                        int num_sms, cudaStream_t stream);

// 3-D bf16 map over [d2][d1][d0] (d0 contiguous), box = [b2][b1][64], SWIZZLE_128B.
bool make_tmap_bf16_3d(CUtensorMap* out, const void* base, int d0, int d1, int d2, int b1, int b2);
// 2-D bf16 tensor map, row-major [rows][cols], box = [box_rows][64 cols], SWIZZLE_128B.
bool make_tmap_bf16(CUtensorMap* out, const void* base, int rows, int cols, int row_stride_elems,
                    int box_rows);

}  // namespace asb
