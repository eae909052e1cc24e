// Device helpers shared by the GEMM epilogues (tcgen05 gemm.cu, decode dgemv.cu) and the
// standalone elementwise kernels (ew.cu), so the fused and unfused paths round at the same
// points with the same operation order (bit-identical results).
#pragma once
#include <cuda_bf16.h>

#include "attn.h"
#include "gemm.h"
#include "sm100.cuh"

namespace asb {

__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

__device__ __forceinline__ float bf16r(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// element offset of (slot, kv_head) in a paged K or V pool (layout of attn.h)
__device__ __forceinline__ size_t pool_off(const RopeEpi& R, int slot, int kv_head) {
    const int blk = slot / kBlockTokens, off = slot % kBlockTokens;
    return ((((size_t)R.layer * R.num_blocks + blk) * R.hkv + kv_head) * kBlockTokens + off) * R.hd;
}

// rotate_half pair at one cos/sin column
__device__ __forceinline__ void rope2(float x1, float x2, float c, float s, float& y1, float& y2) {
    y1 = __fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, s));
    y2 = __fadd_rn(__fmul_rn(x2, c), __fmul_rn(x1, s));
}

// RMSNorm statistics of one row, one warp: lane l sums the 16-byte chunks l, l+32, ... in
// order, then a xor butterfly.  Returns 1/sqrt(mean(x^2)+eps) on every lane.
__device__ __forceinline__ float rms_inv_warp(const __nv_bfloat16* __restrict__ row, int d, float eps,
                                              int lane) {
    const uint4* xr = reinterpret_cast<const uint4*>(row);
    float ss = 0.f;
    for (int i = lane; i < d / 8; i += 32) {
        const uint4 v = xr[i];
        const uint32_t a[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float lo = bf16_lo(a[e]), hi = bf16_hi(a[e]);
            ss = __fadd_rn(ss, __fadd_rn(__fmul_rn(lo, lo), __fmul_rn(hi, hi)));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, static_cast<float>(d)), eps)));
}

// y = bf16(x * inv * w) for a pair of bf16 (packed), the RMSNorm output rounding point
__device__ __forceinline__ uint32_t rms_apply2(uint32_t x, uint32_t w, float inv) {
    return pack_bf16(__fmul_rn(__fmul_rn(bf16_lo(x), inv), bf16_lo(w)),
                     __fmul_rn(__fmul_rn(bf16_hi(x), inv), bf16_hi(w)));
}

}  // namespace asb
