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

// element offset of (slot, kv_head) from the K (k_pool) or V (v_pool = k_pool + one page)
// base of the interleaved paged pool (layout of attn.h)
__device__ __forceinline__ size_t pool_off(const RopeEpi& R, int slot, int kv_head) {
    const int blk = slot / kBlockTokens, off = slot % kBlockTokens;
    return ((((size_t)R.layer * R.num_blocks + blk) * R.hkv + kv_head) * kKvPageRows + off) * R.hd;
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

__device__ __forceinline__ uint4 ldcg128(const void* p) {
    uint4 v;
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// rms_inv_warp for a row other CTAs of the running grid wrote (L2 reads, 4 loads in flight per
// lane); the same summation order, so the result is bit-identical.
__device__ __forceinline__ float rms_inv_warp_cg(const __nv_bfloat16* row, int d, float eps, int lane) {
    float ss = 0.f;
    const int n = d / 8;
    for (int i0 = lane; i0 < n; i0 += 4 * 32) {
        uint4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + 32 * u < n) v[u] = ldcg128(row + 8 * (i0 + 32 * u));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (i0 + 32 * u >= n) break;
            const uint32_t a[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float lo = bf16_lo(a[e]), hi = bf16_hi(a[e]);
                ss = __fadd_rn(ss, __fadd_rn(__fmul_rn(lo, lo), __fmul_rn(hi, hi)));
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    return __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, static_cast<float>(d)), eps)));
}

// True in exactly one CTA of the grid: the last to get here.  Every thread of every CTA must
// call it once, after its global stores; the counter re-arms itself.
__device__ __forceinline__ bool grid_last_arriver(int* counter) {
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int total = static_cast<int>(gridDim.x * gridDim.y * gridDim.z);
        const int prev = atomicAdd(counter, 1);
        s_last = prev == total - 1;
        if (s_last) *counter = 0;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0;
}

// The next layer's pre-norm, run by the last CTA of a residual-writing GEMM once all of x is
// in place: y[r] = bf16(x[src_r] * rms_inv * w) (rmsnorm_kernel's arithmetic), optionally
// zeroing the greedy-argmax keys of the LM head that follows.
__device__ __forceinline__ void post_norm_rows(const PostNorm& q, const __nv_bfloat16* x, int ldx) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int r = warp; r < q.n_rows; r += nw) {
        const int src = q.rows ? q.rows[r] : r;
        const __nv_bfloat16* xr = x + static_cast<size_t>(src) * ldx;
        const float inv = rms_inv_warp_cg(xr, q.d, q.eps, lane);
        uint4* yr = reinterpret_cast<uint4*>(q.out + static_cast<size_t>(r) * q.d);
        const uint4* wr = reinterpret_cast<const uint4*>(q.w);
        for (int i = lane; i < q.d / 8; i += 32) {
            const uint4 v = ldcg128(xr + 8 * i), g = wr[i];
            yr[i] = make_uint4(rms_apply2(v.x, g.x, inv), rms_apply2(v.y, g.y, inv), rms_apply2(v.z, g.z, inv),
                               rms_apply2(v.w, g.w, inv));
        }
        if (q.zero_keys && lane == 0) q.zero_keys[r] = 0ull;
    }
}

}  // namespace asb
