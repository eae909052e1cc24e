// HBM-bound elementwise / row kernels of the forward (K1 + K6 in SURVEY §2.3):
//   weight init (counter-based splitmix64; bit-identical to oracle/forward.c),
//   embedding gather, RMSNorm, RoPE + paged-KV append (the device half of
//   KvCacheRegistry, /root/reference/proj/src/executor.cpp:43-82), greedy argmax.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdint>

#include "attn.h"
#include "epi.cuh"
#include "ew.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace asb {

namespace {

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

// element i of a named tensor: the (i+1)-th draw of Rng::substream(seed, name)
// (/root/reference/proj/src/rng.hpp:28-37), mapped to a uniform bf16.  Source row r lands on
// logical row R = r*row_mult + row_off of the destination; with kb > 0 the destination is a
// tile-packed weight ([N/128][K/64][128][64], see runtime.h) of K = 64*kb columns.
__device__ __forceinline__ size_t packed_off(int64_t R, int64_t c, int kb, int dst_cols) {
    if (kb <= 0) return static_cast<size_t>(R) * dst_cols + c;
    return ((static_cast<size_t>(R >> 7) * kb + (c >> 6)) * 128 + (R & 127)) * 64 + (c & 63);
}

__global__ void init_weights_kernel(__nv_bfloat16* dst, uint64_t state0, int64_t rows, int cols,
                                    int row_mult, int row_off, int dst_cols, int kb, float offset,
                                    float amp_scaled) {
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t u = splitmix_mix(state0 + static_cast<uint64_t>(i + 1) * 0x9e3779b97f4a7c15ull);
        const int32_t t = static_cast<int32_t>(u >> 40) - 8388608;
        const float v = __fadd_rn(offset, __fmul_rn(static_cast<float>(t), amp_scaled));
        const int64_t r = i / cols, c = i % cols;
        dst[packed_off(r * row_mult + row_off, c, kb, dst_cols)] = __float2bfloat16_rn(v);
    }
}

// row-major [rows][cols] -> tile-packed (used for externally supplied weights)
__global__ void pack_weights_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                    int64_t rows, int cols) {
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        dst[packed_off(r, c, cols / 64, cols)] = src[i];
    }
}

// Embedding gather from the tile-packed table: a row is d/64 contiguous 128-byte chunks.
__global__ void embed_kernel(const int32_t* __restrict__ ids, const __nv_bfloat16* __restrict__ emb,
                             __nv_bfloat16* __restrict__ x, int T, int d,
                             unsigned long long* __restrict__ zero_keys, int n_keys,
                             const __nv_bfloat16* __restrict__ norm_w, __nv_bfloat16* __restrict__ h, float eps) {
    pdl_trigger();
    pdl_wait();
    const int t = blockIdx.x;
    // argmax accumulators of this forward's LM head (dgemv path: no final-norm launch)
    if (zero_keys && t == 0)
        for (int i = threadIdx.x; i < n_keys; i += blockDim.x) zero_keys[i] = 0ull;
    if (t >= T) return;
    const int64_t R = ids[t];
    const int kb = d / 64;
    uint4* dst = reinterpret_cast<uint4*>(x + static_cast<size_t>(t) * d);
    for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
        const int chunk = i >> 3, piece = i & 7;
        dst[i] = *reinterpret_cast<const uint4*>(emb + packed_off(R, chunk * 64 + piece * 8, kb, d));
    }
    if (!norm_w) return;
    // layer 0's pre-norm of this row, fused (rmsnorm_kernel's arithmetic, bit-identical)
    __shared__ float inv_s;
    __syncthreads();
    if (threadIdx.x < 32) {
        const float inv = rms_inv_warp(x + static_cast<size_t>(t) * d, d, eps, threadIdx.x);
        if (threadIdx.x == 0) inv_s = inv;
    }
    __syncthreads();
    const float inv = inv_s;
    const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * d);
    const uint4* wr = reinterpret_cast<const uint4*>(norm_w);
    uint4* hr = reinterpret_cast<uint4*>(h + static_cast<size_t>(t) * d);
    for (int i = threadIdx.x; i < d / 8; i += blockDim.x) {
        const uint4 v = xr[i], g = wr[i];
        hr[i] = make_uint4(rms_apply2(v.x, g.x, inv), rms_apply2(v.y, g.y, inv), rms_apply2(v.z, g.z, inv),
                           rms_apply2(v.w, g.w, inv));
    }
}

// One warp per row; y = bf16(x * (1/sqrt(mean(x^2)+eps)) * w).  rows_idx (optional)
// gathers input rows (final norm of the logit rows only).
__global__ void rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ rows_idx,
                               const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ y,
                               int n_rows, int d, float eps, unsigned long long* __restrict__ zero_keys) {
    pdl_trigger();
    pdl_wait();
    const int warps = blockDim.x >> 5;
    const int row = blockIdx.x * warps + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= n_rows) return;
    if (zero_keys && lane == 0) zero_keys[row] = 0ull;  // argmax accumulator of the next GEMM
    const int src_row = rows_idx ? rows_idx[row] : row;
    const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(src_row) * d);
    const uint4* wr = reinterpret_cast<const uint4*>(w);
    uint4* yr = reinterpret_cast<uint4*>(y + static_cast<size_t>(row) * d);
    const int nv = d / 8;
    // 4 loads in flight per lane (rms_inv_warp's summation order: bit-identical)
    const float inv = rms_inv_warp_cg(x + static_cast<size_t>(src_row) * d, d, eps, lane);
#pragma unroll 4
    for (int i = lane; i < nv; i += 32) {
        const uint4 v = xr[i], g = wr[i];
        const uint32_t a[4] = {v.x, v.y, v.z, v.w};
        const uint32_t b[4] = {g.x, g.y, g.z, g.w};
        uint32_t o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float lo = __fmul_rn(__fmul_rn(bf16_lo(a[e]), inv), bf16_lo(b[e]));
            const float hi = __fmul_rn(__fmul_rn(bf16_hi(a[e]), inv), bf16_hi(b[e]));
            o[e] = pack_bf16(lo, hi);
        }
        yr[i] = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// One CTA per token.  qkv row layout: [q heads | k heads | v heads] x hd.
// q -> q_out (rotated), k -> K pool (rotated), v -> V pool at the token's slot.
// Rotation: NeoX / Llama "rotate_half" with a host-built fp32 cos/sin table.
__global__ void rope_append_kernel(const __nv_bfloat16* __restrict__ qkv,
                                   const int32_t* __restrict__ pos,
                                   const int32_t* __restrict__ slot,
                                   const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                                   __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ k_pool,
                                   __nv_bfloat16* __restrict__ v_pool, int T, int hq, int hkv, int hd,
                                   int layer, int num_blocks) {
    pdl_trigger();
    pdl_wait();
    const int t = blockIdx.x;
    if (t >= T) return;
    const int half = hd / 2;
    const int p = pos[t];
    const int sl = slot[t];
    const int blk = sl / kBlockTokens, off = sl % kBlockTokens;
    const __nv_bfloat16* row = qkv + static_cast<size_t>(t) * (hq + 2 * hkv) * hd;
    const float* ct = cos_t + static_cast<size_t>(p) * half;
    const float* st = sin_t + static_cast<size_t>(p) * half;
    // rotated heads: q (hq) then k (hkv)
    for (int i = threadIdx.x; i < (hq + hkv) * half; i += blockDim.x) {
        const int h = i / half, j = i % half;
        const float x1 = __bfloat162float(row[h * hd + j]);
        const float x2 = __bfloat162float(row[h * hd + j + half]);
        const float c = ct[j], s = st[j];
        const float y1 = __fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, s));
        const float y2 = __fadd_rn(__fmul_rn(x2, c), __fmul_rn(x1, s));
        if (h < hq) {
            __nv_bfloat16* qo = q_out + (static_cast<size_t>(t) * hq + h) * hd;
            qo[j] = __float2bfloat16_rn(y1);
            qo[j + half] = __float2bfloat16_rn(y2);
        } else {
            const int kh = h - hq;
            __nv_bfloat16* kd =
                k_pool + (((static_cast<size_t>(layer) * num_blocks + blk) * hkv + kh) * kKvPageRows + off) * hd;
            kd[j] = __float2bfloat16_rn(y1);
            kd[j + half] = __float2bfloat16_rn(y2);
        }
    }
    for (int i = threadIdx.x; i < hkv * hd; i += blockDim.x) {
        const int h = i / hd, j = i % hd;
        __nv_bfloat16* vd =
            v_pool + (((static_cast<size_t>(layer) * num_blocks + blk) * hkv + h) * kKvPageRows + off) * hd;
        vd[j] = row[(hq + hkv + h) * hd + j];
    }
}

// Greedy argmax per logits row (lowest index wins ties) as an argmax_key.  One CTA per row.
// Only for logit batches the fused LM-head epilogue does not cover (> 256 rows).
__global__ void argmax_kernel(const float* __restrict__ logits, int V, int ld,
                              unsigned long long* __restrict__ out_keys) {
    pdl_trigger();
    pdl_wait();
    const float* lr = logits + static_cast<size_t>(blockIdx.x) * ld;
    unsigned long long best = 0ull;
    for (int i = threadIdx.x; i < V; i += blockDim.x) best = max(best, argmax_key(lr[i], i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    __shared__ unsigned long long sb[32];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sb[w] = best;
    __syncthreads();
    if (w == 0) {
        best = l < static_cast<int>(blockDim.x >> 5) ? sb[l] : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (l == 0) out_keys[blockIdx.x] = best;
    }
}

}  // namespace

cudaError_t init_weights(__nv_bfloat16* dst, uint64_t state0, int64_t rows, int cols, int row_mult,
                         int row_off, int packed_kb, float offset, float amp, cudaStream_t stream) {
    const int64_t n = rows * cols;
    int blocks = static_cast<int>((n + 255) / 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    init_weights_kernel<<<blocks, 256, 0, stream>>>(dst, state0, rows, cols, row_mult, row_off, cols,
                                                    packed_kb, offset, amp * (1.0f / 8388608.0f));
    return cudaGetLastError();
}

cudaError_t pack_weights(const __nv_bfloat16* src, __nv_bfloat16* dst, int64_t rows, int cols,
                         cudaStream_t stream) {
    const int64_t n = rows * cols;
    int blocks = static_cast<int>((n + 255) / 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    pack_weights_kernel<<<blocks, 256, 0, stream>>>(src, dst, rows, cols);
    return cudaGetLastError();
}

cudaError_t embed(const int32_t* ids, const __nv_bfloat16* emb, __nv_bfloat16* x, int T, int d,
                  cudaStream_t stream, unsigned long long* zero_keys, int n_keys, const __nv_bfloat16* norm_w,
                  __nv_bfloat16* h, float eps) {
    if (T <= 0) return cudaSuccess;
    return launch_k(embed_kernel, dim3(T), dim3(128), 0, stream, ids, emb, x, T, d, zero_keys, n_keys, norm_w, h,
                    eps);
}

cudaError_t rmsnorm(const __nv_bfloat16* x, const int32_t* rows_idx, const __nv_bfloat16* w,
                    __nv_bfloat16* y, int n_rows, int d, float eps, cudaStream_t stream,
                    unsigned long long* zero_keys) {
    if (n_rows <= 0) return cudaSuccess;
    const int warps = 2;  // one warp per row, rows spread over many SMs (latency-bound)
    return launch_k(rmsnorm_kernel, dim3((n_rows + warps - 1) / warps), dim3(warps * 32), 0, stream, x,
                    rows_idx, w, y, n_rows, d, eps, zero_keys);
}

cudaError_t rope_append(const __nv_bfloat16* qkv, const int32_t* pos, const int32_t* slot,
                        const float* cos_t, const float* sin_t, __nv_bfloat16* q_out,
                        __nv_bfloat16* k_pool, __nv_bfloat16* v_pool, int T, int hq, int hkv, int hd,
                        int layer, int num_blocks, cudaStream_t stream) {
    if (T <= 0) return cudaSuccess;
    return launch_k(rope_append_kernel, dim3(T), dim3(256), 0, stream, qkv, pos, slot, cos_t, sin_t, q_out,
                    k_pool, v_pool, T, hq, hkv, hd, layer, num_blocks);
}

cudaError_t argmax_rows(const float* logits, int rows, int V, int ld, unsigned long long* out_keys,
                        cudaStream_t stream) {
    if (rows <= 0) return cudaSuccess;
    return launch_k(argmax_kernel, dim3(rows), dim3(1024), 0, stream, logits, V, ld, out_keys);
}

}  // namespace asb
