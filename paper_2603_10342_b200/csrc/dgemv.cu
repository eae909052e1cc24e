// Small-batch decode linear layer ("dgemv"): Y[tok][n] = sum_k X[tok][k] * W[n][k] for
// T <= 32 tokens, the regime of the decode steps at C1/C2 (B <= 8 rows + a <= 16-token
// admitted resume chunk).  Replaces, with decode_attention, the mu_D term of the
// reference's decode_step_duration_ms (/root/reference/proj/src/executor.cpp:84-97).
//
// At T <= 32 a linear layer is a pure weight stream: 2 bytes of W per 2*T flops.  The
// tcgen05 kernel (gemm.cu) pays a TMEM allocation, an mbarrier ring, a TMA round trip and —
// for projections with fewer 128-row tiles than SMs — a cluster DSMEM reduction, ~4 us of
// fixed cost per launch against 0.3-3 us of bytes (profiles/r1_ncu_full_c2_decode.json).
// This kernel has none of that:
//   * W is read straight from the tile-packed layout into registers with 128-bit
//     ld.global.nc.L1::no_allocate loads: a warp owns 16 weight rows, and the 16 x 64
//     sub-tile of one k-block is 2 KiB contiguous in the packed chunk (fully coalesced).
//   * The first kDepth k-blocks of weights are requested BEFORE griddepcontrol.wait, so
//     under programmatic dependent launch the weight fetch overlaps the previous kernel.
//   * The register fragments are consumed by legacy warp MMAs (mma.sync m16n8k16, rows =
//     weight rows, n = tokens): each thread's 16-byte chunk holds 8 consecutive k of one
//     row, and a fixed k-permutation shared by A and B maps two chunks onto four k16 steps,
//     so no shuffles or shared-memory staging are needed.
//   * X fragments come from L2/L1 (shared by the row-warps of a CTA); optionally X is
//     RMS-normalised on the fly (fused pre-norm: the CTA computes 1/rms per token with the
//     same operation order as rmsnorm_kernel, so the product is bit-identical).
//   * CTA = 8 or 16 warps = RW row-warps x KW k-warps; the KW partial sums are reduced in shared
//     memory in a fixed order (deterministic) and the epilogue (bias / residual / SiLU·mul /
//     fp32 + greedy-argmax key / QKV bias+RoPE+paged K/V append) is applied by the CTA.
#include <cuda_runtime.h>

#include <algorithm>

#include "epi.cuh"
#include "gemm.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace asb {

namespace {


__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                               uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int NT, int WARPS>
struct DgCfg {
    // k-blocks of W (and X) in flight per warp: W 16 regs + X 8*NT regs per stage
    static constexpr int kDepth = NT == 1 ? 4 : (NT == 2 ? 2 : 2);
    // register budget: 128 (8 warps x 2 CTAs or 16 warps x 1) / 255 (8 warps x 1)
    static constexpr int kMinBlocks = (NT <= 2 && WARPS == 8) ? 2 : 1;
    static constexpr int kThreads = WARPS * 32;
    static constexpr int kTS = 8 * NT;  // token stride of the reduction buffer
};

// Thread (g = lane/4, t = lane%4) of a warp owning weight rows r0..r0+15:
//   w[0] = W[r0+g][kb*64 + 8t .. +8]      w[1] = W[r0+g][kb*64 + 32 + 8t .. +8]
//   w[2] = W[r0+g+8][same as w[0]]        w[3] = W[r0+g+8][same as w[1]]
// k16 step s uses chunk c = s/2 (0: w[0]/w[2], 1: w[1]/w[3]) and half h = s%2 (words
// {x,y} or {z,w}); the B fragment of token 8j+g takes the same words of X, so A and B see the
// same k-permutation and the dot product is exact up to fp32 summation order.
// Pipeline: stage s of a kDepth-deep register ring holds W and raw X of one k-block.  W of the
// first kDepth blocks is requested before griddepcontrol.wait, X right after it (together with
// the RMSNorm statistics), so the warp waits for one L2 round trip, not one per k-block.
template <int NT, int WARPS>
__global__ void __launch_bounds__(WARPS * 32, (DgCfg<NT, WARPS>::kMinBlocks)) dgemv_kernel(const DgemvParams p) {
    using C = DgCfg<NT, WARPS>;
    constexpr int D = C::kDepth;
    constexpr int kThreadsG = C::kThreads;
    __shared__ float red[WARPS * 16 * C::kTS];  // [kw][row in CTA][token]
    __shared__ float inv_s[32];
    __shared__ unsigned long long key_s[32];

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int RW = p.rw, KW = WARPS / p.rw;
    const int rw = warp % RW, kw = warp / RW;
    const int R = 16 * RW;
    const int row_cta = blockIdx.x * R;
    // rows of this warp: consecutive 16-row slabs, except for the fused RoPE epilogue, where a
    // CTA (RW = 2) owns slab c of the first half of head `hq_` and the same slab of the second
    // half, so every rotate_half pair (j, j + hd/2) is reduced inside the CTA
    // (RW/2 pairs per CTA: warp rw serves half rw % 2 of pair unit blockIdx.x * RW/2 + rw / 2)
    const int spp = p.epi == EPI_QKV ? p.rope.hd / 32 : 1;  // slabs per half head
    const int unit_ = blockIdx.x * (RW / 2) + rw / 2;
    const int head_ = unit_ / spp, slab_ = unit_ % spp;
    const int r0 = p.epi == EPI_QKV ? (unit_ < p.n_out / 32 ? head_ * p.rope.hd + (rw & 1) * (p.rope.hd / 2) + 16 * slab_
                                                            : p.rows_pad)
                                    : row_cta + 16 * rw;
    const int KB = p.K / 64;
    const bool rows_ok = r0 < p.rows_pad;
    const int nk = rows_ok && kw < KB ? (KB - kw + KW - 1) / KW : 0;
    // packed chunk of (row tile r0/128, k-block kb) + this warp's 16-row slab + thread offset
    const __nv_bfloat16* wbase = p.w + (size_t)(r0 >> 7) * KB * 8192 + (size_t)(r0 & 127) * 64;
    const int toff0 = g * 64 + 8 * t, toff1 = (g + 8) * 64 + 8 * t;

    uint4 wr[D][4];
    uint4 xr[D][NT][2];
    auto load_w = [&](uint4 (&w)[4], int i) {
        const __nv_bfloat16* c = wbase + (size_t)(kw + i * KW) * 8192;
        w[0] = ldg_stream(c + toff0);
        w[1] = ldg_stream(c + toff0 + 32);
        w[2] = ldg_stream(c + toff1);
        w[3] = ldg_stream(c + toff1 + 32);
    };
#pragma unroll
    for (int s = 0; s < D; ++s)
        if (s < nk) load_w(wr[s], s);

    pdl_trigger();
    pdl_wait();  // X (and the residual / output buffers) belong to the previous kernels

    // per n-tile token rows of this thread (g-th token of tile j)
    const __nv_bfloat16* xrow[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const int tok = 8 * j + g;
        const int src = tok < p.T ? (p.x_rows ? p.x_rows[tok] : tok) : -1;
        xrow[j] = src >= 0 ? p.x + (size_t)src * p.ldx : nullptr;
    }
    auto load_x = [&](uint4 (&x)[NT][2], int i) {
        const int k0 = (kw + i * KW) * 64 + 8 * t;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            if (xrow[j]) {
                x[j][0] = *reinterpret_cast<const uint4*>(xrow[j] + k0);
                x[j][1] = *reinterpret_cast<const uint4*>(xrow[j] + k0 + 32);
            } else {
                x[j][0] = x[j][1] = make_uint4(0u, 0u, 0u, 0u);
            }
        }
    };
#pragma unroll
    for (int s = 0; s < D; ++s)
        if (s < nk) load_x(xr[s], s);

    if (p.norm_w) {
        for (int tok = warp; tok < p.T; tok += WARPS) {
            const int src = p.x_rows ? p.x_rows[tok] : tok;
            const float inv = rms_inv_warp(p.x + (size_t)src * p.ldx, p.K, p.eps, lane);
            if (lane == 0) inv_s[tok] = inv;
        }
    }
    if (p.epi == EPI_F32 && p.amax && threadIdx.x < 32) key_s[threadIdx.x] = 0ull;
    if (p.norm_w) __syncthreads();
    float inv_r[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) inv_r[j] = (p.norm_w && 8 * j + g < p.T) ? inv_s[8 * j + g] : 0.f;

    float acc[NT][4];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;

    auto compute = [&](const uint4 (&w)[4], uint4 (&x)[NT][2], int i) {
        if (p.norm_w) {
            const int k0 = (kw + i * KW) * 64 + 8 * t;
            const uint4 gm[2] = {*reinterpret_cast<const uint4*>(p.norm_w + k0),
                                 *reinterpret_cast<const uint4*>(p.norm_w + k0 + 32)};
#pragma unroll
            for (int j = 0; j < NT; ++j) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    x[j][c].x = rms_apply2(x[j][c].x, gm[c].x, inv_r[j]);
                    x[j][c].y = rms_apply2(x[j][c].y, gm[c].y, inv_r[j]);
                    x[j][c].z = rms_apply2(x[j][c].z, gm[c].z, inv_r[j]);
                    x[j][c].w = rms_apply2(x[j][c].w, gm[c].w, inv_r[j]);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                mma_bf16_16816(acc[j], w[c].x, w[c + 2].x, w[c].y, w[c + 2].y, x[j][c].x, x[j][c].y);
                mma_bf16_16816(acc[j], w[c].z, w[c + 2].z, w[c].w, w[c + 2].w, x[j][c].z, x[j][c].w);
            }
        }
    };

    for (int i0 = 0; i0 < nk; i0 += D) {
#pragma unroll
        for (int s = 0; s < D; ++s) {
            const int i = i0 + s;
            if (i < nk) {
                compute(wr[s], xr[s], i);
                if (i + D < nk) {
                    load_w(wr[s], i + D);
                    load_x(xr[s], i + D);
                }
            }
        }
    }

    // ---- reduce the KW k-partials: red[kw][rl][tok]
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const int rl = 16 * rw + g;
        const int tk = 8 * j + 2 * t;
        float* b = red + (size_t)(kw * R) * C::kTS;
        b[rl * C::kTS + tk] = acc[j][0];
        b[rl * C::kTS + tk + 1] = acc[j][1];
        b[(rl + 8) * C::kTS + tk] = acc[j][2];
        b[(rl + 8) * C::kTS + tk + 1] = acc[j][3];
    }
    __syncthreads();
    auto sum = [&](int rl, int tok) {
        float v = 0.f;
        for (int q = 0; q < KW; ++q) v += red[(q * R + rl) * C::kTS + tok];
        return v;
    };

    const int T = p.T;
    switch (p.epi) {
    case EPI_SILU: {
        // interleaved gate/up rows (2j, 2j+1) -> output column j
        const int np = R / 2;
        for (int e = threadIdx.x; e < np * T; e += kThreadsG) {
            const int pr = e % np, tok = e / np;
            const int n = row_cta + 2 * pr;
            if (n + 1 >= p.n_out) continue;
            p.out[(size_t)tok * p.ldo + (n >> 1)] = __float2bfloat16_rn(silu(sum(2 * pr, tok)) * sum(2 * pr + 1, tok));
        }
        break;
    }
    case EPI_QKV: {
        // pair-slab CTA: red rows [32 pi, 32 pi + 16) = features f1 = head*hd + 16c + j of the
        // first half of pair unit pi, rows [32 pi + 16, 32 pi + 32) = f1 + hd/2.  q/k heads
        // rotate the pair, v heads copy it.
        const RopeEpi& Rp = p.rope;
        const int hd = Rp.hd, H = hd / 2, qd = Rp.hq * hd, kvd = Rp.hkv * hd;
        const int P = RW / 2;
        for (int e = threadIdx.x; e < P * 16 * T; e += kThreadsG) {
            const int jj = e & 15, pi = (e >> 4) % P, tok = (e >> 4) / P;
            const int u = blockIdx.x * P + pi;
            if (u >= p.n_out / 32) continue;
            const int f0 = (u / spp) * hd, j = 16 * (u % spp) + jj;
            const int sl = Rp.slot[tok];
            float x1 = sum(32 * pi + jj, tok), x2 = sum(32 * pi + 16 + jj, tok);
            if (p.bias) {
                x1 += __bfloat162float(p.bias[f0 + j]);
                x2 += __bfloat162float(p.bias[f0 + j + H]);
            }
            if (f0 >= qd + kvd) {
                __nv_bfloat16* v = Rp.v_pool + pool_off(Rp, sl, (f0 - qd - kvd) / hd);
                v[j] = __float2bfloat16_rn(x1);
                v[j + H] = __float2bfloat16_rn(x2);
                continue;
            }
            const int pos = Rp.pos[tok];
            float y1, y2;
            rope2(bf16r(x1), bf16r(x2), Rp.cos_t[(size_t)pos * H + j], Rp.sin_t[(size_t)pos * H + j], y1, y2);
            __nv_bfloat16* dst = f0 < qd ? Rp.q_out + ((size_t)tok * Rp.hq + f0 / hd) * hd
                                         : Rp.k_pool + pool_off(Rp, sl, (f0 - qd) / hd);
            dst[j] = __float2bfloat16_rn(y1);
            dst[j + H] = __float2bfloat16_rn(y2);
        }
        break;
    }
    default: {
        // <= 16 elements per thread (R x T <= 128 x 32 over >= 256 threads); residual loads all
        // issued before the first (possibly aliasing, in-place) store
        float rv[16];
        if (p.epi == EPI_RESID) {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const int e = threadIdx.x + u * kThreadsG, rl = e % R, tok = e / R, n = row_cta + rl;
                rv[u] = (e < R * T && n < p.n_out) ? __bfloat162float(p.resid[(size_t)tok * p.ldr + n]) : 0.f;
            }
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int e = threadIdx.x + u * kThreadsG;
            if (e >= R * T) break;
            const int rl = e % R, tok = e / R;
            const int n = row_cta + rl;
            if (n >= p.n_out) continue;
            float v = sum(rl, tok);
            const size_t o = (size_t)tok * p.ldo + n;
            if (p.epi == EPI_F32) {
                p.out_f32[o] = v;
                if (p.amax) {
                    const unsigned long long k = argmax_key(v, n);
                    if (k) atomicMax(&key_s[tok], k);
                }
            } else {
                if (p.epi == EPI_RESID) v += rv[u];
                else if (p.bias) v += __bfloat162float(p.bias[n]);
                p.out[o] = __float2bfloat16_rn(v);
            }
        }
        if (p.epi == EPI_F32 && p.amax) {
            __syncthreads();
            if (threadIdx.x < T && key_s[threadIdx.x]) atomicMax(p.amax + threadIdx.x, key_s[threadIdx.x]);
        }
        break;
    }
    }
    // fused next pre-norm (decode steps): the last CTA normalises the updated residual rows
    if (p.post.w && grid_last_arriver(p.post.counter)) post_norm_rows(p.post, p.out, p.ldo);
}

template <int NT, int WARPS>
cudaError_t launch_nt(const DgemvParams& p, int grid, cudaStream_t st) {
    return launch_k(dgemv_kernel<NT, WARPS>, dim3(grid), dim3(WARPS * 32), 0, st, p);
}

template <int WARPS>
cudaError_t launch_w(const DgemvParams& p, int grid, cudaStream_t st) {
    switch ((p.T + 7) / 8) {
    case 1: return launch_nt<1, WARPS>(p, grid, st);
    case 2: return launch_nt<2, WARPS>(p, grid, st);
    case 3: return launch_nt<3, WARPS>(p, grid, st);
    default: return launch_nt<4, WARPS>(p, grid, st);
    }
}

}  // namespace

int dgemv_max_tokens() { return 32; }

cudaError_t dgemv_launch(DgemvParams p, int num_sms, cudaStream_t stream) {
    if (p.T < 1 || p.T > 32 || p.K % 64 != 0) return cudaErrorInvalidValue;
    if (p.epi == EPI_QKV && (p.rope.hd % 32 != 0 || p.n_out % p.rope.hd != 0)) return cudaErrorInvalidValue;
    // Rows per CTA: the fewest (most CTAs, least weight per SM) that still fit ONE wave of
    // resident CTAs -- a second partial wave doubles the latency of these launch-bound
    // projections on a small Green Context partition.  Fused RoPE: pairs of half-head slabs.
    const int tiles16 = (p.n_out + 15) / 16;
    const int slots = num_sms * ((p.T + 7) / 8 <= 2 ? 2 : 1);
    int rw = 1, grid = 0;
    if (p.epi == EPI_QKV) {
        const int pairs = p.n_out / 32;
        int P = 1;
        while (P < 4 && (pairs + P - 1) / P > slots) P *= 2;
        rw = 2 * P;
        grid = (pairs + P - 1) / P;
    } else {
        while (rw < 8 && (tiles16 + rw - 1) / rw > slots) rw *= 2;
        grid = (p.n_out + 16 * rw - 1) / (16 * rw);
    }
    p.rw = rw;
    // a grid that does not fill the SMs gets 16 warps per CTA (twice the K split)
    if (grid <= num_sms) return launch_w<16>(p, grid, stream);
    return launch_w<8>(p, grid, stream);
}

}  // namespace asb
