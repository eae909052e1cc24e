// Paged decode attention (K2 in SURVEY §2.3) — one query token per decode row, all G query
// heads of one KV head per CTA.  HBM-bound: every context token's K and V row is streamed
// exactly once per (row, KV head).  Replaces the mu_D term of the reference's
// decode_step_duration_ms (/root/reference/proj/src/executor.cpp:213-215).
//
// CTA = 1 producer warp + kWarps consumer warps, split-KV over gridDim.z:
//   producer   : 1-D bulk copies (cp.async.bulk, evict-first) of contiguous 32-token K and V
//                sub-blocks ([block][kv_head][64][hd] pool layout) into a kStages-deep smem
//                ring, completion on mbarriers (expect_tx)
//   consumers  : each warp owns whole sub-blocks (no CTA-wide barrier per block); lane l owns
//                head-dim slice [l*DPL, (l+1)*DPL); K slice kept in registers; per head the
//                32 partial dot products are reduce-scattered across lanes (31 shuffles) so
//                lane t ends with key t's score; online softmax per warp; P broadcast through
//                a per-warp smem row; O slice accumulated in registers
//   epilogue   : warps merge (m, l, O) in smem; CTA writes bf16 output (one split) or fp32
//                partials merged by decode_combine_kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>

#include "attn.h"
#include "sm100.cuh"

namespace asb {

namespace {

constexpr int kSub = 32;    // tokens per streamed sub-block (half a KV block)
constexpr int kWarps = 4;   // consumer warps per CTA
constexpr int kThreadsD = (kWarps + 1) * 32;

template <int HD>
struct DC {
    static constexpr int kDpl = HD / 32;                  // head dims per lane
    static constexpr int kSubBytes = kSub * HD * 2;       // one K (or V) sub-block
    static constexpr int kStages = HD == 128 ? 5 : 10;    // 80 KB ring -> 2 CTAs / SM
    static constexpr int kRing = kStages * 2 * kSubBytes;
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// lane l returns sum over lanes of v[l] (reduce-scatter of 32 partials)
__device__ __forceinline__ float reduce_scatter32(float (&v)[32], int lane) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < o; ++k) {
            const float send = up ? v[k] : v[k + o];
            const float keep = up ? v[k + o] : v[k];
            v[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    return v[0];
}

template <int HD, int G>
__global__ void __launch_bounds__(kThreadsD, 2)
    decode_attn_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k_pool,
                       const __nv_bfloat16* __restrict__ v_pool, const DecodeItem* __restrict__ items,
                       const int32_t* __restrict__ tables, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ part_o, float* __restrict__ part_ml, int subs_per_split,
                       AttnShape s) {
    using C = DC<HD>;
    constexpr int DPL = C::kDpl;
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* ring = smem;                                                // [stage][K|V][sub]
    float* pbuf = reinterpret_cast<float*>(smem + C::kRing);             // [warp][32]
    float* qs = pbuf + kWarps * 32;                                      // [G][HD] scaled q
    float* accs = qs + G * HD;                                           // [warp][G][HD]
    float* mls = accs + kWarps * G * HD;                                 // [warp][G][2]
    uint64_t* full = reinterpret_cast<uint64_t*>(mls + kWarps * G * 2 + 2);
    uint64_t* empty = full + C::kStages;

    const DecodeItem it = items[blockIdx.x];
    const int kvh = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_sub = (it.ctx_len + kSub - 1) / kSub;
    const int s0 = blockIdx.z * subs_per_split;
    const int n_local = max(0, min(n_sub, s0 + subs_per_split) - s0);
    const int32_t* table = tables + it.table_off;

    if (threadIdx.x == 0) {
        for (int i = 0; i < C::kStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_barrier_init();
    }
    for (int e = threadIdx.x; e < G * HD; e += blockDim.x)
        qs[e] = __bfloat162float(q[(size_t)it.q_row * s.hq * HD + kvh * G * HD + e]) * s.scale_log2;
    for (int e = threadIdx.x; e < kWarps * G * HD; e += blockDim.x) accs[e] = 0.f;
    for (int e = threadIdx.x; e < kWarps * G; e += blockDim.x) {
        mls[2 * e] = -FLT_MAX;
        mls[2 * e + 1] = 0.f;
    }
    __syncthreads();

    if (warp == kWarps) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int i = 0; i < n_local; ++i) {
                const int st = i % C::kStages;
                mbar_wait(&empty[st], ((i / C::kStages) & 1) ^ 1);
                mbar_expect_tx(&full[st], 2 * C::kSubBytes);
                const int j = s0 + i;
                const int blk = table[j >> 1];
                const size_t off =
                    ((((size_t)s.layer * s.num_blocks + blk) * s.hkv + kvh) * kBlockTokens + (j & 1) * kSub) * HD;
                uint8_t* dst = ring + (size_t)st * 2 * C::kSubBytes;
                bulk_g2s(dst, k_pool + off, C::kSubBytes, &full[st], pol);
                bulk_g2s(dst + C::kSubBytes, v_pool + off, C::kSubBytes, &full[st], pol);
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    // per-head state (q slice, O slice, m, l) lives in smem so the head loop stays rolled and
    // register use is independent of G
    float* prow = pbuf + warp * 32;
    float* wacc = accs + warp * G * HD;
    float* wml = mls + warp * G * 2;
    for (int i = warp; i < n_local; i += kWarps) {
        const int st = i % C::kStages;
        mbar_wait(&full[st], (i / C::kStages) & 1);
        const uint8_t* kt = ring + (size_t)st * 2 * C::kSubBytes;
        const uint8_t* vt = kt + C::kSubBytes;
        const int kbase = (s0 + i) * kSub;
        const bool valid = kbase + lane < it.ctx_len;
        // K slice of all 32 keys in registers, packed bf16x2 (lane's DPL dims of each row)
        uint32_t kw[kSub][DPL / 2];
#pragma unroll
        for (int t = 0; t < kSub; ++t) {
            if constexpr (DPL == 4) {
                const uint2 w = *reinterpret_cast<const uint2*>(kt + (t * HD + lane * 4) * 2);
                kw[t][0] = w.x;
                kw[t][1] = w.y;
            } else {
                kw[t][0] = *reinterpret_cast<const uint32_t*>(kt + (t * HD + lane * 2) * 2);
            }
        }
#pragma unroll 1
        for (int g = 0; g < G; ++g) {
            float qv[DPL], acc[DPL];
            if constexpr (DPL == 4) {
                const float4 a = *reinterpret_cast<const float4*>(qs + g * HD + lane * 4);
                qv[0] = a.x; qv[1] = a.y; qv[2] = a.z; qv[3] = a.w;
                const float4 c = *reinterpret_cast<const float4*>(wacc + g * HD + lane * 4);
                acc[0] = c.x; acc[1] = c.y; acc[2] = c.z; acc[3] = c.w;
            } else {
                const float2 a = *reinterpret_cast<const float2*>(qs + g * HD + lane * 2);
                qv[0] = a.x; qv[1] = a.y;
                const float2 c = *reinterpret_cast<const float2*>(wacc + g * HD + lane * 2);
                acc[0] = c.x; acc[1] = c.y;
            }
            float part[kSub];
#pragma unroll
            for (int t = 0; t < kSub; ++t) {
                float a = 0.f;
#pragma unroll
                for (int d2 = 0; d2 < DPL / 2; ++d2) {
                    a = fmaf(qv[2 * d2], bf16_lo(kw[t][d2]), a);
                    a = fmaf(qv[2 * d2 + 1], bf16_hi(kw[t][d2]), a);
                }
                part[t] = a;
            }
            const float red = reduce_scatter32(part, lane);  // all lanes take part in the shuffles
            const float sc = valid ? red : -FLT_MAX;
            float mx = sc;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float m_old = wml[2 * g];
            const float m_new = fmaxf(m_old, mx);
            const float p = valid ? exp2f(sc - m_new) : 0.f;
            float sum = p;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            const float alpha = exp2f(m_old - m_new);
            prow[lane] = p;
            __syncwarp();
#pragma unroll
            for (int d = 0; d < DPL; ++d) acc[d] *= alpha;
#pragma unroll
            for (int t = 0; t < kSub; t += 4) {
                const float4 p4 = *reinterpret_cast<const float4*>(prow + t);
                const float pp[4] = {p4.x, p4.y, p4.z, p4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if constexpr (DPL == 4) {
                        const uint2 w = *reinterpret_cast<const uint2*>(vt + ((t + u) * HD + lane * 4) * 2);
                        acc[0] = fmaf(pp[u], bf16_lo(w.x), acc[0]);
                        acc[1] = fmaf(pp[u], bf16_hi(w.x), acc[1]);
                        acc[2] = fmaf(pp[u], bf16_lo(w.y), acc[2]);
                        acc[3] = fmaf(pp[u], bf16_hi(w.y), acc[3]);
                    } else {
                        const uint32_t w = *reinterpret_cast<const uint32_t*>(vt + ((t + u) * HD + lane * 2) * 2);
                        acc[0] = fmaf(pp[u], bf16_lo(w), acc[0]);
                        acc[1] = fmaf(pp[u], bf16_hi(w), acc[1]);
                    }
                }
            }
            if constexpr (DPL == 4) {
                *reinterpret_cast<float4*>(wacc + g * HD + lane * 4) = make_float4(acc[0], acc[1], acc[2], acc[3]);
            } else {
                *reinterpret_cast<float2*>(wacc + g * HD + lane * 2) = make_float2(acc[0], acc[1]);
            }
            __syncwarp();  // prow / wml reads of this head are done before they are overwritten
            if (lane == 0) {
                wml[2 * g] = m_new;
                wml[2 * g + 1] = wml[2 * g + 1] * alpha + sum;
            }
            __syncwarp();
        }
        if (lane == 0) mbar_arrive(&empty[st]);
    }

    // ---------------------------------------------------------------- merge warps
    named_sync(1, kWarps * 32);
    const bool single = gridDim.z == 1;
    for (int e = threadIdx.x; e < G * HD; e += kWarps * 32) {
        const int g = e / HD, d = e % HD;
        float M = -FLT_MAX;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, mls[(w * G + g) * 2]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float lw = mls[(w * G + g) * 2 + 1];
            if (lw == 0.f) continue;
            const float f = exp2f(mls[(w * G + g) * 2] - M);
            L += lw * f;
            O += accs[(w * G + g) * HD + d] * f;
        }
        const int h = kvh * G + g;
        if (single) {
            out[(size_t)it.q_row * s.hq * HD + h * HD + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
        } else {
            const size_t slot = ((size_t)blockIdx.x * s.hq + h) * gridDim.z + blockIdx.z;
            part_o[slot * HD + d] = O;
            if (d == 0) {
                part_ml[slot * 2 + 0] = M;
                part_ml[slot * 2 + 1] = L;
            }
        }
    }
}

// Merge split partials -> normalised bf16 output.  grid = (n_items, hq), block = HD.
template <int HD>
__global__ void decode_combine_kernel(const DecodeItem* __restrict__ items,
                                      const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml, int splits,
                                      __nv_bfloat16* __restrict__ out, int hq) {
    const int row = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
    const size_t base = ((size_t)row * hq + h) * splits;
    float M = -FLT_MAX;
    for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, part_ml[(base + sp) * 2]);
    float L = 0.f, O = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
        const float ls = part_ml[(base + sp) * 2 + 1];
        if (ls == 0.f) continue;
        const float w = exp2f(part_ml[(base + sp) * 2] - M);
        L += ls * w;
        O += part_o[(base + sp) * HD + d] * w;
    }
    out[(size_t)items[row].q_row * hq * HD + h * HD + d] = __float2bfloat16_rn(O / L);
}

template <int HD, int G>
cudaError_t launch_g(const __nv_bfloat16* q, const __nv_bfloat16* kp, const __nv_bfloat16* vp,
                     const DecodeItem* items, int n_items, int splits, int sps, const int32_t* tables,
                     __nv_bfloat16* out, float* po, float* pml, const AttnShape& s, cudaStream_t st) {
    using C = DC<HD>;
    constexpr int smem = C::kRing + kWarps * 32 * 4 + G * HD * 4 + kWarps * G * HD * 4 +
                         (kWarps * G * 2 + 2) * 4 + 2 * C::kStages * 8;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<HD, G>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid(n_items, s.hkv, splits);
    decode_attn_kernel<HD, G><<<grid, kThreadsD, smem, st>>>(q, kp, vp, items, tables, out, po, pml, sps, s);
    if (splits > 1)
        decode_combine_kernel<HD><<<dim3(n_items, s.hq), HD, 0, st>>>(items, po, pml, splits, out, s.hq);
    return cudaGetLastError();
}

template <int HD>
cudaError_t launch_hd(int G, const __nv_bfloat16* q, const __nv_bfloat16* kp, const __nv_bfloat16* vp,
                      const DecodeItem* items, int n_items, int splits, int sps, const int32_t* tables,
                      __nv_bfloat16* out, float* po, float* pml, const AttnShape& s, cudaStream_t st) {
    switch (G) {
    case 1: return launch_g<HD, 1>(q, kp, vp, items, n_items, splits, sps, tables, out, po, pml, s, st);
    case 2: return launch_g<HD, 2>(q, kp, vp, items, n_items, splits, sps, tables, out, po, pml, s, st);
    case 3: return launch_g<HD, 3>(q, kp, vp, items, n_items, splits, sps, tables, out, po, pml, s, st);
    case 4: return launch_g<HD, 4>(q, kp, vp, items, n_items, splits, sps, tables, out, po, pml, s, st);
    case 5: return launch_g<HD, 5>(q, kp, vp, items, n_items, splits, sps, tables, out, po, pml, s, st);
    case 6: return launch_g<HD, 6>(q, kp, vp, items, n_items, splits, sps, tables, out, po, pml, s, st);
    case 7: return launch_g<HD, 7>(q, kp, vp, items, n_items, splits, sps, tables, out, po, pml, s, st);
    case 8: return launch_g<HD, 8>(q, kp, vp, items, n_items, splits, sps, tables, out, po, pml, s, st);
    default: return cudaErrorInvalidValue;
    }
}

}  // namespace

int decode_splits(int n_items, int hkv, int max_ctx, int num_sms, int max_splits) {
    // aim for ~4 resident CTAs per SM-pair worth of work, >= 2 sub-blocks per consumer warp
    const int subs = (max_ctx + kSub - 1) / kSub;
    const int base = n_items * hkv;
    int splits = (4 * num_sms + base - 1) / std::max(base, 1);
    splits = std::min(splits, std::max(1, subs / (2 * kWarps)));
    splits = std::min(splits, max_splits);
    return std::max(splits, 1);
}

cudaError_t decode_attention(const __nv_bfloat16* q, const __nv_bfloat16* k_pool,
                             const __nv_bfloat16* v_pool, const DecodeItem* items, int n_items,
                             int max_ctx, const int32_t* tables, __nv_bfloat16* out,
                             float* part_o, float* part_ml, int max_splits, int num_sms,
                             const AttnShape& s, cudaStream_t stream) {
    if (n_items <= 0) return cudaSuccess;
    const int G = s.hq / s.hkv;
    const int splits0 = decode_splits(n_items, s.hkv, max_ctx, num_sms, max_splits);
    const int subs = (max_ctx + kSub - 1) / kSub;
    const int sps = (subs + splits0 - 1) / splits0;
    const int splits = (subs + sps - 1) / sps;
    if (s.hd == 128)
        return launch_hd<128>(G, q, k_pool, v_pool, items, n_items, splits, sps, tables, out, part_o,
                              part_ml, s, stream);
    if (s.hd == 64)
        return launch_hd<64>(G, q, k_pool, v_pool, items, n_items, splits, sps, tables, out, part_o,
                             part_ml, s, stream);
    return cudaErrorInvalidValue;
}

}  // namespace asb
