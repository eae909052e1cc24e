// Attention over the paged KV cache.
//
// * prefill_attention_kernel (K4/K3 in SURVEY §2.3): causal flash attention for cold and
//   resume prefills and for the admitted resume chunk inside a decode step.  GQA-packed:
//   the 128 MMA rows of a CTA are (token, query head) pairs of ONE KV head, so each K/V
//   block is loaded once for all G query heads (3-D TMA box for Q); split-KV over
//   gridDim.z when the grid is small.  S = Q.K^T and O_blk = P.V run on tcgen05 (TMEM),
//   K/V blocks arrive by TMA straight from the paged pool, softmax is one thread per
//   query row (the TMEM lane it owns).  Replaces the prefill rate x length term of
//   /root/reference/proj/src/engine.cpp:450-475 and the mu_R chunk term of
//   /root/reference/proj/src/executor.cpp:216-218.
// * decode_attention_kernel (K2): one query token per row, all GQA heads of one KV head
//   per CTA, split-K over KV blocks, cp.async double-buffered 128-bit loads, warp-shuffle
//   softmax.  HBM-bound; replaces the mu_D term of executor.cpp:213-215.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>

#include "attn.h"
#include "sm100.cuh"

namespace asb {

namespace {

// ============================================================================ prefill
constexpr int kPThreads = 192;
constexpr int kKvStages = 3;

template <int HD>
struct PCfg {
    static constexpr int kHalves = HD / 64;
    static constexpr int kQBytes = 128 * HD * 2;
    static constexpr int kKBytes = kBlockTokens * HD * 2;
    static constexpr int kStageBytes = 2 * kKBytes;  // K then V
    static constexpr int kPBytes = 128 * kBlockTokens * 2;
    static constexpr int kSmem = kQBytes + kKvStages * kStageBytes + kPBytes + 1024 + 256;
    static constexpr int kTmemCols = 256;  // S0 | S1 | O (HD <= 128)
};

template <int HD>
__global__ void __launch_bounds__(kPThreads, 1)
    prefill_attention_kernel(const __grid_constant__ CUtensorMap tmap_q,
                             const __grid_constant__ CUtensorMap tmap_k,
                             const __grid_constant__ CUtensorMap tmap_v,
                             const PrefillItem* __restrict__ items,
                             const int32_t* __restrict__ tables, __nv_bfloat16* __restrict__ out,
                             float* __restrict__ part_o, float* __restrict__ part_ml,
                             int blocks_per_split, const AttnShape s) {
    using C = PCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
    uint8_t* sq = smem;
    uint8_t* skv = sq + C::kQBytes;
    uint8_t* sp = skv + kKvStages * C::kStageBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sp + C::kPBytes);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;               // [kKvStages]
    uint64_t* kv_empty = kv_full + kKvStages;   // [kKvStages]
    uint64_t* s_full = kv_empty + kKvStages;    // [2]
    uint64_t* s_free = s_full + 2;              // [2]
    uint64_t* p_full = s_free + 2;
    uint64_t* o_full = p_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

    const PrefillItem it = items[blockIdx.x];
    const int kvh = blockIdx.y;
    const int G = s.hq / s.hkv;
    const int n_rows = it.n_q * G;  // valid MMA rows: (token, head-in-group)
    const int total_blocks = (it.q_pos0 + it.n_q + kBlockTokens - 1) / kBlockTokens;
    // split-KV (gridDim.z > 1): this CTA covers KV blocks [blk0, blk0 + n_kv_blocks)
    const int blk0 = blockIdx.z * blocks_per_split;
    const int n_kv_blocks = max(0, min(total_blocks, blk0 + blocks_per_split) - blk0);
    const bool split = gridDim.z > 1;
    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    if (n_kv_blocks == 0) {
        // empty split: neutral partials for the valid rows
        const size_t base = (static_cast<size_t>(blockIdx.x) * gridDim.y + kvh) * gridDim.z + blockIdx.z;
        for (int r = threadIdx.x; r < n_rows; r += blockDim.x) {
            part_ml[(base * 128 + r) * 2 + 0] = -FLT_MAX;
            part_ml[(base * 128 + r) * 2 + 1] = 0.f;
        }
        return;
    }

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_q);
        tma_prefetch_desc(&tmap_k);
        tma_prefetch_desc(&tmap_v);
        mbar_init(q_full, 1);
        for (int i = 0; i < kKvStages; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&s_free[i], 128);
        }
        mbar_init(p_full, 128);
        mbar_init(o_full, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    // The Q box covers (128 / G) * G rows; the remaining (< G) rows stay zero so their
    // (discarded) outputs are finite.
    const int box_rows = (128 / G) * G;
    for (int i = threadIdx.x; i < C::kHalves * (128 - box_rows) * 8; i += blockDim.x) {
        const int h = i / ((128 - box_rows) * 8), rem = i % ((128 - box_rows) * 8);
        reinterpret_cast<uint4*>(sq + h * (128 * 128) + (box_rows + rem / 8) * 128)[rem % 8] = make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int32_t* table = tables + it.table_off;

    if (warp == 0) {
        if (elect_one()) {
            mbar_expect_tx(q_full, C::kHalves * box_rows * 128);  // full box, incl. OOB fill
#pragma unroll
            for (int h = 0; h < C::kHalves; ++h)
                tma_load_3d(sq + h * (128 * 128), &tmap_q, q_full, h * 64, kvh * G, it.q_row0);
            const uint64_t pol = policy_evict_last();  // K/V blocks are re-read by other heads
            for (int j = 0; j < n_kv_blocks; ++j) {
                const int st = j % kKvStages;
                const uint32_t ph = (j / kKvStages) & 1;
                mbar_wait(&kv_empty[st], ph ^ 1);
                mbar_expect_tx(&kv_full[st], C::kStageBytes);
                const int blk = table[blk0 + j];
                const int row =
                    ((s.layer * s.num_blocks + blk) * s.hkv + kvh) * kBlockTokens;
                uint8_t* kdst = skv + st * C::kStageBytes;
                uint8_t* vdst = kdst + C::kKBytes;
#pragma unroll
                for (int h = 0; h < C::kHalves; ++h) {
                    tma_load_2d_hint(kdst + h * (kBlockTokens * 128), &tmap_k, &kv_full[st],
                                     h * 64, row, pol);
                    tma_load_2d_hint(vdst + h * (kBlockTokens * 128), &tmap_v, &kv_full[st],
                                     h * 64, row, pol);
                }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc_s = make_idesc_bf16(128, kBlockTokens, false, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(128, HD, false, true);
        const uint32_t q_addr = smem_u32(sq);
        const uint32_t p_addr = smem_u32(sp);
        mbar_wait(q_full, 0);
        auto issue_s = [&](int j) {
            const int st = j % kKvStages;
            const int sb = j & 1;
            mbar_wait(&kv_full[st], (j / kKvStages) & 1);
            if (j >= 2) mbar_wait(&s_free[sb], ((j - 2) >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t k_addr = smem_u32(skv + st * C::kStageBytes);
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const int h = k / 4, kk = k % 4;
                    const uint64_t ad = make_sw128_desc(q_addr + h * 16384 + kk * 32, 16, 1024);
                    const uint64_t bd =
                        make_sw128_desc(k_addr + h * (kBlockTokens * 128) + kk * 32, 16, 1024);
                    umma_bf16(tmem + sb * kBlockTokens, ad, bd, idesc_s, k > 0 ? 1u : 0u);
                }
                umma_commit(&s_full[sb]);
            }
            __syncwarp();
        };
        auto issue_pv = [&](int j) {
            const int st = j % kKvStages;
            mbar_wait(p_full, j & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t v_addr = smem_u32(skv + st * C::kStageBytes + C::kKBytes);
#pragma unroll
                for (int k = 0; k < kBlockTokens / 16; ++k) {
                    const uint64_t ad = make_sw128_desc(p_addr + k * 32, 16, 1024);
                    // V is MN-major (head_dim contiguous): LBO = distance between 64-wide
                    // head_dim atoms, SBO = 8 key rows; 16 keys per MMA = 2048 bytes.
                    const uint64_t bd =
                        make_sw128_desc(v_addr + k * 2048, kBlockTokens * 128, 1024);
                    umma_bf16(tmem + 2 * kBlockTokens, ad, bd, idesc_o, k > 0 ? 1u : 0u);
                }
                umma_commit(o_full);
                umma_commit(&kv_empty[st]);
            }
            __syncwarp();
        };
        issue_s(0);
        for (int j = 1; j < n_kv_blocks; ++j) {
            issue_s(j);
            issue_pv(j - 1);
        }
        issue_pv(n_kv_blocks - 1);
    } else {
        // Softmax / correction warps: one query row per thread.
        const uint32_t quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const int qpos = it.q_pos0 + r / G;  // row r = (token r / G, head kvh*G + r % G)
        const uint32_t t_lane = tmem + ((quarter * 32u) << 16);
        float o[HD];
#pragma unroll
        for (int d = 0; d < HD; ++d) o[d] = 0.f;
        float m_run = -FLT_MAX, l_run = 0.f, alpha_prev = 1.f;
        uint8_t* prow = sp + r * 128;
        for (int j = 0; j < n_kv_blocks; ++j) {
            const int sb = j & 1;
            mbar_wait(&s_full[sb], (j >> 1) & 1);
            tc_fence_after();
            uint32_t sa[32], sb2[32];
            tmem_ld32(t_lane + sb * kBlockTokens, sa);
            tmem_ld32(t_lane + sb * kBlockTokens + 32, sb2);
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(&s_free[sb]);
            // mask + scale (log2 domain)
            const int kbase = (blk0 + j) * kBlockTokens;
            float mx = m_run;
            float sv[64];
#pragma unroll
            for (int c = 0; c < 64; ++c) {
                const float x = __uint_as_float(c < 32 ? sa[c] : sb2[c - 32]) * s.scale_log2;
                sv[c] = (kbase + c <= qpos) ? x : -FLT_MAX;
                mx = fmaxf(mx, sv[c]);
            }
            const float alpha = exp2f(m_run - mx);
            float psum = 0.f;
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const float p0 = (kbase + 2 * c <= qpos) ? exp2f(sv[2 * c] - mx) : 0.f;
                const float p1 = (kbase + 2 * c + 1 <= qpos) ? exp2f(sv[2 * c + 1] - mx) : 0.f;
                const uint32_t packed = pack_bf16(p0, p1);
                // accumulate the rounded probabilities so l matches what P.V sums
                psum += bf16_lo(packed) + bf16_hi(packed);
                pk[c] = packed;
            }
            l_run = l_run * alpha + psum;
            m_run = mx;
            if (j >= 1) {
                // fold in P_{j-1}.V_{j-1}
                mbar_wait(o_full, (j - 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int c = 0; c < HD; c += 32) {
                    uint32_t ov[32];
                    tmem_ld32(t_lane + 2 * kBlockTokens + c, ov);
                    tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e)
                        o[c + e] = o[c + e] * alpha_prev + __uint_as_float(ov[e]);
                }
                tc_fence_before();
            }
            alpha_prev = alpha;
            // P row -> smem (K-major SWIZZLE_128B: chunk c of row r at (c ^ (r & 7)))
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                uint4 v;
                v.x = pk[4 * c + 0];
                v.y = pk[4 * c + 1];
                v.z = pk[4 * c + 2];
                v.w = pk[4 * c + 3];
                *reinterpret_cast<uint4*>(prow + ((c ^ (r & 7)) * 16)) = v;
            }
            fence_proxy_async_smem();
            mbar_arrive(p_full);
        }
        mbar_wait(o_full, (n_kv_blocks - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int c = 0; c < HD; c += 32) {
            uint32_t ov[32];
            tmem_ld32(t_lane + 2 * kBlockTokens + c, ov);
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[c + e] = o[c + e] * alpha_prev + __uint_as_float(ov[e]);
        }
        tc_fence_before();
        if (split) {
            if (r < n_rows) {
                const size_t base =
                    ((static_cast<size_t>(blockIdx.x) * gridDim.y + kvh) * gridDim.z + blockIdx.z) * 128 + r;
                float4* po = reinterpret_cast<float4*>(part_o + base * HD);
#pragma unroll
                for (int c = 0; c < HD / 4; ++c)
                    po[c] = make_float4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
                part_ml[base * 2 + 0] = m_run;
                part_ml[base * 2 + 1] = l_run;
            }
        } else if (r < n_rows) {
            const float inv = 1.f / l_run;
            uint4* dst = reinterpret_cast<uint4*>(
                out + static_cast<size_t>(it.q_row0 + r / G) * (s.hq * HD) + (kvh * G + r % G) * HD);
#pragma unroll
            for (int c = 0; c < HD / 8; ++c) {
                uint4 v;
                v.x = pack_bf16(o[8 * c + 0] * inv, o[8 * c + 1] * inv);
                v.y = pack_bf16(o[8 * c + 2] * inv, o[8 * c + 3] * inv);
                v.z = pack_bf16(o[8 * c + 4] * inv, o[8 * c + 5] * inv);
                v.w = pack_bf16(o[8 * c + 6] * inv, o[8 * c + 7] * inv);
                dst[c] = v;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem);
    }
}

// ============================================================================ decode
constexpr int kDThreads = 128;
constexpr int kMaxGroup = 8;

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int HD>
__global__ void decode_attention_kernel(const __nv_bfloat16* __restrict__ q,
                                        const __nv_bfloat16* __restrict__ k_pool,
                                        const __nv_bfloat16* __restrict__ v_pool,
                                        const DecodeItem* __restrict__ items,
                                        const int32_t* __restrict__ tables, float* __restrict__ part_o,
                                        float* __restrict__ part_ml, int blocks_per_split, AttnShape s);

template <int HD>
struct DCfg {
    static constexpr int kRow = HD + 8;  // padded smem row (bf16) -> conflict-free 16B reads
    static constexpr int kTile = kBlockTokens * kRow;  // elements per K (or V) tile
    static constexpr int kSmem = 4 * kTile * 2 + kMaxGroup * HD * 4 + kMaxGroup * kBlockTokens * 4;
};

template <int HD>
cudaError_t decode_prepare() {
    static bool done = false;
    if (done) return cudaSuccess;
    done = true;
    return cudaFuncSetAttribute(decode_attention_kernel<HD>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, DCfg<HD>::kSmem);
}

// grid = (n_items, hkv, splits); each CTA: all G query heads of one KV head, a range
// of KV blocks.  Writes un-normalised partial O plus (m, l) per head.
template <int HD>
__global__ void __launch_bounds__(kDThreads)
    decode_attention_kernel(const __nv_bfloat16* __restrict__ q,
                            const __nv_bfloat16* __restrict__ k_pool,
                            const __nv_bfloat16* __restrict__ v_pool,
                            const DecodeItem* __restrict__ items,
                            const int32_t* __restrict__ tables, float* __restrict__ part_o,
                            float* __restrict__ part_ml, int blocks_per_split, AttnShape s) {
    using C = DCfg<HD>;
    extern __shared__ __align__(16) uint8_t dsmem[];
    auto sk = reinterpret_cast<__nv_bfloat16(*)[C::kTile]>(dsmem);
    auto sv = reinterpret_cast<__nv_bfloat16(*)[C::kTile]>(dsmem + 2 * C::kTile * 2);
    auto sq = reinterpret_cast<float(*)[HD]>(dsmem + 4 * C::kTile * 2);
    auto sp = reinterpret_cast<float(*)[kBlockTokens]>(dsmem + 4 * C::kTile * 2 +
                                                         kMaxGroup * HD * 4);
    __shared__ float s_alpha[kMaxGroup], s_m[kMaxGroup], s_l[kMaxGroup];

    const DecodeItem it = items[blockIdx.x];
    const int kvh = blockIdx.y;
    const int split = blockIdx.z;
    const int G = s.hq / s.hkv;
    const int tid = threadIdx.x;
    const int n_blocks = (it.ctx_len + kBlockTokens - 1) / kBlockTokens;
    const int b0 = split * blocks_per_split;
    const int b1 = min(n_blocks, b0 + blocks_per_split);
    const int32_t* table = tables + it.table_off;
    const size_t head_tile = static_cast<size_t>(kBlockTokens) * HD;

    // q (bf16) -> fp32 smem, pre-scaled into the log2 domain
    for (int i = tid; i < G * HD; i += kDThreads) {
        const int g = i / HD, d = i % HD;
        sq[g][d] = __bfloat162float(
                       q[static_cast<size_t>(it.q_row) * s.hq * HD + (kvh * G + g) * HD + d]) *
                   s.scale_log2;
    }
    if (tid < kMaxGroup) {
        s_m[tid] = -FLT_MAX;
        s_l[tid] = 0.f;
    }

    auto load_block = [&](int b, int buf) {
        const int blk = table[b];
        const size_t base = ((static_cast<size_t>(s.layer) * s.num_blocks + blk) * s.hkv + kvh) *
                            head_tile;
        const __nv_bfloat16* ks = k_pool + base;
        const __nv_bfloat16* vs = v_pool + base;
        constexpr int kChunks = kBlockTokens * HD / 8;  // 16-byte chunks per tile
#pragma unroll
        for (int c = tid; c < kChunks; c += kDThreads) {
            const int row = c / (HD / 8), col = (c % (HD / 8)) * 8;
            cp_async16(&sk[buf][row * C::kRow + col], ks + row * HD + col);
            cp_async16(&sv[buf][row * C::kRow + col], vs + row * HD + col);
        }
        cp_async_commit();
    };

    // thread ownership
    const int key = tid & (kBlockTokens - 1);
    const int hgrp = tid >> 6;  // 0 / 1: heads hgrp, hgrp+2, ...
    constexpr int kOutPerPass = kDThreads / HD;  // 1 (HD=128) or 2 (HD=64)
    const int od = tid % HD;
    const int ogrp = tid / HD;
    float acc[kMaxGroup];
#pragma unroll
    for (int g = 0; g < kMaxGroup; ++g) acc[g] = 0.f;

    if (b0 < b1) load_block(b0, 0);
    __syncthreads();
    for (int b = b0; b < b1; ++b) {
        const int buf = (b - b0) & 1;
        if (b + 1 < b1) {
            load_block(b + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        // scores
        const int kpos = b * kBlockTokens + key;
        const __nv_bfloat16* krow = &sk[buf][key * C::kRow];
        float sc[kMaxGroup / 2];
#pragma unroll
        for (int i = 0; i < kMaxGroup / 2; ++i) sc[i] = 0.f;
#pragma unroll 4
        for (int d = 0; d < HD; d += 8) {
            const uint4 kv = *reinterpret_cast<const uint4*>(krow + d);
            const uint32_t w[4] = {kv.x, kv.y, kv.z, kv.w};
            float kf[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                kf[2 * e] = bf16_lo(w[e]);
                kf[2 * e + 1] = bf16_hi(w[e]);
            }
#pragma unroll
            for (int i = 0; i < kMaxGroup / 2; ++i) {
                const int g = hgrp + 2 * i;
                if (g < G) {
                    const float4 q0 = *reinterpret_cast<const float4*>(&sq[g][d]);
                    const float4 q1 = *reinterpret_cast<const float4*>(&sq[g][d + 4]);
                    sc[i] += q0.x * kf[0] + q0.y * kf[1] + q0.z * kf[2] + q0.w * kf[3] +
                             q1.x * kf[4] + q1.y * kf[5] + q1.z * kf[6] + q1.w * kf[7];
                }
            }
        }
#pragma unroll
        for (int i = 0; i < kMaxGroup / 2; ++i) {
            const int g = hgrp + 2 * i;
            if (g < G) sp[g][key] = kpos < it.ctx_len ? sc[i] : -FLT_MAX;
        }
        __syncthreads();
        // online softmax per head: warp w handles heads w, w+4
        {
            const int w = tid >> 5, l = tid & 31;
            for (int g = w; g < G; g += 4) {
                const float a = sp[g][l], c = sp[g][l + 32];
                float mx = fmaxf(a, c);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                const float m_old = s_m[g];
                const float m_new = fmaxf(m_old, mx);
                const float pa = (b * kBlockTokens + l < it.ctx_len) ? exp2f(a - m_new) : 0.f;
                const float pc = (b * kBlockTokens + l + 32 < it.ctx_len) ? exp2f(c - m_new) : 0.f;
                sp[g][l] = pa;
                sp[g][l + 32] = pc;
                float sum = pa + pc;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
                if (l == 0) {
                    const float alpha = exp2f(m_old - m_new);
                    s_alpha[g] = alpha;
                    s_l[g] = s_l[g] * alpha + sum;
                    s_m[g] = m_new;
                }
            }
        }
        __syncthreads();
        // P.V
        {
            const __nv_bfloat16* vcol = &sv[buf][od];
#pragma unroll
            for (int i = 0; i < kMaxGroup; ++i) {
                const int g = ogrp + kOutPerPass * i;
                if (g < G) acc[i] *= s_alpha[g];
            }
#pragma unroll 4
            for (int t = 0; t < kBlockTokens; t += 4) {
                const float v0 = __bfloat162float(vcol[(t + 0) * C::kRow]);
                const float v1 = __bfloat162float(vcol[(t + 1) * C::kRow]);
                const float v2 = __bfloat162float(vcol[(t + 2) * C::kRow]);
                const float v3 = __bfloat162float(vcol[(t + 3) * C::kRow]);
#pragma unroll
                for (int i = 0; i < kMaxGroup; ++i) {
                    const int g = ogrp + kOutPerPass * i;
                    if (g < G) {
                        const float4 p4 = *reinterpret_cast<const float4*>(&sp[g][t]);
                        acc[i] += p4.x * v0 + p4.y * v1 + p4.z * v2 + p4.w * v3;
                    }
                }
            }
        }
        __syncthreads();
    }
    // partials
    const size_t row_base = (static_cast<size_t>(blockIdx.x) * s.hq) * gridDim.z;
#pragma unroll
    for (int i = 0; i < kMaxGroup; ++i) {
        const int g = ogrp + kOutPerPass * i;
        if (g < G) {
            const int h = kvh * G + g;
            const size_t slot = row_base + static_cast<size_t>(h) * gridDim.z + split;
            part_o[slot * HD + od] = acc[i];
        }
    }
    if (tid < G) {
        const int h = kvh * G + tid;
        const size_t slot = row_base + static_cast<size_t>(h) * gridDim.z + split;
        part_ml[slot * 2 + 0] = s_m[tid];
        part_ml[slot * 2 + 1] = s_l[tid];
    }
}

// Merge split partials -> normalised bf16 output.  grid = (n_items, hq), block = HD.
template <int HD>
__global__ void decode_combine_kernel(const DecodeItem* __restrict__ items,
                                      const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml, int splits,
                                      __nv_bfloat16* __restrict__ out, int hq) {
    const int row = blockIdx.x, h = blockIdx.y, d = threadIdx.x;
    const size_t base = (static_cast<size_t>(row) * hq + h) * splits;
    float m = -FLT_MAX;
    for (int sp = 0; sp < splits; ++sp) m = fmaxf(m, part_ml[(base + sp) * 2]);
    float l = 0.f, o = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
        const float ms = part_ml[(base + sp) * 2];
        const float ls = part_ml[(base + sp) * 2 + 1];
        if (ls == 0.f) continue;
        const float w = exp2f(ms - m);
        l += ls * w;
        o += part_o[(base + sp) * HD + d] * w;
    }
    out[static_cast<size_t>(items[row].q_row) * hq * HD + h * HD + d] = __float2bfloat16_rn(o / l);
}

// Merge split-KV partials of prefill rows.  grid = (n_items, hkv, 128 rows), block = HD.
template <int HD>
__global__ void prefill_combine_kernel(const PrefillItem* __restrict__ items,
                                       const float* __restrict__ part_o,
                                       const float* __restrict__ part_ml, int splits,
                                       __nv_bfloat16* __restrict__ out, int hq, int hkv) {
    const PrefillItem it = items[blockIdx.x];
    const int G = hq / hkv;
    const int r = blockIdx.z, kvh = blockIdx.y, d = threadIdx.x;
    if (r >= it.n_q * G) return;
    const size_t base = (static_cast<size_t>(blockIdx.x) * hkv + kvh) * splits;
    float m = -FLT_MAX;
    for (int sp = 0; sp < splits; ++sp) m = fmaxf(m, part_ml[((base + sp) * 128 + r) * 2]);
    float l = 0.f, o = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
        const size_t row = (base + sp) * 128 + r;
        const float ls = part_ml[row * 2 + 1];
        if (ls == 0.f) continue;
        const float w = exp2f(part_ml[row * 2] - m);
        l += ls * w;
        o += part_o[row * HD + d] * w;
    }
    out[static_cast<size_t>(it.q_row0 + r / G) * hq * HD + (kvh * G + r % G) * HD + d] =
        __float2bfloat16_rn(o / l);
}

template <int HD>
cudaError_t prefill_launch(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                           const PrefillItem* items, int n_items, int max_blocks, int splits,
                           const int32_t* tables, __nv_bfloat16* out, float* part_o, float* part_ml,
                           const AttnShape& s, cudaStream_t stream) {
    using C = PCfg<HD>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(prefill_attention_kernel<HD>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int bps = (max_blocks + splits - 1) / splits;
    splits = (max_blocks + bps - 1) / bps;
    dim3 grid(n_items, s.hkv, splits);
    prefill_attention_kernel<HD><<<grid, kPThreads, C::kSmem, stream>>>(tq, tk, tv, items, tables,
                                                                       out, part_o, part_ml, bps, s);
    if (splits > 1)
        prefill_combine_kernel<HD><<<dim3(n_items, s.hkv, 128), HD, 0, stream>>>(
            items, part_o, part_ml, splits, out, s.hq, s.hkv);
    return cudaGetLastError();
}

}  // namespace

int prefill_tokens_per_tile(int hq, int hkv) { return 128 / (hq / hkv); }

int prefill_splits(int n_items, int hkv, int max_blocks, int num_sms, size_t ws_rows) {
    // split the KV range only when the (item, kv head) grid leaves SMs idle
    const int ctas = n_items * hkv;
    int splits = (2 * num_sms + ctas - 1) / ctas;
    splits = std::min(splits, std::max(1, max_blocks / 2));
    splits = std::min(splits, 32);
    while (splits > 1 && static_cast<size_t>(ctas) * splits * 128 > ws_rows) --splits;
    return std::max(splits, 1);
}

cudaError_t prefill_attention(const CUtensorMap& tmap_q, const CUtensorMap& tmap_k,
                              const CUtensorMap& tmap_v, const PrefillItem* items, int n_items,
                              int max_blocks, int splits, const int32_t* tables,
                              __nv_bfloat16* out, float* part_o, float* part_ml, const AttnShape& s,
                              cudaStream_t stream) {
    if (n_items <= 0) return cudaSuccess;
    if (s.hd == 128)
        return prefill_launch<128>(tmap_q, tmap_k, tmap_v, items, n_items, max_blocks, splits, tables,
                                   out, part_o, part_ml, s, stream);
    if (s.hd == 64)
        return prefill_launch<64>(tmap_q, tmap_k, tmap_v, items, n_items, max_blocks, splits, tables,
                                  out, part_o, part_ml, s, stream);
    return cudaErrorInvalidValue;
}

int decode_splits(int n_items, int hkv, int max_ctx, int num_sms, int max_splits) {
    const int blocks = (max_ctx + kBlockTokens - 1) / kBlockTokens;
    const int base = n_items * hkv;
    int splits = (3 * num_sms + base - 1) / (base > 0 ? base : 1);
    if (splits > blocks) splits = blocks;
    if (splits > max_splits) splits = max_splits;
    if (splits < 1) splits = 1;
    return splits;
}

cudaError_t decode_attention(const __nv_bfloat16* q, const __nv_bfloat16* k_pool,
                             const __nv_bfloat16* v_pool, const DecodeItem* items, int n_items,
                             int max_ctx, const int32_t* tables, __nv_bfloat16* out,
                             float* part_o, float* part_ml, int max_splits, int num_sms,
                             const AttnShape& s, cudaStream_t stream) {
    if (n_items <= 0) return cudaSuccess;
    if (s.hq / s.hkv > kMaxGroup) return cudaErrorInvalidValue;
    const int splits = decode_splits(n_items, s.hkv, max_ctx, num_sms, max_splits);
    const int blocks = (max_ctx + kBlockTokens - 1) / kBlockTokens;
    const int bps = (blocks + splits - 1) / splits;
    dim3 grid(n_items, s.hkv, splits);
    if (s.hd == 128) {
        if (cudaError_t e = decode_prepare<128>(); e != cudaSuccess) return e;
        decode_attention_kernel<128><<<grid, kDThreads, DCfg<128>::kSmem, stream>>>(q, k_pool, v_pool, items,
                                                                     tables, part_o, part_ml, bps, s);
        decode_combine_kernel<128><<<dim3(n_items, s.hq), 128, 0, stream>>>(items, part_o, part_ml,
                                                                          splits, out, s.hq);
    } else if (s.hd == 64) {
        if (cudaError_t e = decode_prepare<64>(); e != cudaSuccess) return e;
        decode_attention_kernel<64><<<grid, kDThreads, DCfg<64>::kSmem, stream>>>(q, k_pool, v_pool, items,
                                                                    tables, part_o, part_ml, bps, s);
        decode_combine_kernel<64><<<dim3(n_items, s.hq), 64, 0, stream>>>(items, part_o, part_ml,
                                                                        splits, out, s.hq);
    } else {
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace asb
