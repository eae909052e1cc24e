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
// Decode attention (K2) lives in decode_attn.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>

#include "attn.h"
#include "launch.cuh"
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
    pdl_trigger();
    pdl_wait();  // q / K / V were written by the kernels before us
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
        __syncwarp();  // reconverge before the CTA barrier
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

// Merge split-KV partials of prefill rows.  grid = (n_items, hkv, 128 rows), block = HD.
template <int HD>
__global__ void prefill_combine_kernel(const PrefillItem* __restrict__ items,
                                       const float* __restrict__ part_o,
                                       const float* __restrict__ part_ml, int splits,
                                       __nv_bfloat16* __restrict__ out, int hq, int hkv) {
    pdl_trigger();
    pdl_wait();
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
    cudaError_t e = launch_k(prefill_attention_kernel<HD>, grid, dim3(kPThreads), C::kSmem, stream, tq, tk, tv,
                             items, tables, out, part_o, part_ml, bps, s);
    if (e == cudaSuccess && splits > 1)
        e = launch_k(prefill_combine_kernel<HD>, dim3(n_items, s.hkv, 128), dim3(HD), 0, stream, items,
                     static_cast<const float*>(part_o), static_cast<const float*>(part_ml), splits, out, s.hq,
                     s.hkv);
    return e;
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

}  // namespace asb
