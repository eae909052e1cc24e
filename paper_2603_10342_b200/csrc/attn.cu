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
//   /root/reference/proj/src/executor.cpp:93-95.
// Decode attention (K2) lives in decode_attn.cu.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <vector>
#include <cfloat>

#include "attn.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace asb {

namespace {

// ============================================================================ prefill
// Two GQA-packed query tiles per CTA (256 MMA rows = 2 x (128/G tokens) x G heads of one KV
// head) share every K/V page.  Roles:
//   warp 0     TMA producer (Q once, K/V pages into a ring)
//   warps 1,10 MMA issuers, one per tile: S_t = Q_t.K^T into TMEM, then O_t += P_t.V with P_t
//              read straight from TMEM (the A-from-TMEM form of tcgen05.mma); S_t of page j+1
//              is issued before P_t.V of page j, so the tensor core runs while softmax works.
//              One issuer per tile decouples the tiles: a single in-order issuer made tile 0's
//              next S wait for tile 1's softmax (and vice versa) every page.
//   warps 2-5  softmax of tile 0, warps 6-9 softmax of tile 1: one query row per thread (its
//              TMEM lane), P written back over its own S columns as packed bf16.
// O accumulates in TMEM across pages.  The running max is refreshed lazily: O and l are
// rescaled (in TMEM, by the row's own thread) only when a row max grows by more than 2^8, so
// most pages never touch O outside the MMA.
constexpr int kPThreads = 352;
constexpr float kRescaleLog2 = 8.0f;

template <int HD>
struct PCfg {
    static constexpr int kHalves = HD / 64;
    static constexpr int kQTile = 128 * HD * 2;           // one 128-row Q tile
    static constexpr int kQBytes = 2 * kQTile;
    static constexpr int kKBytes = kBlockTokens * HD * 2;
    static constexpr int kStageBytes = 2 * kKBytes;       // K then V
    static constexpr int kStages = HD == 128 ? 4 : 6;
    static constexpr int kSmem = kQBytes + kStages * kStageBytes + 1024 + 256;
    // TMEM: S[t][b] (64 fp32 cols each, P aliased as bf16 pairs) at (2t+b)*64, O[t] at 256+t*HD
    static constexpr int kTmemCols = 512;
};

__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
        "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]),
        "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]),
        "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

template <int HD>
__global__ void __launch_bounds__(kPThreads, 1)
    prefill_attention_kernel(const __grid_constant__ CUtensorMap tmap_q,
                             const __grid_constant__ CUtensorMap tmap_k,
                             const __grid_constant__ CUtensorMap tmap_v,
                             const PrefillItem* __restrict__ items,
                             const int32_t* __restrict__ tables, __nv_bfloat16* __restrict__ out,
                             float* __restrict__ part_o, float* __restrict__ part_ml,
                             const int4* __restrict__ units, int blocks_per_split, const AttnShape s) {
    using C = PCfg<HD>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
    uint8_t* sq = smem;
    uint8_t* skv = sq + C::kQBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(skv + C::kStages * C::kStageBytes);
    uint64_t* q_full = bars + 0;
    uint64_t* kv_full = bars + 1;                 // [kStages]
    uint64_t* kv_empty = kv_full + C::kStages;    // [kStages]
    uint64_t* s_full = kv_empty + C::kStages;     // [2 tiles][2 bufs]
    uint64_t* p_full = s_full + 4;                // [2][2]
    uint64_t* pv_done = p_full + 4;               // [2][2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 4);

    // heaviest items (most causal pages) first: they define the tail.  Either a uniform split
    // (grid.z splits of blocks_per_split pages) or a work-unit list (item, first page, pages,
    // partial slot or -1): only the long causal items split, so the grid stays one wave.
    const int4 unit = units ? units[gridDim.x - 1 - blockIdx.x] : make_int4(0, 0, 0, 0);
    const int item_idx = units ? unit.x : static_cast<int>(gridDim.x - 1 - blockIdx.x);
    const PrefillItem it = items[item_idx];
    const int kvh = blockIdx.y;
    const int G = s.hq / s.hkv;
    const int tpt = 128 / G;          // tokens per tile
    const int box_rows = tpt * G;     // valid MMA rows of a full tile
    const int total_blocks = (it.q_pos0 + it.n_q + kBlockTokens - 1) / kBlockTokens;
    const int blk0 = units ? unit.y : static_cast<int>(blockIdx.z) * blocks_per_split;
    const int n_kv = max(0, min(total_blocks, blk0 + (units ? unit.z : blocks_per_split)) - blk0);
    const bool split = units ? unit.w >= 0 : gridDim.z > 1;
    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    const size_t pbase = units ? static_cast<size_t>(unit.w < 0 ? 0 : unit.w) * gridDim.y + kvh
                               : (static_cast<size_t>(item_idx) * gridDim.y + kvh) * gridDim.z + blockIdx.z;
    if (n_kv == 0) {
        // empty split: neutral partials (after the PDL wait: the previous layer's combine may
        // still be reading this partial slot)
        pdl_trigger();
        pdl_wait();
        for (int r = threadIdx.x; r < 256; r += blockDim.x) {
            part_ml[(pbase * 256 + r) * 2 + 0] = -FLT_MAX;
            part_ml[(pbase * 256 + r) * 2 + 1] = 0.f;
        }
        return;
    }

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_q);
        tma_prefetch_desc(&tmap_k);
        tma_prefetch_desc(&tmap_v);
        mbar_init(q_full, 1);
        for (int i = 0; i < C::kStages; ++i) {
            mbar_init(&kv_full[i], 1);
            mbar_init(&kv_empty[i], 2);  // released by both tiles' P.V
        }
        for (int i = 0; i < 4; ++i) {
            mbar_init(&s_full[i], 1);
            mbar_init(&p_full[i], 128);
            mbar_init(&pv_done[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<C::kTmemCols>(tmem_slot);
    // rows of a tile beyond box_rows (< G of them) are never loaded: zero them once
    for (int i = threadIdx.x; i < 2 * C::kHalves * (128 - box_rows) * 8; i += blockDim.x) {
        const int per_t = C::kHalves * (128 - box_rows) * 8;
        const int t = i / per_t, j = i % per_t;
        const int h = j / ((128 - box_rows) * 8), rem = j % ((128 - box_rows) * 8);
        reinterpret_cast<uint4*>(sq + t * C::kQTile + h * (128 * 128) + (box_rows + rem / 8) * 128)[rem % 8] =
            make_uint4(0, 0, 0, 0);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_trigger();
    pdl_wait();  // q / K / V were written by the kernels before us
    const uint32_t tmem = *tmem_slot;
    const int32_t* table = tables + it.table_off;

    if (warp == 0) {
        if (elect_one()) {
            mbar_expect_tx(q_full, 2 * C::kHalves * box_rows * 128);  // full boxes incl. OOB fill
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int h = 0; h < C::kHalves; ++h)
                    tma_load_3d(sq + t * C::kQTile + h * (128 * 128), &tmap_q, q_full, h * 64, kvh * G,
                                it.q_row0 + t * tpt);
            const uint64_t pol = policy_evict_last();  // pages are re-read by the other heads
            for (int j = 0; j < n_kv; ++j) {
                const int st = j % C::kStages;
                const int blk = table[blk0 + j];  // issued before the wait: off the refill path
                mbar_wait(&kv_empty[st], ((j / C::kStages) & 1) ^ 1);
                mbar_expect_tx(&kv_full[st], C::kStageBytes);
                const int row = ((s.layer * s.num_blocks + blk) * s.hkv + kvh) * kKvPageRows;
                uint8_t* kdst = skv + st * C::kStageBytes;
                uint8_t* vdst = kdst + C::kKBytes;
#pragma unroll
                for (int h = 0; h < C::kHalves; ++h) {
                    tma_load_2d_hint(kdst + h * (kBlockTokens * 128), &tmap_k, &kv_full[st], h * 64, row, pol);
                    tma_load_2d_hint(vdst + h * (kBlockTokens * 128), &tmap_v, &kv_full[st], h * 64, row, pol);
                }
            }
        }
        __syncwarp();
    } else if (warp == 1 || warp == 10) {
        constexpr uint32_t idesc_s = make_idesc_bf16(128, kBlockTokens, false, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(128, HD, false, true);
        mbar_wait(q_full, 0);
        auto issue_s = [&](int t, int j) {
            const int st = j % C::kStages, b = j & 1;
            if (j >= 2) mbar_wait(&pv_done[2 * t + b], ((j >> 1) - 1) & 1);  // P_t(j-2) consumed
            tc_fence_after();
            if (elect_one()) {
                const uint32_t q_addr = smem_u32(sq + t * C::kQTile);
                const uint32_t k_addr = smem_u32(skv + st * C::kStageBytes);
#pragma unroll
                for (int k = 0; k < HD / 16; ++k) {
                    const int h = k / 4, kk = k % 4;
                    const uint64_t ad = make_sw128_desc(q_addr + h * 16384 + kk * 32, 16, 1024);
                    const uint64_t bd = make_sw128_desc(k_addr + h * (kBlockTokens * 128) + kk * 32, 16, 1024);
                    umma_bf16(tmem + (2 * t + b) * 64, ad, bd, idesc_s, k > 0 ? 1u : 0u);
                }
                umma_commit(&s_full[2 * t + b]);
            }
            __syncwarp();
        };
        auto issue_pv = [&](int t, int j) {
            const int st = j % C::kStages, b = j & 1;
            mbar_wait(&p_full[2 * t + b], (j >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t v_addr = smem_u32(skv + st * C::kStageBytes + C::kKBytes);
#pragma unroll
                for (int k = 0; k < kBlockTokens / 16; ++k) {
                    // V is MN-major (head_dim contiguous): LBO = distance between 64-wide
                    // head_dim atoms, SBO = 8 key rows; 16 keys per MMA = 2048 bytes.
                    const uint64_t bd = make_sw128_desc(v_addr + k * 2048, kBlockTokens * 128, 1024);
                    umma_bf16_ts(tmem + 256 + t * HD, tmem + (2 * t + b) * 64 + 8 * k, bd, idesc_o,
                                 (j > 0 || k > 0) ? 1u : 0u);
                }
                umma_commit(&pv_done[2 * t + b]);
                umma_commit(&kv_empty[st]);
            }
            __syncwarp();
        };
        auto wait_kv = [&](int j) {
            mbar_wait(&kv_full[j % C::kStages], (j / C::kStages) & 1);
        };
        const int t = warp == 1 ? 0 : 1;
        wait_kv(0);
        issue_s(t, 0);
        for (int j = 0; j < n_kv; ++j) {
            if (j + 1 < n_kv) {
                wait_kv(j + 1);
                issue_s(t, j + 1);
            }
            issue_pv(t, j);
        }
    } else {
        // softmax: tile t, one query row per thread (TMEM lane quarter = warp % 4)
        const int t = (warp - 2) / 4;
        const uint32_t quarter = warp & 3;
        const int rr = quarter * 32 + lane;             // row within the tile
        const int tok = t * tpt + rr / G;               // token within the item
        const bool valid = rr < box_rows && tok < it.n_q;
        const int qpos = it.q_pos0 + tok;
        const uint32_t t_lane = tmem + ((quarter * 32u) << 16);
        const uint32_t o_col = t_lane + 256 + t * HD;
        float m_ref = -FLT_MAX, l_run = 0.f;
        for (int j = 0; j < n_kv; ++j) {
            const int b = j & 1;
            const uint32_t s_col = t_lane + (2 * t + b) * 64;
            mbar_wait(&s_full[2 * t + b], (j >> 1) & 1);
            tc_fence_after();
            uint32_t sa[32], sb2[32];
            tmem_ld32(s_col, sa);
            tmem_ld32(s_col + 32, sb2);
            tmem_ld_wait();
            const int kbase = (blk0 + j) * kBlockTokens;
            // pages left of the causal diagonal for every row of the warp take the unmasked
            // path (no per-element compare/select); the row max is a 3-input FMNMX tree
            const bool full_vis = kbase + kBlockTokens - 1 <= qpos;
            const bool warp_full = __all_sync(0xffffffffu, full_vis);
            if (!warp_full) {
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    if (kbase + c > qpos) sa[c] = __float_as_uint(-FLT_MAX);
                    if (kbase + 32 + c > qpos) sb2[c] = __float_as_uint(-FLT_MAX);
                }
            }
            float mx;
            {
                float m3[22];
#pragma unroll
                for (int c = 0; c < 21; ++c) {
                    const int a = 3 * c;
                    m3[c] = fmax3f(__uint_as_float(a < 32 ? sa[a] : sb2[a - 32]),
                                   __uint_as_float(a + 1 < 32 ? sa[a + 1] : sb2[a + 1 - 32]),
                                   __uint_as_float(a + 2 < 32 ? sa[a + 2] : sb2[a + 2 - 32]));
                }
                m3[21] = __uint_as_float(sb2[31]);
                float m1[8];
#pragma unroll
                for (int c = 0; c < 7; ++c) m1[c] = fmax3f(m3[3 * c], m3[3 * c + 1], m3[3 * c + 2]);
                m1[7] = m3[21];
                mx = fmax3f(fmax3f(m1[0], m1[1], m1[2]), fmax3f(m1[3], m1[4], m1[5]), fmaxf(m1[6], m1[7]));
            }
            mx = mx == -FLT_MAX ? -FLT_MAX : mx * s.scale_log2;
            const bool need = mx > m_ref + kRescaleLog2;
            if (__any_sync(0xffffffffu, need)) {
                const float alpha = need ? exp2f(m_ref - mx) : 1.f;
                if (j > 0) {
                    // O_t holds P.V of pages < j: wait for the last of them, rescale in place
                    mbar_wait(&pv_done[2 * t + ((j - 1) & 1)], ((j - 1) >> 1) & 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int c = 0; c < HD; c += 32) {
                        uint32_t ov[32];
                        tmem_ld32(o_col + c, ov);
                        tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * alpha);
                        tmem_st32(o_col + c, ov);
                    }
                    tmem_st_wait();
                }
                if (need) {
                    l_run *= alpha;
                    m_ref = mx;
                }
            }
            // no visible key yet (m_ref still -FLT_MAX): the masked -FLT_MAX scores must map to 0
            const float nm = m_ref == -FLT_MAX ? 0.f : -m_ref;
            // key pairs on the packed fp32x2 pipe (FFMA2 / FADD2); masked keys hold -FLT_MAX:
            // the FMA gives a huge negative input and ex2 flushes it to 0
            const unsigned long long sc2 = f2_pack(s.scale_log2, s.scale_log2), nm2 = f2_pack(nm, nm);
            unsigned long long acc2 = f2_pack(0.f, 0.f);
            uint32_t pk[32];
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const float x0 = __uint_as_float(c < 16 ? sa[2 * c] : sb2[2 * c - 32]);
                const float x1 = __uint_as_float(c < 16 ? sa[2 * c + 1] : sb2[2 * c + 1 - 32]);
                float y0, y1;
                f2_unpack(ffma2(f2_pack(x0, x1), sc2, nm2), y0, y1);
                // (a quarter of the pairs through a degree-3 2^f on the FMA pipe instead of
                // MUFU.EX2, FA4-style, measured slower: 943 -> 907 TF/s at C4 -- the softmax is
                // bound by its per-warp dependency chain, not the XU pipe)
                const float p0 = ex2_ftz(y0), p1 = ex2_ftz(y1);
                acc2 = fadd2(acc2, f2_pack(p0, p1));
                pk[c] = pack_bf16(p0, p1);
            }
            float ps0, ps1;
            f2_unpack(acc2, ps0, ps1);
            l_run += ps0 + ps1;
            tmem_st32(s_col, pk);  // P over its own S columns (A operand of P.V)
            tmem_st_wait();
            tc_fence_before();
            mbar_arrive(&p_full[2 * t + b]);
        }
        mbar_wait(&pv_done[2 * t + ((n_kv - 1) & 1)], ((n_kv - 1) >> 1) & 1);
        tc_fence_after();
        const int prow = t * 128 + rr;
        if (split) {
            const size_t base = pbase * 256 + prow;
            float4* po = reinterpret_cast<float4*>(part_o + base * HD);
#pragma unroll 1
            for (int c = 0; c < HD; c += 32) {
                uint32_t ov[32];
                tmem_ld32(o_col + c, ov);
                tmem_ld_wait();
                if (valid) {
#pragma unroll
                    for (int e = 0; e < 8; ++e)
                        po[c / 4 + e] = make_float4(__uint_as_float(ov[4 * e]), __uint_as_float(ov[4 * e + 1]),
                                                    __uint_as_float(ov[4 * e + 2]), __uint_as_float(ov[4 * e + 3]));
                }
            }
            if (valid) {
                part_ml[base * 2 + 0] = m_ref;
                part_ml[base * 2 + 1] = l_run;
            }
        } else {
            const float inv = 1.f / l_run;
            uint4* dst = reinterpret_cast<uint4*>(
                out + static_cast<size_t>(it.q_row0 + tok) * (s.hq * HD) + (kvh * G + rr % G) * HD);
#pragma unroll 1
            for (int c = 0; c < HD; c += 32) {
                uint32_t ov[32];
                tmem_ld32(o_col + c, ov);
                tmem_ld_wait();
                if (valid) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        uint4 v;
                        v.x = pack_bf16(__uint_as_float(ov[8 * e + 0]) * inv, __uint_as_float(ov[8 * e + 1]) * inv);
                        v.y = pack_bf16(__uint_as_float(ov[8 * e + 2]) * inv, __uint_as_float(ov[8 * e + 3]) * inv);
                        v.z = pack_bf16(__uint_as_float(ov[8 * e + 4]) * inv, __uint_as_float(ov[8 * e + 5]) * inv);
                        v.w = pack_bf16(__uint_as_float(ov[8 * e + 6]) * inv, __uint_as_float(ov[8 * e + 7]) * inv);
                        dst[c / 8 + e] = v;
                    }
                }
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

// Merge split-KV partials of prefill rows.  grid = (n_items, hkv, 256 rows), block = HD.
template <int HD>
__global__ void prefill_combine_kernel(const PrefillItem* __restrict__ items,
                                       const float* __restrict__ part_o,
                                       const float* __restrict__ part_ml, int splits,
                                       __nv_bfloat16* __restrict__ out, int hq, int hkv) {
    pdl_trigger();
    pdl_wait();
    const int item_idx = gridDim.x - 1 - blockIdx.x;  // same item order as the attention grid
    const PrefillItem it = items[item_idx];
    const int G = hq / hkv;
    const int tpt = 128 / G;
    const int prow = blockIdx.z, kvh = blockIdx.y, d = threadIdx.x;
    const int t = prow / 128, rr = prow % 128;
    const int tok = t * tpt + rr / G;
    if (rr >= tpt * G || tok >= it.n_q) return;
    const size_t base = (static_cast<size_t>(item_idx) * hkv + kvh) * splits;
    float m = -FLT_MAX;
    for (int sp = 0; sp < splits; ++sp) m = fmaxf(m, part_ml[((base + sp) * 256 + prow) * 2]);
    float l = 0.f, o = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
        const size_t row = (base + sp) * 256 + prow;
        const float ls = part_ml[row * 2 + 1];
        if (ls == 0.f) continue;
        const float w = exp2f(part_ml[row * 2] - m);
        l += ls * w;
        o += part_o[row * HD + d] * w;
    }
    out[static_cast<size_t>(it.q_row0 + tok) * hq * HD + (kvh * G + rr % G) * HD + d] =
        __float2bfloat16_rn(o / l);
}

// Merge the partials of the items the unit list split.  grid = (n_split_items, hkv, 256 / 8),
// block = (HD, 8 rows); comb[i] = (item, first partial slot, slots).
template <int HD>
__global__ void prefill_combine_units_kernel(const PrefillItem* __restrict__ items, const int4* __restrict__ comb,
                                             const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                             __nv_bfloat16* __restrict__ out, int hq, int hkv) {
    pdl_trigger();
    pdl_wait();
    const int4 c = comb[blockIdx.x];
    const PrefillItem it = items[c.x];
    const int G = hq / hkv;
    const int tpt = 128 / G;
    const int prow = blockIdx.z * 8 + threadIdx.y, kvh = blockIdx.y, d = threadIdx.x;
    const int t = prow / 128, rr = prow % 128;
    const int tok = t * tpt + rr / G;
    if (rr >= tpt * G || tok >= it.n_q) return;
    float m = -FLT_MAX;
    for (int q = 0; q < c.z; ++q) m = fmaxf(m, part_ml[((static_cast<size_t>(c.y + q) * hkv + kvh) * 256 + prow) * 2]);
    float l = 0.f, o = 0.f;
    for (int q = 0; q < c.z; ++q) {
        const size_t row = (static_cast<size_t>(c.y + q) * hkv + kvh) * 256 + prow;
        const float ls = part_ml[row * 2 + 1];
        if (ls == 0.f) continue;
        const float w = exp2f(part_ml[row * 2] - m);
        l += ls * w;
        o += part_o[row * HD + d] * w;
    }
    out[static_cast<size_t>(it.q_row0 + tok) * hq * HD + (kvh * G + rr % G) * HD + d] = __float2bfloat16_rn(o / l);
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
                             items, tables, out, part_o, part_ml, static_cast<const int4*>(nullptr), bps, s);
    if (e == cudaSuccess && splits > 1)
        e = launch_k(prefill_combine_kernel<HD>, dim3(n_items, s.hkv, 256), dim3(HD), 0, stream, items,
                     static_cast<const float*>(part_o), static_cast<const float*>(part_ml), splits, out, s.hq,
                     s.hkv);
    return e;
}

}  // namespace

int prefill_tokens_per_tile(int hq, int hkv) { return 128 / (hq / hkv); }
int prefill_tokens_per_cta(int hq, int hkv) { return 2 * prefill_tokens_per_tile(hq, hkv); }

int prefill_splits(int n_items, int hkv, int max_blocks, int num_sms, size_t ws_rows) {
    // split the KV range only when the (item, kv head) grid leaves SMs idle, up to one wave:
    // a second wave of split CTAs plus the combine costs more than the longest causal row
    // saves (C2 cold prefill, 114 CTAs on 148 SMs: 140 TF/s unsplit vs 107 with 2 splits)
    const int ctas = n_items * hkv;
    int splits = num_sms / ctas;
    splits = std::min(splits, std::max(1, max_blocks / 2));
    splits = std::min(splits, 32);
    while (splits > 1 && static_cast<size_t>(ctas) * splits * 256 > ws_rows) --splits;
    return std::max(splits, 1);
}

int prefill_units(const PrefillItem* items, int n_items, int hkv, int num_sms, size_t ws_rows,
                  std::vector<int4>& units, std::vector<int4>& comb) {
    // One wave of CTAs (one per SM), the smallest per-CTA page budget B that fits: items with
    // more than B causal pages split into balanced ranges, the rest run whole.  The tail of a
    // causal batch is its longest item, so this shortens the critical path from max_i b_i to
    // ~B pages where the uniform split could not (it splits every item or none).
    units.clear();
    comb.clear();
    if (n_items <= 0 || n_items * hkv > num_sms) return 0;
    std::vector<int> b(n_items);
    int maxb = 0;
    for (int i = 0; i < n_items; ++i) {
        b[i] = (items[i].q_pos0 + items[i].n_q + kBlockTokens - 1) / kBlockTokens;
        maxb = std::max(maxb, b[i]);
    }
    auto ctas = [&](int B) {
        long long c = 0;
        for (int i = 0; i < n_items; ++i) c += (b[i] + B - 1) / B;
        return c * hkv;
    };
    int B = maxb;
    while (B > 2 && ctas(B - 1) <= num_sms) --B;
    if (B >= maxb) return 0;
    int parts = 0;
    for (int i = 0; i < n_items; ++i) {
        const int n = (b[i] + B - 1) / B;
        const int per = (b[i] + n - 1) / n;
        if (n > 1) comb.push_back(make_int4(i, parts, n, 0));
        for (int z = 0; z < n; ++z)
            units.push_back(make_int4(i, z * per, std::min(per, b[i] - z * per), n > 1 ? parts + z : -1));
        if (n > 1) parts += n;
    }
    if (static_cast<size_t>(parts) * hkv * 256 > ws_rows) {
        units.clear();
        comb.clear();
        return 0;
    }
    return static_cast<int>(units.size());
}

cudaError_t prefill_attention_units(const CUtensorMap& tmap_q, const CUtensorMap& tmap_k,
                                    const CUtensorMap& tmap_v, const PrefillItem* items, const int4* units,
                                    int n_units, const int4* comb, int n_comb, const int32_t* tables,
                                    __nv_bfloat16* out, float* part_o, float* part_ml, const AttnShape& s,
                                    cudaStream_t stream) {
    if (n_units <= 0) return cudaSuccess;
    auto run = [&](auto hd_tag) -> cudaError_t {
        constexpr int HD = decltype(hd_tag)::value;
        using C = PCfg<HD>;
        static bool attr = false;
        if (!attr) {
            cudaError_t e = cudaFuncSetAttribute(prefill_attention_kernel<HD>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
            if (e != cudaSuccess) return e;
            attr = true;
        }
        cudaError_t e = launch_k(prefill_attention_kernel<HD>, dim3(n_units, s.hkv, 1), dim3(kPThreads), C::kSmem,
                                 stream, tmap_q, tmap_k, tmap_v, items, tables, out, part_o, part_ml, units, 0, s);
        if (e == cudaSuccess && n_comb > 0)
            e = launch_k(prefill_combine_units_kernel<HD>, dim3(n_comb, s.hkv, 256 / 8), dim3(HD, 8), 0, stream, items, comb,
                         static_cast<const float*>(part_o), static_cast<const float*>(part_ml), out, s.hq, s.hkv);
        return e;
    };
    if (s.hd == 128) return run(std::integral_constant<int, 128>{});
    if (s.hd == 64) return run(std::integral_constant<int, 64>{});
    return cudaErrorInvalidValue;
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
