// Paged decode attention (K2 in SURVEY §2.3) — one query token per decode row, the G query
// heads of one KV head per CTA.  HBM-bound: each context token's K and V row is streamed
// from HBM exactly once per (row, KV head).  Replaces the mu_D term of the reference's
// decode_step_duration_ms (/root/reference/proj/src/executor.cpp:90-92).
//
// CTA = 1 producer warp + 4 consumer warps, two CTAs per SM, split-KV over gridDim.z:
//   producer  : ONE TMA request per 64-token KV block: the block's K page and V page are
//               adjacent in the pool (attn.h), so a 5-D box (col, row, half, K|V, page) moves
//               both as a single 32 KiB (hd 128) / 16 KiB (hd 64) SWIZZLE_128B copy into a
//               3-stage (hd 128) / 6-stage ring, evict-first.  The per-SM TMA issue rate caps
//               small requests (~7.5 M requests/s per SM: 4 KiB boxes -> ~60 GB/s/SM, 32 KiB
//               -> ~175 GB/s/SM, profiles/r2_partition_probe.txt), which is what bounds decode
//               on a 16-64 SM Green Context partition, where HBM itself is not the limit.
//   consumers : all four warps share each stage, 16 keys each.  Keys are the M rows of a
//               warp-level bf16 MMA (m16n8k16) and the G <= 8 heads its N columns, so no MMA
//               row is padding:
//                 S^T = K . Q^T          (A = K by ldmatrix, B = Q^T held in registers)
//                 online softmax per head column (3 shuffles per head pair for the max; the
//                 running sum stays per-thread until the end)
//                 O^T += V^T . P^T       (A = V^T by ldmatrix.trans, B = P^T by movmatrix.trans
//                                        of the S^T fragments)
//               16 MMAs and 16 ldmatrix per warp per 64-token block.  (tcgen05 needs M >= 64
//               and a TMEM round trip per block; a register-resident warp MMA is the better fit
//               for this memory-bound shape.)
//   epilogue  : warps merge (m, l, O) through smem; the CTA writes bf16 output (one split),
//               or the splits of a (row, kv head) merge over DSMEM in a cluster / through fp32
//               partials.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "attn.h"
#include "launch.cuh"
#include "sm100.cuh"
#include "warpmma.cuh"

namespace asb {

namespace {

constexpr int kWarps = 4;  // consumer warps per CTA, 16 keys of each 64-token block apiece
constexpr int kThreadsD = (kWarps + 1) * 32;

template <int HD>
struct DC {
    static constexpr int kStage = 2 * kBlockTokens * HD * 2;   // K page + V page of one block
    // 96 KiB of K/V in flight per CTA, two CTAs per SM (192 KiB per SM)
    static constexpr int kStages = HD == 128 ? 3 : 6;
    static constexpr int kRing = kStages * kStage;
};

// transpose an 8x8 bf16 matrix held one row-pair per thread (the mma / ldmatrix fragment)
__device__ __forceinline__ uint32_t movmatrix_t(uint32_t x) {
    uint32_t y;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

// byte offset of 16-byte chunk c (0..HD/8-1) of row r (0..63) of the K (kv = 0) or V (kv = 1)
// page in a stage: the box lands as [K|V][half][64 rows][128 B] and SWIZZLE_128B XORs the
// chunk with the 128-byte line index mod 8 (= r mod 8)
template <int HD>
__device__ __forceinline__ uint32_t kv_off(int kv, int r, int c) {
    constexpr int H = HD / 64;
    const int line = ((kv * H + (c >> 3)) * kBlockTokens) + r;
    return line * 128 + (((c & 7) ^ (r & 7)) << 4);
}

// Column c (0..7) of an item's MMA N tile: token j = (col0 + c) / G of its group, query head
// (col0 + c) % G of the KV head's G, q / out row q_row + j, keys 0 .. ctx_len + j - 1 (lim 0:
// a padding column, everything masked)
struct DCol {
    int row, head, lim;
};
__device__ __forceinline__ DCol dcol(const DecodeItem& it, int c, int G) {
    const int cc = it.col0 + c;
    const int j = cc / G;
    DCol d;
    d.row = it.q_row + j;
    d.head = cc - j * G;
    d.lim = cc < it.ncols ? it.ctx_len + j : 0;
    return d;
}
// keys of the item's last column: the block range it streams
__device__ __forceinline__ int item_keys(const DecodeItem& it, int G) {
    return it.ctx_len + min(it.col0 + 7, it.ncols - 1) / G;
}
__device__ __forceinline__ int item_cols(const DecodeItem& it) { return min(8, it.ncols - it.col0); }

// One 64-token K|V block of the online softmax for this warp's 16 keys (kw..kw+15 of the
// block, absolute key index kbase + ..): S^T = K Q^T, running max / sum per head column,
// O^T = alpha O^T + V^T P^T.
template <int HD>
__device__ __forceinline__ void attn_page(uint32_t base, int kw, int kbase, const int (&lim)[2], const uint32_t (&qb)[HD / 16][2],
                                          float (&o)[HD / 16][4], float (&m_run)[2], float (&l_run)[2],
                                          float scale_log2, int lane) {
    constexpr int MT = HD / 16;
    const int g = lane >> 2, mi = lane >> 3;
    // ---- S^T = K . Q^T : 16 keys x 8 heads, two accumulation chains over the dims
    float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
    {
        const int key = kw + (mi & 1) * 8 + (lane & 7);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4(base + kv_off<HD>(0, key, 2 * kk + (mi >> 1)), a0, a1, a2, a3);
            if (kk & 1) mma16816(sb, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
            else mma16816(sa, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
        }
    }
    // ---- online softmax per column: values (key g | g+8, column 2t + j), causal per column
    float sv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const bool ok = kbase + g + (e < 2 ? 0 : 8) < lim[e & 1];
        sv[e] = ok ? (sa[e] + sb[e]) * scale_log2 : -FLT_MAX;
    }
    float alpha[2], mx[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        float m = fmax3f(m_run[j], sv[j], sv[2 + j]);
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 4));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 8));
        m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 16));
        mx[j] = m;
        alpha[j] = ex2_ftz(m_run[j] - m);
        m_run[j] = m;
    }
    float p[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) p[e] = sv[e] == -FLT_MAX ? 0.f : ex2_ftz(sv[e] - mx[e & 1]);
    const uint32_t p01 = pack_bf16(p[0], p[1]), p23 = pack_bf16(p[2], p[3]);
    // sum what P.V will actually use (the bf16-rounded weights)
    l_run[0] = l_run[0] * alpha[0] + (bf16_lo(p01) + bf16_lo(p23));
    l_run[1] = l_run[1] * alpha[1] + (bf16_hi(p01) + bf16_hi(p23));
    // P^T B-fragments: (keys 2t, 2t+1 | 2t+8, 2t+9; head g)
    const uint32_t b0 = movmatrix_t(p01), b1 = movmatrix_t(p23);
    const unsigned long long al2 = f2_pack(alpha[0], alpha[1]);
    // ---- O^T = alpha O^T + V^T . P^T : MT m-tiles of 16 dims
    {
        const int key = kw + (mi >> 1) * 8 + (lane & 7);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            uint32_t a0, a1, a2, a3;
            ldsm_x4_t(base + kv_off<HD>(1, key, 2 * mt + (mi & 1)), a0, a1, a2, a3);
            // (dim g | g+8, heads 2t, 2t+1) pairs scale by (alpha0, alpha1) on the fp32x2 pipe
            f2_unpack(fmul2(f2_pack(o[mt][0], o[mt][1]), al2), o[mt][0], o[mt][1]);
            f2_unpack(fmul2(f2_pack(o[mt][2], o[mt][3]), al2), o[mt][2], o[mt][3]);
            mma16816(o[mt], a0, a1, a2, a3, b0, b1);
        }
    }
}

template <int HD>
__global__ void __launch_bounds__(kThreadsD, 2)
    decode_attn_kernel(const __grid_constant__ CUtensorMap tmap_kv,
                       const __nv_bfloat16* __restrict__ q, const DecodeItem* __restrict__ items,
                       const int32_t* __restrict__ tables, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ part_o, float* __restrict__ part_ml,
                       int* __restrict__ counters, int pages_per_split, int cluster_merge,
                       AttnShape s) {
    using C = DC<HD>;
    constexpr int MT = HD / 16;  // O^T m-tiles (16 dims each)
    constexpr int kStagesR = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
    uint8_t* ring = smem;
    // after the ring drains: per-warp O^T [warp][8 heads][HD] at its start (merge), the
    // cluster-merge record behind it
    float* mrg = reinterpret_cast<float*>(ring);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kRing);
    uint64_t* empty = full + kStagesR;
    float* mls = reinterpret_cast<float*>(empty + kStagesR);  // [warp][8][2]

    const int cta_id = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    auto stamp = [&](int k) {
        if (s.dbg && cta_id < 1024) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            s.dbg[cta_id * 8 + k] = t;
        }
    };
    if (threadIdx.x == 0) stamp(0);
    const DecodeItem it = items[blockIdx.x];
    const int kvh = blockIdx.y;
    const int G = s.hq / s.hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NC = item_cols(it);  // live columns of this item
    const int n_pages = (item_keys(it, G) + kBlockTokens - 1) / kBlockTokens;
    const int p0 = blockIdx.z * pages_per_split;
    const int n_local = max(0, min(n_pages, p0 + pages_per_split) - p0);
    const int32_t* table = tables + it.table_off;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_kv);
        for (int i = 0; i < kStagesR; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();
    pdl_trigger();

    if (warp == kWarps) {
        // ------------------------------------------------------------ producer
        // K/V of positions before this step's token were written by earlier steps: stream them
        // while the kernel before us (the QKV projection appending the new token) is still
        // running, and wait for it only before the block that holds the new token.
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const int new_page = s.no_prewait ? 0 : it.pad / kBlockTokens;  // first block this step writes
            bool waited = false;
            for (int i = 0; i < n_local; ++i) {
                if (!waited && p0 + i >= new_page) {
                    pdl_wait();
                    // the QKV kernel wrote this step's K/V with generic stores; the blocks are read
                    // by TMA (async proxy)
                    fence_proxy_async_global();
                    waited = true;
                }
                const int st = i % kStagesR;
                mbar_wait(&empty[st], ((i / kStagesR) & 1) ^ 1);
                mbar_expect_tx(&full[st], C::kStage);
                const int page = (s.layer * s.num_blocks + table[p0 + i]) * s.hkv + kvh;
                tma_load_5d_hint(ring + st * C::kStage, &tmap_kv, &full[st], 0, 0, 0, 0, page, pol);
            }
            if (!waited) pdl_wait();
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    pdl_wait();  // q comes from the kernel before us
    if (threadIdx.x == 0) stamp(1);
    const int g = lane >> 2, t = lane & 3;  // fragment row / column-pair owner
    const int kw = warp * 16;               // this warp's keys within each block
    // Q^T B-fragments (k = dims, n = heads): head g, dims (2t, 2t+1) and (2t+8, 2t+9) of each
    // 16-dim k-step; heads >= G are zero columns
    uint32_t qb[HD / 16][2];
    {
        const DCol qc = dcol(it, g, G);
        const __nv_bfloat16* qrow = q + (size_t)qc.row * s.hq * HD + (size_t)(kvh * G + qc.head) * HD;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
            if (qc.lim > 0) {
                qb[kk][0] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t);
                qb[kk][1] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t + 8);
            } else {
                qb[kk][0] = qb[kk][1] = 0u;
            }
        }
    }
    const int lim[2] = {dcol(it, 2 * t, G).lim, dcol(it, 2 * t + 1, G).lim};  // this thread's columns
    // O^T accumulators: m-tile mt holds (dim mt*16+g, heads 2t, 2t+1) and (dim +8, same heads)
    float o[MT][4];
#pragma unroll
    for (int n = 0; n < MT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_run[2] = {-FLT_MAX, -FLT_MAX}, l_run[2] = {0.f, 0.f};  // heads 2t, 2t+1
    const int mi = lane >> 3;

    for (int i = 0; i < n_local; ++i) {
        const int st = i % kStagesR;
        mbar_wait(&full[st], (i / kStagesR) & 1);
        if (i == 0 && threadIdx.x == 0) stamp(2);
        if (s.dbg_load_only) {  // timing ablation (ASB_DEBUG_SKIP=attnmath): the load stream alone
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            continue;
        }
        attn_page<HD>(smem_u32(ring + st * C::kStage), kw, (p0 + i) * kBlockTokens + kw, lim, qb, o, m_run,
                      l_run, s.scale_log2, lane);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }
    // per-thread partial sums -> the head's sum over this warp's keys
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        l_run[j] += __shfl_xor_sync(0xffffffffu, l_run[j], 4);
        l_run[j] += __shfl_xor_sync(0xffffffffu, l_run[j], 8);
        l_run[j] += __shfl_xor_sync(0xffffffffu, l_run[j], 16);
    }

    // ---------------------------------------------------------------- merge warps
    if (threadIdx.x == 0) stamp(3);
    named_sync(1, kWarps * 32);  // every warp is done with the ring: it becomes merge space
    float* mw = mrg + warp * 8 * HD;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const int h = 2 * t + j;  // column
        if (h < NC) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                mw[h * HD + mt * 16 + g] = o[mt][j];
                mw[h * HD + mt * 16 + g + 8] = o[mt][2 + j];
            }
            if (g == 0) {
                mls[(warp * 8 + h) * 2] = m_run[j];
                mls[(warp * 8 + h) * 2 + 1] = l_run[j];
            }
        }
    }
    named_sync(1, kWarps * 32);
    const bool single = gridDim.z == 1;
    const bool cmerge = !single && cluster_merge;
    // cluster merge: this CTA's (M, L, O) parked at the start of the drained ring
    float* cO = mrg + kWarps * 8 * HD;           // [column][HD], behind the warp records
    float* cM = cO + 8 * HD;                     // [column]
    float* cL = cM + 8;                          // [column]
    for (int e = threadIdx.x; e < NC * HD; e += kWarps * 32) {
        const int h = e / HD, d = e % HD;
        float M = -FLT_MAX;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, mls[(w * 8 + h) * 2]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const float lw = mls[(w * 8 + h) * 2 + 1];
            if (lw == 0.f) continue;
            const float f = exp2f(mls[(w * 8 + h) * 2] - M);
            L += lw * f;
            O += mrg[(w * 8 + h) * HD + d] * f;
        }
        if (single) {
            const DCol oc = dcol(it, h, G);
            out[(size_t)oc.row * s.hq * HD + (kvh * G + oc.head) * HD + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
        } else if (cmerge) {
            cO[h * HD + d] = O;
            if (d == 0) {
                cM[h] = M;
                cL[h] = L;
            }
        } else {
            const size_t slot = (((size_t)blockIdx.x * s.hkv + kvh) * 8 + h) * gridDim.z + blockIdx.z;
            part_o[slot * HD + d] = O;
            if (d == 0) {
                part_ml[slot * 2 + 0] = M;
                part_ml[slot * 2 + 1] = L;
            }
        }
    }
    if (single) {
        if (threadIdx.x == 0) stamp(5);
        return;
    }
    if (cmerge) {
        // ---------------------------------------------------------- cluster split merge
        // The S splits of this (row, kv head) are the S CTAs of one thread-block cluster: after
        // a cluster barrier, CTA rank r merges slice r of the G x HD outputs straight from its
        // peers' shared memory (DSMEM), in split order -- the arithmetic of
        // decode_combine_kernel, with no global partials, fences or atomics.
        cluster_sync();
        if (threadIdx.x == 0) stamp(4);
        const int S = gridDim.z, r = blockIdx.z;
        const int n = NC * HD, lo = (n * r) / S, hi = (n * (r + 1)) / S;
        const uint32_t bO = smem_u32(cO), bM = smem_u32(cM), bL = smem_u32(cL);
        for (int e = lo + threadIdx.x; e < hi; e += kWarps * 32) {
            const int h = e / HD, d = e % HD;
            float mq[8], lq[8], oq[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q < S) {
                    mq[q] = ld_dsmem_f32(mapa_shared(bM + 4 * h, q));
                    lq[q] = ld_dsmem_f32(mapa_shared(bL + 4 * h, q));
                    oq[q] = ld_dsmem_f32(mapa_shared(bO + 4 * e, q));
                }
            }
            float M = -FLT_MAX;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < S) M = fmaxf(M, mq[q]);
            float L = 0.f, O = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (q >= S || lq[q] == 0.f) continue;
                const float w = exp2f(mq[q] - M);
                L += lq[q] * w;
                O += oq[q] * w;
            }
            const DCol oc = dcol(it, h, G);
            out[(size_t)oc.row * s.hq * HD + (kvh * G + oc.head) * HD + d] = __float2bfloat16_rn(O / L);
        }
        cluster_sync();  // peers may still be reading this CTA's partial
        if (threadIdx.x == 0) stamp(5);
        return;
    }
    // ---------------------------------------------------------------- split merge
    // Last-arriving split of this (row, kv head) merges all splits in split order (the same
    // arithmetic as decode_combine_kernel: deterministic), then re-arms the counter.
    __shared__ int last_s;
    __threadfence();
    named_sync(1, kWarps * 32);
    if (threadIdx.x == 0) {
        int* cnt = counters + blockIdx.x * gridDim.y + kvh;
        const int prev = atomicAdd(cnt, 1);
        last_s = prev == static_cast<int>(gridDim.z) - 1;
        if (last_s) *cnt = 0;
    }
    named_sync(1, kWarps * 32);
    if (threadIdx.x == 0) stamp(4);
    if (!last_s) return;
    __threadfence();
    // per (head, split) weight exp2(m - M) and the normaliser L, once per head, in smem (the
    // ring is drained); then one pass over part_o with every split's load in flight
    const int splits = gridDim.z;
    float* wsp = reinterpret_cast<float*>(smem);  // [column][splits]
    float* linv = wsp + 8 * splits;               // [column]
    float* lsp = linv + 8;  // [column][splits] l
    const size_t slot0 = ((size_t)blockIdx.x * s.hkv + kvh) * 8;  // column h: (slot0 + h) * splits + split
    for (int i = threadIdx.x; i < NC * splits; i += kWarps * 32) {  // all (m, l) loads at once
        const int h = i / splits, sp = i % splits;
        const size_t sl = (slot0 + h) * splits + sp;
        wsp[i] = __ldcg(part_ml + sl * 2);
        lsp[i] = __ldcg(part_ml + sl * 2 + 1);
    }
    named_sync(1, kWarps * 32);
    if (threadIdx.x < NC) {
        float M = -FLT_MAX;
        for (int sp = 0; sp < splits; ++sp) M = fmaxf(M, wsp[threadIdx.x * splits + sp]);
        float L = 0.f;
        for (int sp = 0; sp < splits; ++sp) {
            const float ls = lsp[threadIdx.x * splits + sp];
            const float w = ls == 0.f ? 0.f : exp2f(wsp[threadIdx.x * splits + sp] - M);
            wsp[threadIdx.x * splits + sp] = w;
            L += ls * w;
        }
        linv[threadIdx.x] = L;
    }
    named_sync(1, kWarps * 32);
    for (int e = threadIdx.x; e < NC * HD; e += kWarps * 32) {
        const int h = e / HD, d = e % HD;
        const float* po = part_o + (slot0 + h) * splits * HD + d;
        // every split's load in flight at once (splits <= 16), then the weighted sum in order
        float pv[16];
#pragma unroll
        for (int sp = 0; sp < 16; ++sp) pv[sp] = sp < splits ? __ldcg(po + (size_t)sp * HD) : 0.f;
        float O = 0.f;
#pragma unroll
        for (int sp = 0; sp < 16; ++sp) {
            const float w = sp < splits ? wsp[h * splits + sp] : 0.f;
            if (w != 0.f) O += pv[sp] * w;
        }
        const DCol oc = dcol(it, h, G);
        out[(size_t)oc.row * s.hq * HD + (kvh * G + oc.head) * HD + d] = __float2bfloat16_rn(O / linv[h]);
    }
    if (threadIdx.x == 0) stamp(5);
}

// Merge split partials -> normalised bf16 output.  grid = (n_items, hkv * 8 columns), block = HD.
template <int HD>
__global__ void decode_combine_kernel(const DecodeItem* __restrict__ items,
                                      const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml, int splits,
                                      __nv_bfloat16* __restrict__ out, int hq, int hkv) {
    pdl_trigger();
    pdl_wait();
    const int row = blockIdx.x, kvh = blockIdx.y / 8, c = blockIdx.y % 8, d = threadIdx.x;
    const DecodeItem it = items[row];
    if (c >= item_cols(it)) return;
    const int G = hq / hkv;
    const size_t base = (((size_t)row * hkv + kvh) * 8 + c) * splits;
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
    const DCol oc = dcol(it, c, G);
    out[(size_t)oc.row * hq * HD + (kvh * G + oc.head) * HD + d] = __float2bfloat16_rn(O / L);
}

// Persistent form for grids of more than one wave (small Green Context partitions): one wave
// of CTAs (two per SM) walks the (row, kv head, split) units round-robin, the producer streams
// the next unit's blocks while the consumers finish the current one (no CTA prologue / ring
// fill per unit).  The block a unit ends on is held past its last use as the warps' merge
// scratch and released after the unit's output; splits merge through fp32 partials by the
// last-arriving split (the arithmetic of the non-persistent path, split order: deterministic).
template <int HD>
__global__ void __launch_bounds__(kThreadsD, 2)
    decode_attn_persist_kernel(const __grid_constant__ CUtensorMap tmap_kv, const __nv_bfloat16* __restrict__ q,
                               const DecodeItem* __restrict__ items, const int32_t* __restrict__ tables,
                               __nv_bfloat16* __restrict__ out, float* __restrict__ part_o,
                               float* __restrict__ part_ml, int* __restrict__ counters, int n_items, int splits,
                               int pps, AttnShape s) {
    using C = DC<HD>;
    constexpr int MT = HD / 16;
    constexpr int kS = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
    uint8_t* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kRing);
    uint64_t* empty = full + kS;
    float* mls = reinterpret_cast<float*>(empty + kS);  // [warp][8][2]
    float* wsp = mls + kWarps * 16;                      // [8][16] split m -> weights (last arriver)
    float* lsp = wsp + 8 * 16;                           // [8][16] split l
    float* linv = lsp + 8 * 16;                          // [8]
    __shared__ int s_last;

    const int G = s.hq / s.hkv;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int units = n_items * s.hkv * splits;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_kv);
        for (int i = 0; i < kS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();
    pdl_trigger();

    if (warp == kWarps) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            bool waited = false;
            int gi = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const int item = u / (s.hkv * splits), kvh = (u / splits) % s.hkv, sp = u % splits;
                const DecodeItem it = items[item];
                const int n_pages = (item_keys(it, G) + kBlockTokens - 1) / kBlockTokens;
                const int p0 = sp * pps, n_local = max(0, min(n_pages, p0 + pps) - p0);
                const int new_page = s.no_prewait ? 0 : it.pad / kBlockTokens;  // first block this step writes
                const int32_t* table = tables + it.table_off;
                for (int i = 0; i < n_local; ++i, ++gi) {
                    // only the block holding this step's token depends on the kernel before us
                    if (!waited && p0 + i >= new_page) {
                        pdl_wait();
                        waited = true;
                    }
                    const int st = gi % kS;
                    mbar_wait(&empty[st], ((gi / kS) & 1) ^ 1);
                    mbar_expect_tx(&full[st], C::kStage);
                    const int page = (s.layer * s.num_blocks + table[p0 + i]) * s.hkv + kvh;
                    tma_load_5d_hint(ring + st * C::kStage, &tmap_kv, &full[st], 0, 0, 0, 0, page, pol);
                }
            }
            if (!waited) pdl_wait();
        }
        return;  // the producer warp takes no part in the consumers' named barriers
    }

    // ---------------------------------------------------------------- consumers
    pdl_wait();  // q comes from the kernel before us
    const int tid = threadIdx.x;
    const int g = lane >> 2, t = lane & 3;
    const int kw = warp * 16;
    int gi = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const int item = u / (s.hkv * splits), kvh = (u / splits) % s.hkv, sp = u % splits;
        const DecodeItem it = items[item];
        const int NC = item_cols(it);
        const int n_pages = (item_keys(it, G) + kBlockTokens - 1) / kBlockTokens;
        const int p0 = sp * pps, n_local = max(0, min(n_pages, p0 + pps) - p0);
        uint32_t qb[HD / 16][2];
        {
            const DCol qc = dcol(it, g, G);
            const __nv_bfloat16* qrow = q + (size_t)qc.row * s.hq * HD + (size_t)(kvh * G + qc.head) * HD;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                if (qc.lim > 0) {
                    qb[kk][0] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t);
                    qb[kk][1] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t + 8);
                } else {
                    qb[kk][0] = qb[kk][1] = 0u;
                }
            }
        }
        float o[MT][4];
#pragma unroll
        for (int n = 0; n < MT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
        float m_run[2] = {-FLT_MAX, -FLT_MAX}, l_run[2] = {0.f, 0.f};
        const int lim[2] = {dcol(it, 2 * t, G).lim, dcol(it, 2 * t + 1, G).lim};
        int st = 0;
        for (int i = 0; i < n_local; ++i, ++gi) {
            st = gi % kS;
            mbar_wait(&full[st], (gi / kS) & 1);
            if (!s.dbg_load_only)
                attn_page<HD>(smem_u32(ring + st * C::kStage), kw, (p0 + i) * kBlockTokens + kw, lim, qb, o,
                              m_run, l_run, s.scale_log2, lane);
            __syncwarp();
            if (lane == 0 && i + 1 < n_local) mbar_arrive(&empty[st]);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            l_run[j] += __shfl_xor_sync(0xffffffffu, l_run[j], 4);
            l_run[j] += __shfl_xor_sync(0xffffffffu, l_run[j], 8);
            l_run[j] += __shfl_xor_sync(0xffffffffu, l_run[j], 16);
        }
        const size_t slot0 = ((size_t)item * s.hkv + kvh) * 8 * splits + sp;  // column h: slot0 + h * splits
        if (n_local > 0) {
            // ---- merge the warps through the held block, then this unit's output
            float* mrg = reinterpret_cast<float*>(ring + st * C::kStage);  // [warp][8][HD]
            named_sync(1, kWarps * 32);
            float* mw = mrg + warp * 8 * HD;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const int h = 2 * t + j;  // column
                if (h < NC) {
#pragma unroll
                    for (int mt = 0; mt < MT; ++mt) {
                        mw[h * HD + mt * 16 + g] = o[mt][j];
                        mw[h * HD + mt * 16 + g + 8] = o[mt][2 + j];
                    }
                    if (g == 0) {
                        mls[(warp * 8 + h) * 2] = m_run[j];
                        mls[(warp * 8 + h) * 2 + 1] = l_run[j];
                    }
                }
            }
            named_sync(1, kWarps * 32);
            for (int e = tid; e < NC * HD; e += kWarps * 32) {
                const int h = e / HD, d = e % HD;
                float M = -FLT_MAX;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) M = fmaxf(M, mls[(w * 8 + h) * 2]);
                float L = 0.f, O = 0.f;
#pragma unroll
                for (int w = 0; w < kWarps; ++w) {
                    const float lw = mls[(w * 8 + h) * 2 + 1];
                    if (lw == 0.f) continue;
                    const float f = exp2f(mls[(w * 8 + h) * 2] - M);
                    L += lw * f;
                    O += mrg[(w * 8 + h) * HD + d] * f;
                }
                if (splits == 1) {
                    const DCol oc = dcol(it, h, G);
                    out[(size_t)oc.row * s.hq * HD + (kvh * G + oc.head) * HD + d] =
                        __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
                } else {
                    const size_t sl = slot0 + (size_t)h * splits;
                    part_o[sl * HD + d] = O;
                    if (d == 0) {
                        part_ml[sl * 2 + 0] = M;
                        part_ml[sl * 2 + 1] = L;
                    }
                }
            }
            named_sync(1, kWarps * 32);  // done with the held block
            fence_proxy_async_smem();    // the merge scratch's generic writes before the next TMA
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
        } else if (tid < NC) {
            // an empty split (ragged contexts): contributes nothing to the merge
            const size_t sl = slot0 + (size_t)tid * splits;
            part_ml[sl * 2 + 0] = -FLT_MAX;
            part_ml[sl * 2 + 1] = 0.f;
        }
        if (splits == 1) continue;
        // ---- last-arriving split of (row, kv head) merges all splits in split order
        __threadfence();
        named_sync(1, kWarps * 32);
        if (tid == 0) {
            int* cnt = counters + item * s.hkv + kvh;
            const int prev = atomicAdd(cnt, 1);
            s_last = prev == splits - 1;
            if (s_last) *cnt = 0;
        }
        named_sync(1, kWarps * 32);
        if (!s_last) continue;
        __threadfence();
        for (int i = tid; i < NC * splits; i += kWarps * 32) {
            const int h = i / splits, q2 = i % splits;
            const size_t sl = slot0 - sp + ((size_t)h * splits + q2);
            wsp[h * 16 + q2] = __ldcg(part_ml + sl * 2);
            lsp[h * 16 + q2] = __ldcg(part_ml + sl * 2 + 1);
        }
        named_sync(1, kWarps * 32);
        if (tid < NC) {
            float M = -FLT_MAX;
            for (int q2 = 0; q2 < splits; ++q2) M = fmaxf(M, wsp[tid * 16 + q2]);
            float L = 0.f;
            for (int q2 = 0; q2 < splits; ++q2) {
                const float ls = lsp[tid * 16 + q2];
                const float w = ls == 0.f ? 0.f : exp2f(wsp[tid * 16 + q2] - M);
                wsp[tid * 16 + q2] = w;
                L += ls * w;
            }
            linv[tid] = L;
        }
        named_sync(1, kWarps * 32);
        for (int e = tid; e < NC * HD; e += kWarps * 32) {
            const int h = e / HD, d = e % HD;
            const float* po = part_o + (slot0 - sp + (size_t)h * splits) * HD + d;
            float pv[16];
#pragma unroll
            for (int q2 = 0; q2 < 16; ++q2) pv[q2] = q2 < splits ? __ldcg(po + (size_t)q2 * HD) : 0.f;
            float O = 0.f;
#pragma unroll
            for (int q2 = 0; q2 < 16; ++q2) {
                const float w = q2 < splits ? wsp[h * 16 + q2] : 0.f;
                if (w != 0.f) O += pv[q2] * w;
            }
            const DCol oc = dcol(it, h, G);
            out[(size_t)oc.row * s.hq * HD + (kvh * G + oc.head) * HD + d] = __float2bfloat16_rn(O / linv[h]);
        }
        named_sync(1, kWarps * 32);  // wsp / mls reused by the next unit
    }
}

template <int HD>
cudaError_t launch_persist(const CUtensorMap& tkv, const __nv_bfloat16* q, const DecodeItem* items, int n_items,
                           int splits, int pps, const int32_t* tables, __nv_bfloat16* out, float* po, float* pml,
                           int* cnt, int num_sms, const AttnShape& s, cudaStream_t st) {
    using C = DC<HD>;
    const int smem = C::kRing + 2 * C::kStages * 8 + (kWarps * 16 + 2 * 8 * 16 + 8) * 4 + 1024;
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(decode_attn_persist_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int units = n_items * s.hkv * splits;
    const int grid = std::min(units, 2 * std::max(1, num_sms));
    return launch_k(decode_attn_persist_kernel<HD>, dim3(grid), dim3(kThreadsD), smem, st, tkv, q, items, tables, out,
                    po, pml, cnt, n_items, splits, pps, s);
}

template <int HD>
cudaError_t launch_hd(const CUtensorMap& tkv, const __nv_bfloat16* q, const DecodeItem* items, int n_items,
                      int splits, int pps, const int32_t* tables, __nv_bfloat16* out, float* po, float* pml,
                      int* cnt, const AttnShape& s, cudaStream_t st) {
    using C = DC<HD>;
    const int smem = C::kRing + 2 * C::kStages * 8 + kWarps * 16 * 4 + 1024;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid(n_items, s.hkv, splits);
    // splits <= 8: one thread-block cluster per (row, kv head), merged over DSMEM
    static const bool no_cluster = std::getenv("ASB_ATTN_NO_CLUSTER") != nullptr;
    const int cmerge = (splits > 1 && splits <= 8 && !no_cluster) ? 1 : 0;
    cudaError_t e;
    if (cmerge) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(kThreadsD);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute a[2];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 1;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = splits;
        int na = 1;
        if (pdl_for_launch(true)) {
            a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            a[1].val.programmaticStreamSerializationAllowed = 1;
            na = 2;
        }
        cfg.attrs = a;
        cfg.numAttrs = na;
        return cudaLaunchKernelEx(&cfg, decode_attn_kernel<HD>, tkv, q, items, tables, out, po, pml, cnt, pps,
                                  cmerge, s);
    }
    e = launch_k(decode_attn_kernel<HD>, grid, dim3(kThreadsD), smem, st, tkv, q, items, tables, out, po, pml,
                 cnt, pps, 0, s);
    if (e == cudaSuccess && splits > 1 && !cnt)
        e = launch_k(decode_combine_kernel<HD>, dim3(n_items, s.hkv * 8), dim3(HD), 0, st, items,
                     static_cast<const float*>(po), static_cast<const float*>(pml), splits, out, s.hq, s.hkv);
    return e;
}

}  // namespace

int decode_splits(int n_items, int hkv, int max_ctx, int num_sms, int max_splits) {
    // Split-KV count of the one-wave grid (items <= two resident CTAs per SM; larger batches
    // take the persistent kernel): the most splits that still fit ONE wave, >= 3 blocks (192
    // keys) per split.  A second wave is never cheaper here: a CTA costs a fixed ~12 us (q
    // load, ring fill, merge) on top of ~0.5 us per block, so the old makespan-in-waves rule
    // (which took 5 splits = 4 waves at 80 SMs, 7 at 112 for 128 (row, head) items) ran the
    // C3 B=16 attention at 53-60 us/layer on 80-112 SM partitions against 37 us with one
    // split (profiles/r2_decode_attn_levels.txt).
    const int pages = (max_ctx + kBlockTokens - 1) / kBlockTokens;
    const int base = std::max(n_items * hkv, 1);
    const int slots = 2 * std::max(num_sms, 1);
    const int cap = std::max(1, std::min(max_splits, pages / 3));
    // powers of two only: the split merge runs in a thread-block cluster of `splits` CTAs, and
    // 5-7 CTA clusters place badly (B=4 on 80-112 SMs: 25 us/layer with 5-7 splits vs 18.5 with
    // 4 or 8, profiles/r2_decode_attn_levels.txt)
    int sp = std::max(1, std::min(cap, slots / base));
    while (sp & (sp - 1)) sp &= sp - 1;
    return sp;
}

int decode_splits_persist(int base, int pages, int num_sms, int max_splits) {
    // The persistent grid runs when the (row, kv head) items already exceed one wave of CTAs, so
    // splitting KV only adds units, merges and per-unit fills: one split was fastest or tied at
    // every partition size measured (32-80 SMs, B=24/32 ctx 3000: e.g. 80 SMs B=32 68.8 us/layer
    // vs 84.7 with the old makespan model's 3 splits, profiles/r2_decode_attn_persist_splits.txt).
    (void)base;
    (void)pages;
    (void)num_sms;
    (void)max_splits;
    return 1;
}

cudaError_t decode_attention(const CUtensorMap& tmap_kv, const __nv_bfloat16* q, const DecodeItem* items,
                             int n_items, int max_ctx, const int32_t* tables, __nv_bfloat16* out,
                             float* part_o, float* part_ml, int* counters, int max_splits, int num_sms,
                             const AttnShape& s, cudaStream_t stream) {
    if (n_items <= 0) return cudaSuccess;
    if (s.hq / s.hkv > 8) return cudaErrorInvalidValue;
    // the cluster merge (launch_hd) takes up to 8 splits: a portable cluster
    static const bool no_cluster = std::getenv("ASB_ATTN_NO_CLUSTER") != nullptr;
    static const int force = std::getenv("ASB_DECODE_SPLITS") ? std::atoi(std::getenv("ASB_DECODE_SPLITS")) : 0;
    const int splits0 = force > 0 ? std::min(force, max_splits)  // partial buffers hold max_splits
                                  : decode_splits(n_items, s.hkv, max_ctx, num_sms,
                                                  no_cluster ? max_splits : std::min(max_splits, 8));
    const int pages = (max_ctx + kBlockTokens - 1) / kBlockTokens;
    // more (row, kv head) items than one wave of CTAs (small partitions, large batches): the
    // persistent kernel, splits by makespan with a per-unit overhead (ASB_DECODE_PERSIST=0: off)
    static const int persist_env = std::getenv("ASB_DECODE_PERSIST") ? std::atoi(std::getenv("ASB_DECODE_PERSIST")) : -1;
    const bool persist = force <= 0 && persist_env != 0 &&
                         (persist_env == 1 || n_items * s.hkv > 2 * std::max(1, num_sms)) && counters;
    if (persist) {
        static const int force_p = std::getenv("ASB_DECODE_PERSIST_SPLITS") ? std::atoi(std::getenv("ASB_DECODE_PERSIST_SPLITS")) : 0;
        const int sp = force_p > 0 ? std::min(force_p, std::min(max_splits, 16))
                                   : decode_splits_persist(n_items * s.hkv, pages, num_sms, max_splits);
        const int pps = (pages + sp - 1) / sp;
        const int splits = (pages + pps - 1) / pps;
        if (s.hd == 128)
            return launch_persist<128>(tmap_kv, q, items, n_items, splits, pps, tables, out, part_o, part_ml, counters,
                                       num_sms, s, stream);
        if (s.hd == 64)
            return launch_persist<64>(tmap_kv, q, items, n_items, splits, pps, tables, out, part_o, part_ml, counters,
                                      num_sms, s, stream);
        return cudaErrorInvalidValue;
    }
    const int pps = (pages + splits0 - 1) / splits0;
    const int splits = (pages + pps - 1) / pps;
    if (s.hd == 128)
        return launch_hd<128>(tmap_kv, q, items, n_items, splits, pps, tables, out, part_o, part_ml, counters, s,
                              stream);
    if (s.hd == 64)
        return launch_hd<64>(tmap_kv, q, items, n_items, splits, pps, tables, out, part_o, part_ml, counters, s,
                             stream);
    return cudaErrorInvalidValue;
}

}  // namespace asb
