// Paged decode attention (K2 in SURVEY §2.3) — one query token per decode row, the G query
// heads of one KV head per CTA.  HBM-bound: each context token's K and V row is streamed
// from HBM exactly once per (row, KV head).  Replaces the mu_D term of the reference's
// decode_step_duration_ms (/root/reference/proj/src/executor.cpp:90-92).
//
// CTA = 1 producer warp + kWarps consumer warps, split-KV over gridDim.z:
//   producer  : TMA (SWIZZLE_128B, evict-first) loads of 32-token K and V sub-blocks straight
//               from the paged pool into a kStages-deep smem ring, completion on mbarriers
//   consumers : each warp owns whole sub-blocks (no CTA-wide barrier per block).  The G <= 8
//               heads are the M rows of a warp-level bf16 tensor-core tile (m16n8k16):
//                 S = Q . K^T   (B fragments by ldmatrix from the swizzled K tile)
//                 online softmax on the S fragments (quad shuffles, per-warp m / l)
//                 O += P . V    (P re-packed from the S fragments in registers, V fragments
//                                by ldmatrix.trans)
//               ~230 instructions per 32-key sub-block for all heads at once, so the kernel
//               stays bandwidth-bound.  (tcgen05 needs M >= 64 — >= 8x wasted rows for
//               G <= 8 — and a TMEM round trip per block; a register-resident warp MMA is
//               the better fit for this memory-bound shape.)
//   epilogue  : warps merge (m, l, O) through smem; the CTA writes bf16 output (one split)
//               or fp32 partials merged by decode_combine_kernel.
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

constexpr int kSub = 32;   // tokens per streamed sub-block (half a KV block)
constexpr int kWarps = 4;  // consumer warps per CTA (two CTAs per SM, see DC::kStages)
constexpr int kThreadsD = (kWarps + 1) * 32;

template <int HD>
struct DC {
    static constexpr int kHalves = HD / 64;                // 64-column SW128 boxes per row
    static constexpr int kTile = kSub * HD * 2;            // one K (or V) sub-block, bytes
    static constexpr int kStage = 2 * kTile;
    // One stage per consumer warp (HD=128: 64 KB ring + 16 KB merge) or two (HD=64): two
    // CTAs per SM, i.e. 8 consumer warps and 128 KB of K/V in flight per SM.  Measured best
    // of the (warps, stages) sweep in profiles/r1_decode_attn_sweep.txt.
    static constexpr int kStages = HD == 128 ? 4 : 8;
    static constexpr int kRing = kStages * kStage;
};

// Stage of item i.  Item i is consumed by warp i % W; giving every warp its own S / W stages
// (visited in order) means each mbarrier has exactly one waiter that waits its phases
// strictly in sequence — with round-robin consumers sharing a ring, a fast warp could wait
// for phase k+2 of a stage while phase k+1 is still pending, and the parity-based wait would
// alias and return early.
__device__ __forceinline__ int stage_of(int i, int W, int S) { return (i % W) + W * ((i / W) % (S / W)); }

template <int HD>
__global__ void __launch_bounds__(kThreadsD, 2)
    decode_attn_kernel(const __grid_constant__ CUtensorMap tmap_k,
                       const __grid_constant__ CUtensorMap tmap_v,
                       const __nv_bfloat16* __restrict__ q, const DecodeItem* __restrict__ items,
                       const int32_t* __restrict__ tables, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ part_o, float* __restrict__ part_ml,
                       int* __restrict__ counters, int subs_per_split, int n_stages, int cluster_merge,
                       AttnShape s) {
    using C = DC<HD>;
    constexpr int NT = HD / 8;  // O n-tiles (8 dims each)
    const int kWarpsR = blockDim.x / 32 - 1;  // consumer warps
    const int kStagesR = n_stages;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
    uint8_t* ring = smem;
    float* mrg = reinterpret_cast<float*>(smem + kStagesR * C::kStage);  // [warp][8][HD]
    float* mls = mrg + kWarpsR * 8 * HD;                                 // [warp][8][2]
    uint64_t* full = reinterpret_cast<uint64_t*>(mls + kWarpsR * 16);
    uint64_t* empty = full + kStagesR;

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
    const int n_sub = (it.ctx_len + kSub - 1) / kSub;
    const int s0 = blockIdx.z * subs_per_split;
    const int n_local = max(0, min(n_sub, s0 + subs_per_split) - s0);
    const int32_t* table = tables + it.table_off;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_k);
        tma_prefetch_desc(&tmap_v);
        for (int i = 0; i < kStagesR; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        fence_barrier_init();
    }
    __syncthreads();
    pdl_trigger();

    if (warp == kWarpsR) {
        // ------------------------------------------------------------ producer
        // K/V of positions before this step's token were written by earlier steps: stream them
        // while the kernel before us (the QKV projection appending the new token) is still
        // running, and wait for it only before the sub-block that holds the new token.
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const int new_sub = (it.ctx_len - 1) / kSub;
            bool waited = false;
            for (int i = 0; i < n_local; ++i) {
                if (!waited && s0 + i >= new_sub) {
                    pdl_wait();
                    waited = true;
                }
                const int st = stage_of(i, kWarpsR, kStagesR);
                mbar_wait(&empty[st], ((i / kStagesR) & 1) ^ 1);
                mbar_expect_tx(&full[st], C::kStage);
                const int j = s0 + i;
                const int blk = table[j >> 1];
                const int row = ((s.layer * s.num_blocks + blk) * s.hkv + kvh) * kKvPageRows + (j & 1) * kSub;
                uint8_t* kd = ring + st * C::kStage;
                uint8_t* vd = kd + C::kTile;
#pragma unroll
                for (int h = 0; h < C::kHalves; ++h) {
                    tma_load_2d_hint(kd + h * (kSub * 128), &tmap_k, &full[st], h * 64, row, pol);
                    tma_load_2d_hint(vd + h * (kSub * 128), &tmap_v, &full[st], h * 64, row, pol);
                }
            }
            if (!waited) pdl_wait();
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    pdl_wait();  // q comes from the kernel before us
    if (threadIdx.x == 0) stamp(1);
    const int g = lane >> 2, t = lane & 3;  // fragment row / column-pair owner
    // Q A-fragments (rows = heads): (row g, k 2t..2t+1) and (row g, k 2t+8..2t+9); the
    // fragment registers of rows g+8 and of rows >= G are zero
    uint32_t qa[HD / 16][2];
    {
        const __nv_bfloat16* qrow = q + (size_t)it.q_row * s.hq * HD + (size_t)(kvh * G + g) * HD;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
            if (g < G) {
                qa[kk][0] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t);
                qa[kk][1] = *reinterpret_cast<const uint32_t*>(qrow + kk * 16 + 2 * t + 8);
            } else {
                qa[kk][0] = qa[kk][1] = 0u;
            }
        }
    }
    float o[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_run = -FLT_MAX, l_run = 0.f;

    for (int i = warp; i < n_local; i += kWarpsR) {
        const int st = stage_of(i, kWarpsR, kStagesR);
        mbar_wait(&full[st], (i / kStagesR) & 1);
        if (i == 0 && lane == 0) stamp(2);
        if (s.dbg_load_only) {  // timing ablation (ASB_DEBUG_SKIP=attnmath): the load stream alone
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            continue;
        }
        const uint32_t kt = smem_u32(ring + st * C::kStage);
        const uint32_t vt = kt + C::kTile;
        // ---- S = Q K^T : 4 n-tiles of 8 keys
        float sacc[4][4];
#pragma unroll
        for (int n = 0; n < 4; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
            for (int np = 0; np < 2; ++np) {  // pairs of key n-tiles
                // matrices: (ntile 2np, k lo), (2np, k hi), (2np+1, k lo), (2np+1, k hi)
                const int mi = lane >> 3;
                const int key = (2 * np + (mi >> 1)) * 8 + (lane & 7);
                const int chunk = 2 * kk + (mi & 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4(kt + sw_off<HD>(key, chunk), b0, b1, b2, b3);
                mma16816(sacc[2 * np], qa[kk][0], 0u, qa[kk][1], 0u, b0, b1);
                mma16816(sacc[2 * np + 1], qa[kk][0], 0u, qa[kk][1], 0u, b2, b3);
            }
        }
        // ---- online softmax on row g (keys 8n + 2t + {0,1})
        const int kbase = (s0 + i) * kSub;
        float mx = m_run;
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const bool ok = kbase + 8 * n + 2 * t + e < it.ctx_len;
                sacc[n][e] = ok ? sacc[n][e] * s.scale_log2 : -FLT_MAX;
                mx = fmaxf(mx, sacc[n][e]);
            }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        const float alpha = exp2f(m_run - mx);
        float psum = 0.f;
        uint32_t pa[2][2];  // P A-fragments for the two 16-key k-steps (row g)
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            const float p0 = sacc[n][0] == -FLT_MAX ? 0.f : exp2f(sacc[n][0] - mx);
            const float p1 = sacc[n][1] == -FLT_MAX ? 0.f : exp2f(sacc[n][1] - mx);
            const uint32_t pk = pack_bf16(p0, p1);
            psum += bf16_lo(pk) + bf16_hi(pk);  // sum what P.V will actually use
            pa[n >> 1][n & 1] = pk;
        }
        psum += __shfl_xor_sync(0xffffffffu, psum, 1);
        psum += __shfl_xor_sync(0xffffffffu, psum, 2);
        l_run = l_run * alpha + psum;
        m_run = mx;
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            o[n][0] *= alpha;
            o[n][1] *= alpha;
        }
        // ---- O += P V : 2 k-steps of 16 keys x NT n-tiles of 8 dims
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
            for (int dp = 0; dp < NT / 2; ++dp) {  // pairs of dim n-tiles
                const int mi = lane >> 3;
                const int key = ks * 16 + (mi & 1) * 8 + (lane & 7);
                const int chunk = 2 * dp + (mi >> 1);
                uint32_t b0, b1, b2, b3;
                ldsm_x4_t(vt + sw_off<HD>(key, chunk), b0, b1, b2, b3);
                mma16816(o[2 * dp], pa[ks][0], 0u, pa[ks][1], 0u, b0, b1);
                mma16816(o[2 * dp + 1], pa[ks][0], 0u, pa[ks][1], 0u, b2, b3);
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    }

    // ---------------------------------------------------------------- merge warps
    if (threadIdx.x == 0) stamp(3);
    float* mw = mrg + warp * 8 * HD;
    if (g < G) {
#pragma unroll
        for (int n = 0; n < NT; ++n) {
            mw[g * HD + n * 8 + 2 * t] = o[n][0];
            mw[g * HD + n * 8 + 2 * t + 1] = o[n][1];
        }
        if (t == 0) {
            mls[(warp * 8 + g) * 2] = m_run;
            mls[(warp * 8 + g) * 2 + 1] = l_run;
        }
    }
    named_sync(1, kWarpsR * 32);
    const bool single = gridDim.z == 1;
    const bool cmerge = !single && cluster_merge;
    // cluster merge: this CTA's (M, L, O) parked at the start of the drained ring
    float* cO = reinterpret_cast<float*>(ring);  // [G][HD]
    float* cM = cO + 8 * HD;                     // [G]
    float* cL = cM + 8;                          // [G]
    for (int e = threadIdx.x; e < G * HD; e += kWarpsR * 32) {
        const int h = e / HD, d = e % HD;
        float M = -FLT_MAX;
#pragma unroll
        for (int w = 0; w < kWarpsR; ++w) M = fmaxf(M, mls[(w * 8 + h) * 2]);
        float L = 0.f, O = 0.f;
#pragma unroll
        for (int w = 0; w < kWarpsR; ++w) {
            const float lw = mls[(w * 8 + h) * 2 + 1];
            if (lw == 0.f) continue;
            const float f = exp2f(mls[(w * 8 + h) * 2] - M);
            L += lw * f;
            O += mrg[(w * 8 + h) * HD + d] * f;
        }
        const int hh = kvh * G + h;
        if (single) {
            out[(size_t)it.q_row * s.hq * HD + hh * HD + d] = __float2bfloat16_rn(L > 0.f ? O / L : 0.f);
        } else if (cmerge) {
            cO[h * HD + d] = O;
            if (d == 0) {
                cM[h] = M;
                cL[h] = L;
            }
        } else {
            const size_t slot = ((size_t)blockIdx.x * s.hq + hh) * gridDim.z + blockIdx.z;
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
        const int n = G * HD, lo = (n * r) / S, hi = (n * (r + 1)) / S;
        const uint32_t bO = smem_u32(cO), bM = smem_u32(cM), bL = smem_u32(cL);
        for (int e = lo + threadIdx.x; e < hi; e += kWarpsR * 32) {
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
            out[(size_t)it.q_row * s.hq * HD + (kvh * G + h) * HD + d] = __float2bfloat16_rn(O / L);
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
    named_sync(1, kWarpsR * 32);
    if (threadIdx.x == 0) {
        int* cnt = counters + blockIdx.x * gridDim.y + kvh;
        const int prev = atomicAdd(cnt, 1);
        last_s = prev == static_cast<int>(gridDim.z) - 1;
        if (last_s) *cnt = 0;
    }
    named_sync(1, kWarpsR * 32);
    if (threadIdx.x == 0) stamp(4);
    if (!last_s) return;
    __threadfence();
    // per (head, split) weight exp2(m - M) and the normaliser L, once per head, in smem (the
    // ring is drained); then one pass over part_o with every split's load in flight
    const int splits = gridDim.z;
    float* wsp = reinterpret_cast<float*>(smem);  // [G][splits]
    float* linv = wsp + 8 * splits;               // [G]
    float* lsp = linv + 8;  // [G][splits] l
    for (int i = threadIdx.x; i < G * splits; i += kWarpsR * 32) {  // all (m, l) loads at once
        const int h = i / splits, sp = i % splits;
        const size_t sl = ((size_t)blockIdx.x * s.hq + kvh * G + h) * splits + sp;
        wsp[i] = __ldcg(part_ml + sl * 2);
        lsp[i] = __ldcg(part_ml + sl * 2 + 1);
    }
    named_sync(1, kWarpsR * 32);
    if (threadIdx.x < G) {
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
    named_sync(1, kWarpsR * 32);
    for (int e = threadIdx.x; e < G * HD; e += kWarpsR * 32) {
        const int h = e / HD, d = e % HD;
        const int hh = kvh * G + h;
        const float* po = part_o + ((size_t)blockIdx.x * s.hq + hh) * splits * HD + d;
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
        out[(size_t)it.q_row * s.hq * HD + hh * HD + d] = __float2bfloat16_rn(O / linv[h]);
    }
    if (threadIdx.x == 0) stamp(5);
}

// Merge split partials -> normalised bf16 output.  grid = (n_items, hq), block = HD.
template <int HD>
__global__ void decode_combine_kernel(const DecodeItem* __restrict__ items,
                                      const float* __restrict__ part_o,
                                      const float* __restrict__ part_ml, int splits,
                                      __nv_bfloat16* __restrict__ out, int hq) {
    pdl_trigger();
    pdl_wait();
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

template <int HD>
cudaError_t launch_hd(const CUtensorMap& tk, const CUtensorMap& tv, const __nv_bfloat16* q,
                      const DecodeItem* items, int n_items, int splits, int sps, const int32_t* tables,
                      __nv_bfloat16* out, float* po, float* pml, int* cnt, const AttnShape& s, cudaStream_t st) {
    using C = DC<HD>;
    static const int warps = std::getenv("ASB_DECODE_WARPS") ? std::atoi(std::getenv("ASB_DECODE_WARPS")) : kWarps;
    static const int stages0 = std::getenv("ASB_DECODE_STAGES") ? std::atoi(std::getenv("ASB_DECODE_STAGES")) : C::kStages;
    static const int stages = std::max(warps, (stages0 / warps) * warps);  // multiple of warps
    const int smem = stages * C::kStage + warps * 8 * HD * 4 + warps * 16 * 4 + 2 * stages * 8 + 1024;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(decode_attn_kernel<HD>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, 232448 - 1024);
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
        cfg.blockDim = dim3((warps + 1) * 32);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute a[2];
        a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = 1;
        a[0].val.clusterDim.y = 1;
        a[0].val.clusterDim.z = splits;
        int na = 1;
        if (tl_pdl) {
            a[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            a[1].val.programmaticStreamSerializationAllowed = 1;
            na = 2;
        }
        cfg.attrs = a;
        cfg.numAttrs = na;
        e = cudaLaunchKernelEx(&cfg, decode_attn_kernel<HD>, tk, tv, q, items, tables, out, po, pml, cnt, sps,
                               stages, cmerge, s);
        return e;
    }
    e = launch_k(decode_attn_kernel<HD>, grid, dim3((warps + 1) * 32), smem, st, tk, tv, q, items,
                 tables, out, po, pml, cnt, sps, stages, 0, s);
    if (e == cudaSuccess && splits > 1 && !cnt)
        e = launch_k(decode_combine_kernel<HD>, dim3(n_items, s.hq), dim3(HD), 0, st, items,
                     static_cast<const float*>(po), static_cast<const float*>(pml), splits, out, s.hq);
    return e;
}

}  // namespace

int decode_splits(int n_items, int hkv, int max_ctx, int num_sms, int max_splits) {
    // Split-KV count minimising the makespan in waves of two resident CTAs per SM: a CTA of
    // s splits does 1/s of an item's stream, so the cost is ceil(items*s / slots) / s, plus a
    // small merge charge per extra split.  With items <= slots this is the one-wave rule
    // (C3 73% -> 84%, C4 84% -> 92% of HBM peak on the full device); on a Green Context
    // partition it also avoids ragged second waves (128 (row, head) items on a 48-SM
    // partition: 1 split = 2 waves of full items, 3 splits = 4 waves of 1/3 items = 1.33).
    // >= 2 sub-blocks per consumer warp.
    const int subs = (max_ctx + kSub - 1) / kSub;
    const int base = std::max(n_items * hkv, 1);
    const int slots = 2 * std::max(num_sms, 1);
    const int cap = std::max(1, std::min(max_splits, subs / (2 * kWarps)));
    int best = 1;
    double best_t = 1e30;
    for (int sp = 1; sp <= cap; ++sp) {
        const double waves = double((int64_t(base) * sp + slots - 1) / slots);
        const double t = waves / sp * (1.0 + 0.03 * (sp - 1));
        if (t < best_t - 1e-9) {
            best_t = t;
            best = sp;
        }
    }
    return best;
}

cudaError_t decode_attention(const CUtensorMap& tmap_k32, const CUtensorMap& tmap_v32,
                             const __nv_bfloat16* q, const DecodeItem* items, int n_items,
                             int max_ctx, const int32_t* tables, __nv_bfloat16* out,
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
    const int subs = (max_ctx + kSub - 1) / kSub;
    const int sps = (subs + splits0 - 1) / splits0;
    const int splits = (subs + sps - 1) / sps;
    if (s.hd == 128)
        return launch_hd<128>(tmap_k32, tmap_v32, q, items, n_items, splits, sps, tables, out, part_o,
                              part_ml, counters, s, stream);
    if (s.hd == 64)
        return launch_hd<64>(tmap_k32, tmap_v32, q, items, n_items, splits, sps, tables, out, part_o,
                             part_ml, counters, s, stream);
    return cudaErrorInvalidValue;
}

}  // namespace asb
