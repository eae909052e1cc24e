// tcgen05 GEMM for the SLM linear layers (K5 in SURVEY §2.3):
//   Y[tok][n] = sum_k X[tok][k] * W[n][k]   (+ bias / + residual / SiLU·mul / fp32)
//
// Replaces the simulated cost terms of the reference's executor
// (decode_step_duration_ms, /root/reference/proj/src/executor.cpp:84-97, and the
// prefill rate x length arithmetic, /root/reference/proj/src/engine.cpp:450-475).
//
// Structure (192 threads, one CTA per SM):
//   warp 0      : TMA producer   (A/B tiles -> smem ring, SWIZZLE_128B, mbarrier tx)
//   warp 1      : MMA issuer     (one elected lane, tcgen05.mma kind::f16, commit)
//   warps 2..5  : epilogue       (tcgen05.ld TMEM -> regs -> fused epilogue -> HBM)
//
// Two operand orders:
//   normal (prefill, many tokens):  A = X (tokens, M = 128 rows/tile), B = W (BN = 256/128)
//   swap   (decode, <= 256 tokens): A = W (128 weight rows/tile),       B = X (BN = tokens)
// and two schedules:
//   persistent (splits == 1): CTAs stride over tiles; TMEM holds two accumulators so the
//     epilogue of tile i overlaps the MMAs of tile i+1.
//   cluster split-K (swap, splits = S > 1): the S CTAs of one thread-block cluster each
//     stream 1/S of a weight tile's K range, park their fp32 partial in shared memory and
//     reduce it through DSMEM in rank order -- a fixed summation order (bit-reproducible),
//     no workspace, no atomics, no second launch.  This is what lets a 9-tile projection
//     stream its weights on ~all SMs at decode batch sizes.
// Launches carry the programmatic-dependent-launch attribute: the producer streams the first
// ring of WEIGHT tiles before griddepcontrol.wait (weights never depend on the previous
// kernel), so the weight fetch overlaps the tail of the kernel before it.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>

#include "attn.h"
#include "epi.cuh"
#include "gemm.h"
#include "launch.cuh"
#include "sm100.cuh"

namespace asb {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kThreads = 192;

// KP = 64-wide k-blocks per pipeline stage.  The decode (swap) path at BN <= 64 uses KP = 2:
// one 32 KiB weight box + one activation box per stage.  TMA throughput per SM is set by the
// request size more than by the requests in flight (scripts/probes/stream.cu on a 16-SM
// partition: 16 KiB requests ~90 GB/s/SM, 32 KiB ~150), and a decode step on a small Green
// Context partition is exactly that per-SM stream.
template <int BN, int KP = 1>
struct GemmCfg {
    static constexpr int kStages = KP == 2 ? (BN <= 32 ? 5 : 4) : (BN >= 256 ? 4 : (BN >= 128 ? 6 : 8));
    static constexpr int kBytesA = BM * BK * 2 * KP;
    static constexpr int kBytesB = BN * BK * 2 * KP;
    static constexpr int kStageBytes = kBytesA + kBytesB;
    static constexpr int kTmemCols = (2 * BN) <= 32 ? 32 : 2 * BN;  // power of two >= 32
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
    // cluster split-K parks a [BN tokens][128 rows] fp32 partial in the (drained) ring
    static_assert(BN * BM * 4 <= kStages * kStageBytes, "partial does not fit the ring");
};

// Apply the epilogue to one output value (all modes except SiLU).
struct Epi {
    GemmParams p;

    __device__ __forceinline__ void store(int tok, int n, float v) const {
        if (tok >= p.tokens || n >= p.n_out) return;
        switch (p.epi) {
        case EPI_BF16: {
            if (p.bias) v += __bfloat162float(p.bias[n]);
            p.out[static_cast<size_t>(tok) * p.ldo + n] = __float2bfloat16_rn(v);
            break;
        }
        case EPI_RESID: {
            v += __bfloat162float(p.resid[static_cast<size_t>(tok) * p.ldr + n]);
            p.out[static_cast<size_t>(tok) * p.ldo + n] = __float2bfloat16_rn(v);
            break;
        }
        case EPI_F32:
            p.out_f32[static_cast<size_t>(tok) * p.ldo + n] = v;
            break;
        default:
            break;
        }
    }

    // Swap-path pair (weight rows m, m+1; m even) for one token: SiLU consumes the pair
    // (interleaved gate/up rows), every other mode stores two neighbouring outputs.
    __device__ __forceinline__ void store_pair(int tok, int m, float v0, float v1) const {
        if (tok >= p.tokens || m >= p.n_out) return;
        const size_t o = static_cast<size_t>(tok) * p.ldo;
        if (p.epi == EPI_SILU) {
            p.out[o + (m >> 1)] = __float2bfloat16_rn(silu(v0) * v1);
            return;
        }
        const bool two = m + 1 < p.n_out;
        if (p.epi == EPI_BF16 && p.bias) {
            v0 += __bfloat162float(p.bias[m]);
            if (two) v1 += __bfloat162float(p.bias[m + 1]);
        }
        if (p.epi == EPI_RESID) {
            const __nv_bfloat16* r = p.resid + static_cast<size_t>(tok) * p.ldr + m;
            if (two && ((p.ldr & 1) == 0)) {
                const uint32_t w = *reinterpret_cast<const uint32_t*>(r);
                v0 += bf16_lo(w);
                v1 += bf16_hi(w);
            } else {
                v0 += __bfloat162float(r[0]);
                if (two) v1 += __bfloat162float(r[1]);
            }
        }
        if (p.epi == EPI_F32) {
            if (two && ((p.ldo & 1) == 0)) {
                *reinterpret_cast<float2*>(p.out_f32 + o + m) = make_float2(v0, v1);
            } else {
                p.out_f32[o + m] = v0;
                if (two) p.out_f32[o + m + 1] = v1;
            }
            return;
        }
        if (two && ((p.ldo & 1) == 0)) {
            *reinterpret_cast<uint32_t*>(p.out + o + m) = pack_bf16(v0, v1);
        } else {
            p.out[o + m] = __float2bfloat16_rn(v0);
            if (two) p.out[o + m + 1] = __float2bfloat16_rn(v1);
        }
    }
};

// ---- fused QKV epilogue helpers (EPI_QKV); bf16r / pool_off / rope2 live in epi.cuh
__device__ __forceinline__ void store32_bf16(__nv_bfloat16* dst, const float (&v)[32]) {
    uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int q = 0; q < 4; ++q)
        d4[q] = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                           pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
}

// Destination of the rotated head `head` (q heads first, then k heads) for one token.
__device__ __forceinline__ __nv_bfloat16* rot_dst(const RopeEpi& R, int tok, int sl, int head) {
    return head < R.hq ? R.q_out + ((size_t)tok * R.hq + head) * R.hd
                       : R.k_pool + pool_off(R, sl, head - R.hq);
}

// Work decomposition shared by the producer, MMA and epilogue roles: units (tile, split)
// strided over the grid.  splits == 1: persistent over tiles.  splits > 1: grid == units,
// one unit per CTA, and the S splits of a tile are the S CTAs of one cluster (rank = split).
struct Work {
    int tiles_m, k_blocks, units, splits, kbps, u;
    __device__ void init(const GemmParams& p, int tm_, int tn_, int kb) {
        tiles_m = tm_;
        k_blocks = kb;
        splits = p.splits > 1 ? p.splits : 1;
        kbps = splits > 1 ? p.kb_per_split : kb;
        units = tm_ * tn_ * splits;
        u = blockIdx.x;
    }
    __device__ bool next(int& tm, int& tn, int& kb0, int& kb1) {
        if (u >= units) return false;
        const int split = u % splits;
        const int tile = u / splits;
        kb0 = split * kbps;
        kb1 = min(k_blocks, kb0 + kbps);
        u += gridDim.x;
        tm = tile % tiles_m;
        tn = tile / tiles_m;
        return true;
    }
};

template <int BN, int KP>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b, const GemmParams p) {
    using C = GemmCfg<BN, KP>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + C::kStages * C::kBytesA;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty_bar = full_bar + C::kStages;
    uint64_t* tfull_bar = empty_bar + C::kStages;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint64_t* recv_bar = tempty_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(recv_bar + 1);
    float* part = reinterpret_cast<float*>(smem);  // cluster split-K partial [BN][128]

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    // staged swap epilogue: the tile's fp32 partial is parked in smem and finished from there
    // (cluster split-K reduction over DSMEM, and/or the cross-row QKV/RoPE epilogue)
    const bool clustered = p.swap && (p.splits > 1 || p.epi == EPI_QKV);
    // Split-K reduction by bulk push: CTA r of the S-CTA cluster finishes the weight rows of
    // slice r (4-row units, [ro(r), ro(r+1))); every CTA parks its partial slice-major
    // ([slice][token][row]) and pushes slice q to CTA q with one cp.async.bulk smem->DSMEM
    // copy, landing in q's (now idle) operand ring; q sums the S slices from local smem in
    // rank order (the pull reduction's order: bit-identical).  The QKV/RoPE epilogue needs
    // row pairs (j, j + hd/2) from different slices and keeps the DSMEM-load reduction.
    const int S_ = p.splits > 1 ? p.splits : 1;
    // (from 32 tokens: below that the DSMEM loads are few and the copy + fence latency loses)
    const bool bulk = clustered && S_ > 1 && p.epi != EPI_QKV && !p.reduce_pull && BN <= 128 && p.tokens >= 32;
    const int Tp = p.tokens < BN ? p.tokens : BN;
    auto ro = [&](int r) { return 4 * ((32 * r) / S_); };
    auto stamp = [&](int k) {
        if (p.dbg_times) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            p.dbg_times[blockIdx.x * 8 + k] = t;
        }
    };
    if (threadIdx.x == 0) stamp(0);

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmap_a);
        tma_prefetch_desc(&tmap_b);
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull_bar[b], 1);
            mbar_init(&tempty_bar[b], 128);
        }
        mbar_init(recv_bar, 1);
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc<C::kTmemCols>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) stamp(6);
    pdl_trigger();

    const int tiles_m = (p.M + BM - 1) / BM;
    const int tiles_n = (p.N + BN - 1) / BN;
    const int k_blocks = ((p.K + BK - 1) / BK + KP - 1) / KP;  // pipeline k-units of KP blocks

    if (warp == 0) {
        if (elect_one()) {
            // swap (decode): each weight tile is read by exactly one CTA -> evict-first; the
            // tiny activation operand is shared by all -> evict-last.  normal (prefill): a
            // weight tile is re-read by every M-tile in flight and the activation panel by
            // every N-tile, so both are kept (evict-last).
            const uint64_t pol_w = p.swap ? policy_evict_first() : policy_evict_last();
            const uint64_t pol_x = policy_evict_last();
            // Weight operand: A in swap, B in normal.  Activations: the other one.
            auto load_w = [&](int stage, int kb, int tm, int tn) {
                if (p.swap) {
                    if (p.a_packed)  // box = KP consecutive k-blocks of one packed 128-row tile
                        tma_load_4d_hint(smem_a + stage * C::kBytesA, &tmap_a, &full_bar[stage], 0, 0, kb * KP, tm, pol_w);
                    else
                        tma_load_2d_hint(smem_a + stage * C::kBytesA, &tmap_a, &full_bar[stage], kb * BK, tm * BM, pol_w);
                } else {
                    if (p.b_packed)
                        tma_load_4d_hint(smem_b + stage * C::kBytesB, &tmap_b, &full_bar[stage], 0, 0, kb,
                                         tn * (BN / 128), pol_w);
                    else
                        tma_load_2d_hint(smem_b + stage * C::kBytesB, &tmap_b, &full_bar[stage], kb * BK, tn * BN, pol_w);
                }
            };
            auto load_x = [&](int stage, int kb, int tm, int tn) {
                if (p.swap && KP == 2)  // 3-D view (64 cols, tokens, k-block): box [2][BN][64]
                    tma_load_3d(smem_b + stage * C::kBytesB, &tmap_b, &full_bar[stage], 0, tn * BN, kb * KP);
                else if (p.swap)
                    tma_load_2d_hint(smem_b + stage * C::kBytesB, &tmap_b, &full_bar[stage], kb * BK, tn * BN, pol_x);
                else
                    tma_load_2d_hint(smem_a + stage * C::kBytesA, &tmap_a, &full_bar[stage], kb * BK, tm * BM, pol_x);
            };
            // Swap path: the smem ring holds only a few units of the weight stream, so on a small
            // partition the in-flight bytes per SM (not HBM) bound the rate.  Prefetch the
            // weight stream l2_pf units ahead of the TMA loads into L2 (no smem needed).
            const int pf = (p.swap && p.a_packed && p.w_packed) ? p.l2_pf : 0;
            auto pf_w = [&](int kb, int tm) {
                const int k0 = kb * KP;
                const int nk = min(KP, p.w_kblocks - k0);
                if (nk <= 0) return;
                prefetch_l2_bulk(p.w_packed + (static_cast<size_t>(tm) * p.w_kblocks + k0) * (BM * BK),
                                 static_cast<uint32_t>(nk * BM * BK * 2));
            };
            Work w;
            w.init(p, tiles_m, tiles_n, k_blocks);
            // Weights do not depend on the previous kernel: fill the first ring with weight
            // tiles, then wait for the producer of our activations.
            int pre = 0;
            {
                Work w0 = w;
                int tm, tn, kb0, kb1;
                if (w0.next(tm, tn, kb0, kb1)) {
                    for (int kb = kb0; kb < kb1 && pre < C::kStages; ++kb, ++pre) {
                        mbar_expect_tx(&full_bar[pre], C::kStageBytes);
                        load_w(pre, kb, tm, tn);
                    }
                    for (int kb = kb0 + pre; kb < kb1 && kb < kb0 + pre + pf; ++kb) pf_w(kb, tm);
                }
            }
            pdl_wait();
            uint32_t stage = 0, phase = 0;
            int i = 0;
            int tm, tn, kb0, kb1;
            while (w.next(tm, tn, kb0, kb1)) {
                for (int kb = kb0; kb < kb1; ++kb, ++i) {
                    if (i >= pre) {
                        if (pf) {
                            if (kb == kb0)  // a later tile of a persistent CTA: open its window
                                for (int u = kb0 + 1; u < kb1 && u < kb0 + pf; ++u) pf_w(u, tm);
                            if (kb + pf < kb1) pf_w(kb + pf, tm);
                        }
                        mbar_wait(&empty_bar[stage], phase ^ 1);
                        mbar_expect_tx(&full_bar[stage], C::kStageBytes);
                        load_w(stage, kb, tm, tn);
                    }
                    load_x(stage, kb, tm, tn);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
        __syncwarp();  // reconverge before the CTA barrier (bar.sync is warp-aligned)
    } else if (warp == 1) {
        constexpr uint32_t idesc = make_idesc_bf16(BM, BN, false, false);
        uint32_t stage = 0, phase = 0;
        uint32_t local = 0;
        Work w;
        w.init(p, tiles_m, tiles_n, k_blocks);
        int tm, tn, kb0, kb1;
        for (; w.next(tm, tn, kb0, kb1); ++local) {
            const uint32_t ab = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tempty_bar[ab], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + ab * BN;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&full_bar[stage], phase);
                if (local == 0 && kb == kb0 && lane == 0) stamp(4);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a_addr = smem_u32(smem_a + stage * C::kBytesA);
                    const uint32_t b_addr = smem_u32(smem_b + stage * C::kBytesB);
#pragma unroll
                    for (int kk = 0; kk < KP; ++kk)
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k) {
                            const uint64_t ad = make_sw128_desc(a_addr + kk * (BM * 128) + k * 32, 16, 1024);
                            const uint64_t bd = make_sw128_desc(b_addr + kk * (BN * 128) + k * 32, 16, 1024);
                            umma_bf16(d_tmem, ad, bd, idesc, (kb > kb0 || kk > 0 || k > 0) ? 1u : 0u);
                        }
                    umma_commit(&empty_bar[stage]);
                }
                __syncwarp();
                if (++stage == C::kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (elect_one()) umma_commit(&tfull_bar[ab]);
            __syncwarp();
        }
        if (lane == 0) stamp(1);
    } else {
        // Epilogue warps 2..5: TMEM lane quarter = warp % 4.
        pdl_wait();  // residual / output buffers belong to the previous kernels
        const uint32_t quarter = warp & 3;
        const uint32_t row_in_tile = quarter * 32 + lane;
        Epi epi{p};
        uint32_t local = 0;
        Work w;
        w.init(p, tiles_m, tiles_n, k_blocks);
        int tm, tn, kb0, kb1;
        for (; w.next(tm, tn, kb0, kb1); ++local) {
            const uint32_t ab = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            mbar_wait(&tfull_bar[ab], acc_phase);
            if (local == 0 && threadIdx.x == 64) stamp(5);
            tc_fence_after();
            const int m = tm * BM + row_in_tile;
            const uint32_t t_row = tmem_base + ((quarter * 32u) << 16) + ab * BN;
            if (clustered) {
                // park the partial: part[tok][row] (pull) or slice-major (bulk), lanes =
                // consecutive rows (conflict-free); every MMA of this CTA has completed, so the
                // operand ring is free
                int sr = 0;
                while (bulk && sr + 1 < S_ && ro(sr + 1) <= static_cast<int>(row_in_tile)) ++sr;
                const int r0 = bulk ? ro(sr) : 0;
                const int stride = bulk ? ro(sr + 1) - r0 : BM;
                float* dst = part + (bulk ? Tp * r0 : 0) + (row_in_tile - r0);
                for (int c = 0; c < BN && c < p.tokens; c += 32) {
                    uint32_t r[32];
                    tmem_ld32(t_row + c, r);
                    tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (!bulk || c + j < Tp) dst[(c + j) * stride] = __uint_as_float(r[j]);
                }
                continue;
            }
            if (p.epi == EPI_QKV) {
                // normal path (prefill): thread = token m, columns = features; one head at a
                // time, rotate_half partners (j, j + hd/2) both come from this thread's TMEM lane
                const RopeEpi& R = p.rope;
                const int hd = R.hd, H = hd / 2, qd = R.hq * hd, kvd = R.hkv * hd;
                const bool tok_ok = m < p.tokens;
                const int sl = tok_ok ? R.slot[m] : 0;
                const int pos = tok_ok ? R.pos[m] : 0;
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += hd) {
                    const int f0 = tn * BN + c0;
                    const bool ok = tok_ok && f0 < p.n_out;
                    if (f0 >= qd + kvd) {
#pragma unroll 1
                        for (int c = 0; c < hd; c += 32) {
                            uint32_t r[32];
                            tmem_ld32(t_row + c0 + c, r);
                            tmem_ld_wait();
                            if (ok) {
                                float v[32];
#pragma unroll
                                for (int j = 0; j < 32; ++j)
                                    v[j] = __uint_as_float(r[j]) + (p.bias ? __bfloat162float(p.bias[f0 + c + j]) : 0.f);
                                store32_bf16(R.v_pool + pool_off(R, sl, (f0 - qd - kvd) / hd) + c, v);
                            }
                        }
                        continue;
                    }
                    __nv_bfloat16* dst = ok ? rot_dst(R, m, sl, f0 / hd) : nullptr;
#pragma unroll 1
                    for (int sub = 0; sub < H; sub += 32) {
                        uint32_t r1[32], r2[32];
                        tmem_ld32(t_row + c0 + sub, r1);
                        tmem_ld32(t_row + c0 + H + sub, r2);
                        tmem_ld_wait();
                        if (ok) {
                            // each thread reads its own position's cos/sin row: 128-bit loads
                            // (a warp-wide scalar load touches 32 rows = 32 L1 wavefronts; the
                            // per-element form kept the LSU pipe 51% busy, profiles/
                            // r2_ncu_prefill_qkv_epilogue.txt)
                            const float4* ct = reinterpret_cast<const float4*>(R.cos_t + (size_t)pos * H + sub);
                            const float4* st = reinterpret_cast<const float4*>(R.sin_t + (size_t)pos * H + sub);
                            float cs[32], sn[32];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 c4 = ct[q], s4 = st[q];
                                cs[4 * q] = c4.x, cs[4 * q + 1] = c4.y, cs[4 * q + 2] = c4.z, cs[4 * q + 3] = c4.w;
                                sn[4 * q] = s4.x, sn[4 * q + 1] = s4.y, sn[4 * q + 2] = s4.z, sn[4 * q + 3] = s4.w;
                            }
                            float y1[32], y2[32];
#pragma unroll
                            for (int j = 0; j < 32; ++j) {
                                float x1 = __uint_as_float(r1[j]), x2 = __uint_as_float(r2[j]);
                                if (p.bias) {
                                    x1 += __bfloat162float(p.bias[f0 + sub + j]);
                                    x2 += __bfloat162float(p.bias[f0 + H + sub + j]);
                                }
                                rope2(bf16r(x1), bf16r(x2), cs[j], sn[j], y1[j], y2[j]);
                            }
                            store32_bf16(dst + sub, y1);
                            store32_bf16(dst + H + sub, y2);
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(&tempty_bar[ab]);
                continue;
            }
#pragma unroll 1
            for (int c = 0; c < BN && (!p.swap || c < p.tokens) && !p.dbg_no_epi; c += 32) {
                uint32_t r[32];
                tmem_ld32(t_row + c, r);
                tmem_ld_wait();
                const int n0 = tn * BN + c;
                if (p.epi == EPI_SILU) {
                    // Interleaved gate/up rows: (2j, 2j+1) -> out column j.
                    if (!p.swap) {
                        if (m < p.tokens) {
                            __nv_bfloat16* o =
                                p.out + static_cast<size_t>(m) * p.ldo + (n0 >> 1);
                            if (n0 + 32 <= p.n_out && ((p.ldo & 7) == 0)) {
                                // 16 outputs = two 16-byte stores
                                uint32_t pk[8];
#pragma unroll
                                for (int j = 0; j < 8; ++j) {
                                    const float g0 = __uint_as_float(r[4 * j]), v0 = __uint_as_float(r[4 * j + 1]);
                                    const float g1 = __uint_as_float(r[4 * j + 2]), v1 = __uint_as_float(r[4 * j + 3]);
                                    pk[j] = pack_bf16(silu(g0) * v0, silu(g1) * v1);
                                }
                                uint4* o4 = reinterpret_cast<uint4*>(o);
                                o4[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                                o4[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                            } else {
#pragma unroll
                                for (int j = 0; j < 16; ++j) {
                                    const float g = __uint_as_float(r[2 * j]);
                                    const float v = __uint_as_float(r[2 * j + 1]);
                                    if (n0 + 2 * j + 1 < p.n_out)
                                        o[j] = __float2bfloat16_rn(silu(g) * v);
                                }
                            }
                        }
                    } else {
                        // weight rows are TMEM lanes: pair with the neighbouring lane.
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const float mine = __uint_as_float(r[j]);
                            const float other = __shfl_xor_sync(0xffffffffu, mine, 1);
                            const int tok = n0 + j;
                            if ((lane & 1) == 0 && tok < p.tokens && m + 1 < p.n_out) {
                                p.out[static_cast<size_t>(tok) * p.ldo + (m >> 1)] =
                                    __float2bfloat16_rn(silu(mine) * other);
                            }
                        }
                    }
                } else if (!p.swap) {
                    if (m < p.tokens) {
                        if (p.epi == EPI_BF16 || p.epi == EPI_RESID) {
                            // 32 contiguous outputs of one row: vectorised 16-byte stores.
                            const bool full = (n0 + 32 <= p.n_out) && ((p.ldo & 7) == 0);
                            if (full) {
                                float v[32];
#pragma unroll
                                for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
                                if (p.epi == EPI_BF16 && p.bias) {
#pragma unroll
                                    for (int j = 0; j < 32; ++j)
                                        v[j] += __bfloat162float(p.bias[n0 + j]);
                                }
                                if (p.epi == EPI_RESID) {
                                    const uint4* rp = reinterpret_cast<const uint4*>(
                                        p.resid + static_cast<size_t>(m) * p.ldr + n0);
#pragma unroll
                                    for (int q = 0; q < 4; ++q) {
                                        uint4 w = rp[q];
                                        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
                                        for (int e = 0; e < 4; ++e) {
                                            v[q * 8 + 2 * e] += bf16_lo(ww[e]);
                                            v[q * 8 + 2 * e + 1] += bf16_hi(ww[e]);
                                        }
                                    }
                                }
                                uint4* op = reinterpret_cast<uint4*>(
                                    p.out + static_cast<size_t>(m) * p.ldo + n0);
#pragma unroll
                                for (int q = 0; q < 4; ++q) {
                                    uint4 w;
                                    w.x = pack_bf16(v[q * 8 + 0], v[q * 8 + 1]);
                                    w.y = pack_bf16(v[q * 8 + 2], v[q * 8 + 3]);
                                    w.z = pack_bf16(v[q * 8 + 4], v[q * 8 + 5]);
                                    w.w = pack_bf16(v[q * 8 + 6], v[q * 8 + 7]);
                                    op[q] = w;
                                }
                            } else {
#pragma unroll
                                for (int j = 0; j < 32; ++j)
                                    epi.store(m, n0 + j, __uint_as_float(r[j]));
                            }
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j) epi.store(m, n0 + j, __uint_as_float(r[j]));
                        }
                    }
                } else {
                    // swap: D[m = weight row][n = token] -> Y[token][weight row].  Residual: all
                    // 32 loads first (the in-place store would otherwise serialise them)
                    if (p.epi == EPI_RESID) {
                        float rv[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            rv[j] = (n0 + j < p.tokens && m < p.n_out)
                                        ? __bfloat162float(p.resid[static_cast<size_t>(n0 + j) * p.ldr + m]) : 0.f;
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (n0 + j < p.tokens && m < p.n_out)
                                p.out[static_cast<size_t>(n0 + j) * p.ldo + m] =
                                    __float2bfloat16_rn(__uint_as_float(r[j]) + rv[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) epi.store(n0 + j, m, __uint_as_float(r[j]));
                    }
                    if (p.amax) {
                        // fused greedy sample: key[j] per lane, then a butterfly reduce-scatter
                        // leaves lane l with the max over the warp's 32 rows for token n0 + l
                        unsigned long long k[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            k[j] = m < p.n_out ? argmax_key(__uint_as_float(r[j]), m) : 0ull;
#pragma unroll
                        for (int o = 16; o >= 1; o >>= 1) {
                            const bool upper = (lane & o) != 0;
#pragma unroll
                            for (int i = 0; i < o; ++i) {
                                const unsigned long long send = upper ? k[i] : k[i + o];
                                const unsigned long long keep = upper ? k[i + o] : k[i];
                                const unsigned long long got = __shfl_xor_sync(0xffffffffu, send, o);
                                k[i] = keep > got ? keep : got;
                            }
                        }
                        if (n0 + static_cast<int>(lane) < p.tokens && k[0]) atomicMax(p.amax + n0 + lane, k[0]);
                    }
                }
            }

            tc_fence_before();
            mbar_arrive(&tempty_bar[ab]);
        }
    }

    if (threadIdx.x == 64) stamp(2);
    tc_fence_before();
    if (clustered && bulk) {
        Epi epi{p};
        const int rank = blockIdx.x % S_;
        const int tile = blockIdx.x / S_;
        const int r0 = ro(rank), nr = ro(rank + 1) - r0, nu = nr / 4;
        const uint32_t part_s = smem_u32(part);
        const uint32_t recv_s = part_s + BM * BN * 4;  // S slots of [Tp][nr] fp32
        const uint32_t slot_bytes = static_cast<uint32_t>(Tp * nr * 4);
        fence_proxy_async_smem();  // parked partial -> visible to the bulk-copy engine
        if (threadIdx.x == 0) mbar_expect_tx(recv_bar, (S_ - 1) * slot_bytes);
        cluster_sync();  // every CTA has parked its partial and armed its receive barrier
        if (threadIdx.x == 0) {
            stamp(7);
            for (int q = 0; q < S_; ++q) {
                if (q == rank) continue;
                const int q0 = ro(q);
                const uint32_t bytes = static_cast<uint32_t>(Tp * (ro(q + 1) - q0) * 4);
                bulk_s2cluster(mapa_shared(recv_s + rank * bytes, q), part_s + Tp * q0 * 4, bytes,
                               mapa_shared(smem_u32(recv_bar), q));
            }
        }
        const int n_el = Tp * nu;
        const int m_base = (tile % tiles_m) * BM + r0;
        const bool vec_r = (p.ldr & 3) == 0, vec_o = (p.ldo & 3) == 0;
        constexpr int CH = 4;
        for (int e0 = threadIdx.x, round = 0; round == 0 || e0 < n_el; e0 += kThreads * CH, ++round) {
            // residual rows first: their HBM/L2 latency overlaps the incoming copies
            float rr[CH][4];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int e = e0 + c * kThreads;
                rr[c][0] = rr[c][1] = rr[c][2] = rr[c][3] = 0.f;
                if (p.epi != EPI_RESID || e >= n_el) continue;
                const int tok = e / nu, m = m_base + 4 * (e % nu);
                const __nv_bfloat16* rp = p.resid + static_cast<size_t>(tok) * p.ldr + m;
                if (vec_r && m + 3 < p.n_out) {
                    const uint2 w = *reinterpret_cast<const uint2*>(rp);
                    rr[c][0] = bf16_lo(w.x), rr[c][1] = bf16_hi(w.x), rr[c][2] = bf16_lo(w.y), rr[c][3] = bf16_hi(w.y);
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (m + k < p.n_out) rr[c][k] = __bfloat162float(rp[k]);
                }
            }
            if (round == 0) {
                mbar_wait(recv_bar, 0);
                cluster_arrive();  // all our incoming copies landed: peers may exit after this
            }
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int e = e0 + c * kThreads;
                if (e >= n_el) continue;
                const int tok = e / nu, u = e % nu;
                const uint32_t off = static_cast<uint32_t>((tok * nr + 4 * u) * 4);
                float4 v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < S_) v[q] = lds128f(q == rank ? part_s + Tp * r0 * 4 + off : recv_s + q * slot_bytes + off);
                float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < S_) {
                        a0 += v[q].x;
                        a1 += v[q].y;
                        a2 += v[q].z;
                        a3 += v[q].w;
                    }
                const int m = m_base + 4 * u;
                if (p.epi == EPI_RESID) {
                    const float y[4] = {a0 + rr[c][0], a1 + rr[c][1], a2 + rr[c][2], a3 + rr[c][3]};
                    __nv_bfloat16* op = p.out + static_cast<size_t>(tok) * p.ldo + m;
                    if (vec_o && m + 3 < p.n_out) {
                        *reinterpret_cast<uint2*>(op) = make_uint2(pack_bf16(y[0], y[1]), pack_bf16(y[2], y[3]));
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (m + k < p.n_out) op[k] = __float2bfloat16_rn(y[k]);
                    }
                } else {
                    epi.store_pair(tok, m, a0, a1);
                    epi.store_pair(tok, m + 2, a2, a3);
                }
                if (p.amax) {
                    const float a[4] = {a0, a1, a2, a3};
                    unsigned long long k = 0ull;
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (m + i < p.n_out) k = max(k, argmax_key(a[i], m + i));
                    if (k) atomicMax(p.amax + tok, k);
                }
            }
        }
        cluster_wait();  // every CTA has received: no copy still reads our partial
    } else if (clustered) {
        // Reduce the tile over the cluster: CTA `rank` finishes row pairs
        // [64*rank/S, 64*(rank+1)/S), summing the S partials in rank order.
        cluster_sync();
        if (threadIdx.x == 0) stamp(7);
        const int S = p.splits > 1 ? p.splits : 1;
        const int rank = blockIdx.x % S;
        const int tile = blockIdx.x / S;
        const uint32_t base = smem_u32(part);
        auto sum2 = [&](int tok, int row) {  // all S loads in flight, then the sum in rank order
            const uint32_t off = base + static_cast<uint32_t>((tok * BM + row) * 4);
            float2 v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < S) v[q] = ld_dsmem_f2(mapa_shared(off, q));
            float2 acc = make_float2(0.f, 0.f);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < S) {
                    acc.x += v[q].x;
                    acc.y += v[q].y;
                }
            return acc;
        };
        if (p.epi == EPI_QKV) {
            const RopeEpi& R = p.rope;
            const int hd = R.hd, H = hd / 2, qd = R.hq * hd, kvd = R.hkv * hd;
            const int f0 = (tile % tiles_m) * BM;
            const bool vt = f0 >= qd + kvd;
            const int per_tok = vt ? 64 : 32;  // V: row pairs; q/k: (j, j+1) x (lo, hi half) quads
            const int n = p.tokens * per_tok;
            const int lo = static_cast<int>((static_cast<long long>(n) * rank) / S);
            const int hi = static_cast<int>((static_cast<long long>(n) * (rank + 1)) / S);
            for (int e = lo + threadIdx.x; e < hi; e += kThreads) {
                const int tok = e / per_tok, i = e % per_tok;
                const int sl = R.slot[tok];
                if (vt) {
                    const int mrow = 2 * i, f = f0 + mrow;
                    if (f >= p.n_out) continue;
                    float2 a = sum2(tok, mrow);
                    if (p.bias) {
                        a.x += __bfloat162float(p.bias[f]);
                        a.y += __bfloat162float(p.bias[f + 1]);
                    }
                    const int fv = f - qd - kvd;
                    *reinterpret_cast<uint32_t*>(R.v_pool + pool_off(R, sl, fv / hd) + fv % hd) = pack_bf16(a.x, a.y);
                } else {
                    const int hl = i / (H / 2), j = 2 * (i % (H / 2));
                    const int m1 = hl * hd + j, f1 = f0 + m1;
                    if (f1 >= p.n_out) continue;
                    float2 a = sum2(tok, m1), b = sum2(tok, m1 + H);
                    if (p.bias) {
                        a.x += __bfloat162float(p.bias[f1]);
                        a.y += __bfloat162float(p.bias[f1 + 1]);
                        b.x += __bfloat162float(p.bias[f1 + H]);
                        b.y += __bfloat162float(p.bias[f1 + H + 1]);
                    }
                    const int pos = R.pos[tok];
                    const float* ct = R.cos_t + (size_t)pos * H + j;
                    const float* st = R.sin_t + (size_t)pos * H + j;
                    float y1a, y2a, y1b, y2b;
                    rope2(bf16r(a.x), bf16r(b.x), ct[0], st[0], y1a, y2a);
                    rope2(bf16r(a.y), bf16r(b.y), ct[1], st[1], y1b, y2b);
                    __nv_bfloat16* dst = rot_dst(R, tok, sl, (f0 + hl * hd) / hd);
                    *reinterpret_cast<uint32_t*>(dst + j) = pack_bf16(y1a, y1b);
                    *reinterpret_cast<uint32_t*>(dst + j + H) = pack_bf16(y2a, y2b);
                }
            }
            cluster_sync();
            if (threadIdx.x == 0) stamp(3);
            if (warp == 1) {
                tc_fence_after();
                tmem_dealloc<C::kTmemCols>(tmem_base);
            }
            return;
        }
        const int p0 = (64 * rank) / S, p1 = (64 * (rank + 1)) / S, np = p1 - p0;
        Epi epi{p};
        // CH elements per thread per round: every DSMEM partial and residual load of the round
        // is issued before the first sum (a per-element load -> add -> store chain would
        // serialise ~S+1 round trips per element, and the in-place residual store keeps the
        // compiler from hoisting the next residual load)
        constexpr int CH = 4;
        for (int e0 = threadIdx.x; e0 < np * p.tokens; e0 += kThreads * CH) {
            float2 v[CH][8];
            float2 rr[CH];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int e = e0 + c * kThreads;
                rr[c] = make_float2(0.f, 0.f);
                if (e >= np * p.tokens) continue;
                const int tok = e / np, row = 2 * (p0 + e % np);
                const uint32_t off = base + static_cast<uint32_t>((tok * BM + row) * 4);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < S) v[c][q] = ld_dsmem_f2(mapa_shared(off, q));
                const int m = (tile % tiles_m) * BM + row;
                if (p.epi == EPI_RESID && m < p.n_out) {
                    const __nv_bfloat16* rp = p.resid + static_cast<size_t>(tok) * p.ldr + m;
                    if (m + 1 < p.n_out && (p.ldr & 1) == 0) {
                        const uint32_t w2 = *reinterpret_cast<const uint32_t*>(rp);
                        rr[c] = make_float2(bf16_lo(w2), bf16_hi(w2));
                    } else {
                        rr[c] = make_float2(__bfloat162float(rp[0]), m + 1 < p.n_out ? __bfloat162float(rp[1]) : 0.f);
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int e = e0 + c * kThreads;
                if (e >= np * p.tokens) continue;
                const int tok = e / np, row = 2 * (p0 + e % np);
                float2 acc = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < S) {
                        acc.x += v[c][q].x;
                        acc.y += v[c][q].y;
                    }
                const int m = (tile % tiles_m) * BM + row;
                if (p.epi == EPI_RESID) {
                    if (tok < p.tokens && m < p.n_out) {
                        const size_t o = static_cast<size_t>(tok) * p.ldo + m;
                        const float y0 = acc.x + rr[c].x, y1 = acc.y + rr[c].y;
                        if (m + 1 < p.n_out && (p.ldo & 1) == 0) {
                            *reinterpret_cast<uint32_t*>(p.out + o) = pack_bf16(y0, y1);
                        } else {
                            p.out[o] = __float2bfloat16_rn(y0);
                            if (m + 1 < p.n_out) p.out[o + 1] = __float2bfloat16_rn(y1);
                        }
                    }
                } else {
                    epi.store_pair(tok, m, acc.x, acc.y);
                }
                if (p.amax && m < p.n_out) {
                    unsigned long long k = argmax_key(acc.x, m);
                    if (m + 1 < p.n_out) k = max(k, argmax_key(acc.y, m + 1));
                    if (k) atomicMax(p.amax + tok, k);
                }
            }
        }
        cluster_sync();  // peers may still be reading our partial
    } else {
        __syncthreads();
    }
    if (threadIdx.x == 0) stamp(3);
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem_base);
    }
    // fused next pre-norm (decode steps): the last CTA normalises the updated residual rows
    if (p.post.w && grid_last_arriver(p.post.counter)) post_norm_rows(p.post, p.out, p.ldo);
}

// Occupancy of S-CTA clusters of this kernel (cached per configuration).
template <int BN, int KP>
cudaError_t set_smem_attr();

template <int BN, int KP = 1>
int max_active_clusters(int S, cudaStream_t stream) {
    if (set_smem_attr<BN, KP>() != cudaSuccess) return 0;
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find({S, stream});
    if (it != cache.end()) return it->second;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(S * 64, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = GemmCfg<BN, KP>::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = S;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_tn_kernel<BN, KP>, &cfg) != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    cache[{S, stream}] = n;
    return n;
}

template <int BN, int KP>
cudaError_t set_smem_attr() {
    static bool attr_set = false;  // per-process; harmless race (idempotent)
    if (attr_set) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(gemm_tn_kernel<BN, KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         GemmCfg<BN, KP>::kSmemBytes);
    if (e == cudaSuccess) attr_set = true;
    return e;
}

template <int BN, int KP = 1>
cudaError_t launch_bn(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                      int num_sms, cudaStream_t stream, bool pdl) {
    using C = GemmCfg<BN, KP>;
    cudaError_t e = set_smem_attr<BN, KP>();
    if (e != cudaSuccess) return e;
    const int tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
    const bool staged = p.swap && (p.splits > 1 || p.epi == EPI_QKV);
    const bool clustered = p.swap && p.splits > 1;
    const int grid = staged ? tiles * std::max(1, p.splits) : std::min(tiles, num_sms);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = C::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (clustered) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = p.splits;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    const bool use_pdl = pdl_for_launch(clustered) && pdl;  // launch.cuh: no PDL right after a cluster launch
    if (use_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, gemm_tn_kernel<BN, KP>, ta, tb, p);
}

}  // namespace

int gemm_pick_bn(int n) {
    if (n <= 32) return 32;
    if (n <= 64) return 64;
    if (n <= 128) return 128;
    return 256;
}

int gemm_cluster_splits(int tiles, int k_blocks, int bn, int num_sms, cudaStream_t stream, int force, int kp) {
    // k_blocks: pipeline k-units of kp 64-wide blocks
    auto fits = [&](int S) {
        if (S < 2) return true;
        const int kbps = (k_blocks + S - 1) / S;
        if ((S - 1) * kbps >= k_blocks) return false;  // an empty split
        int act = 0;
        switch (bn * 4 + kp) {
        case 32 * 4 + 1: act = max_active_clusters<32, 1>(S, stream); break;
        case 32 * 4 + 2: act = max_active_clusters<32, 2>(S, stream); break;
        case 64 * 4 + 1: act = max_active_clusters<64, 1>(S, stream); break;
        case 64 * 4 + 2: act = max_active_clusters<64, 2>(S, stream); break;
        case 128 * 4 + 1: act = max_active_clusters<128, 1>(S, stream); break;
        default: act = max_active_clusters<256, 1>(S, stream); break;
        }
        return act >= tiles && tiles * S <= num_sms;
    };
    if (force > 0) {
        int S = std::min(force, 8);
        while (S > 1 && (S - 1) * ((k_blocks + S - 1) / S) >= k_blocks) --S;
        return S;
    }
    if (tiles >= num_sms) return 1;
    int S = std::min({8, num_sms / tiles, k_blocks});
    while (S > 1 && !fits(S)) --S;
    return std::max(S, 1);
}

cudaError_t gemm_launch(const CUtensorMap& ta, const CUtensorMap& tb, GemmParams p, int bn,
                        int num_sms, cudaStream_t stream, bool pdl, int kp) {
    if (kp != 1 && !(kp == 2 && p.swap && bn <= 64)) return cudaErrorInvalidValue;
    const int k_units = ((p.K + BK - 1) / BK + kp - 1) / kp;
    if (!p.swap || p.splits <= 1) {
        p.splits = 1;
        p.kb_per_split = k_units;
    } else {
        p.kb_per_split = (k_units + p.splits - 1) / p.splits;
    }
    switch (bn * 4 + kp) {
    case 32 * 4 + 1: return launch_bn<32, 1>(ta, tb, p, num_sms, stream, pdl);
    case 32 * 4 + 2: return launch_bn<32, 2>(ta, tb, p, num_sms, stream, pdl);
    case 64 * 4 + 1: return launch_bn<64, 1>(ta, tb, p, num_sms, stream, pdl);
    case 64 * 4 + 2: return launch_bn<64, 2>(ta, tb, p, num_sms, stream, pdl);
    case 128 * 4 + 1: return launch_bn<128, 1>(ta, tb, p, num_sms, stream, pdl);
    case 256 * 4 + 1: return launch_bn<256, 1>(ta, tb, p, num_sms, stream, pdl);
    default: return cudaErrorInvalidValue;
    }
}

int gemm_smem_bytes(int bn) {
    switch (bn) {
    case 32: return GemmCfg<32>::kSmemBytes;
    case 64: return GemmCfg<64>::kSmemBytes;
    case 128: return GemmCfg<128>::kSmemBytes;
    default: return GemmCfg<256>::kSmemBytes;
    }
}

}  // namespace asb
