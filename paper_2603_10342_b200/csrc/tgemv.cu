// Decode linear layer on a TMA-fed smem ring ("tgemv"): Y[tok][n] = sum_k X[tok][k] * W[n][k]
// for T <= 32 tokens, the weight-streaming regime of every decode step (B rows + an admitted
// resume chunk).  Replaces, with decode_attention, the mu_D term of the reference's
// decode_step_duration_ms (/root/reference/proj/src/executor.cpp:84-97).
//
// Why a third decode-linear kernel.  On a Green Context partition of 16-64 SMs a decode step
// is bound by how fast each SM can pull bytes, not by HBM: the per-SM TMA stream reaches
// ~160-175 GB/s with 32 KiB requests and ~200 KiB in flight (profiles/r2_tma_pair_probe.txt,
// the activation box riding along costs nothing), but
//   * the tcgen05 swap-AB kernel (gemm.cu) sustains ~80 GB/s/SM: each 128x32 UMMA of a stage
//     holds the stage ~2x longer than its bytes take to arrive (tensor pipe 46% busy at 2.4
//     TB/s, profiles/r2_ncu_gemm_gate_up_l2.txt), so the ring turnaround, not the stream,
//     sets the rate;
//   * dgemv (register ring, ld.global) keeps only 4-8 KiB per warp in flight: 40-60 GB/s/SM.
// Here the weight stream is one 32 KiB TMA box (128 rows x 2 k-blocks of the tile-packed
// layout) + one 8 KiB activation box per stage into a 5-stage ring (200 KiB in flight), and
// 8 consumer warps (2 row groups x 4 k groups) run legacy warp MMAs (m16n8k16, rows = weight
// rows, n = tokens) on ldmatrix fragments -- ~2 cycles per MMA per SM (scripts/probes/hmma.cu),
// i.e. at <= 16 tokens a stage's math and smem traffic take less than its bytes' arrival time.
//
// Work = (128-row tile, K split) units; the split factor S makes tiles*S fill the SMs of the
// partition in whole waves.  Split partials go to a workspace and the last-arriving split of
// a tile sums them in split order (deterministic) and runs the epilogue: +bias, +residual
// (in place) with the fused next pre-norm, SiLU(gate)*up, fp32 logits + greedy-argmax key, or
// the QKV bias + RoPE + paged K/V append (a 128-row tile holds whole heads, so every
// rotate_half pair is inside the tile).  Same rounding points as the other GEMM epilogues.
#include <cuda_runtime.h>

#include <algorithm>

#include "epi.cuh"
#include "gemm.h"
#include "launch.cuh"
#include "sm100.cuh"
#include "warpmma.cuh"

namespace asb {

namespace {

constexpr int kTgW = 128 * 128 * 2;  // 128 weight rows x 2 k-blocks
constexpr int kTgRS = 33;            // red row stride (floats)

// <= 16 tokens: 16-row activation boxes, 6 stages (216 KiB); <= 32: 32 rows, 5 stages.  The
// stage a unit ends on is released only after the unit's reduction + epilogue, which use it as
// scratch (red), so the other stages keep streaming the next unit meanwhile.
template <int NT>
struct TgCfg {
    // consumer warps = RG row groups x 4 k groups: 8 warps (64 rows each) up to 16 tokens, 16
    // warps (32 rows each) above, where the 4 n-tiles of MMAs per fragment need more warps in
    // flight to keep the MMA pipe fed
    static constexpr int kRG = NT <= 2 ? 2 : 4;
    static constexpr int kWarps = 4 * kRG;
    static constexpr int kThreads = (kWarps + 1) * 32;
    static constexpr int kMT = 8 / kRG;  // 16-row m-tiles per warp
    static constexpr int kXRows = NT <= 2 ? 16 : 32;
    static constexpr int kX = kXRows * 128 * 2;
    static constexpr int kStage = kTgW + kX;
    static constexpr int kStages = NT <= 2 ? 6 : 5;
    static constexpr int kSmem = kStages * kStage + 2 * kStages * 8 + 32 * 8 + 1024;
    static_assert(128 * kTgRS * 4 <= kStage, "red must fit one stage");
};

template <int NT>
__global__ void __launch_bounds__(TgCfg<NT>::kThreads, 1)
    tgemv_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_x,
                 const TgemvParams p) {
    using C = TgCfg<NT>;
    constexpr int kTgStages = C::kStages, kTgStage = C::kStage, kTgX = C::kX;
    constexpr int kTgWarps = C::kWarps, MTW = C::kMT, RG = C::kRG;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
    uint8_t* ring = smem;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + kTgStages * kTgStage);
    uint64_t* empty = full + kTgStages;
    unsigned long long* key_s = reinterpret_cast<unsigned long long*>(empty + kTgStages);  // [32]
    __shared__ int s_last;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int S = p.splits, units = p.tiles * S;
    if (threadIdx.x == 0) {
        tma_prefetch_desc(&tmap_w);
        tma_prefetch_desc(&tmap_x);
        for (int i = 0; i < kTgStages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kTgWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();
    pdl_trigger();

    if (warp == kTgWarps) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
            // weights do not depend on the previous kernel: fill the ring with the first
            // unit's weight boxes, then wait for the activations
            int pre = 0;
            if (static_cast<int>(blockIdx.x) < units) {
                const int u = blockIdx.x, tile = u / S, k0 = (u % S) * p.kups;
                const int k1 = min(p.kunits, k0 + p.kups);
                for (int ku = k0; ku < k1 && pre < kTgStages; ++ku, ++pre) {
                    mbar_expect_tx(&full[pre], kTgStage);
                    tma_load_4d_hint(ring + pre * kTgStage, &tmap_w, &full[pre], 0, 0, 2 * ku, tile, pol_w);
                }
            }
            pdl_wait();
            int i = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const int tile = u / S, k0 = (u % S) * p.kups, k1 = min(p.kunits, k0 + p.kups);
                for (int ku = k0; ku < k1; ++ku, ++i) {
                    const int st = i % kTgStages;
                    uint8_t* d = ring + st * kTgStage;
                    if (i >= pre) {
                        mbar_wait(&empty[st], ((i / kTgStages) & 1) ^ 1);
                        mbar_expect_tx(&full[st], kTgStage);
                        tma_load_4d_hint(d, &tmap_w, &full[st], 0, 0, 2 * ku, tile, pol_w);
                    }
                    tma_load_3d_hint(d + kTgW, &tmap_x, &full[st], 0, 0, 2 * ku, pol_x);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ consumers
        // 8 warps = 2 row groups (64 weight rows, 4 m-tiles) x 4 k groups (k16 steps kg and
        // kg + 4 of each 128-k stage).  Every W byte is read from smem once and each X
        // fragment twice (ldmatrix traffic per 32 KiB stage: 32 KiB + 2 x X), so neither the
        // shared-memory pipe nor the MMA pipe (128 m16n8k16 per stage at 16 tokens) holds a
        // stage longer than its bytes take to arrive.
        pdl_wait();  // residual / output buffers belong to the previous kernels
        const int tid = threadIdx.x;  // 0..255
        const int g = lane >> 2, t = lane & 3, mi = lane >> 3;
        const int rg = warp % RG, kg = warp / RG;
        const int T = p.T;
        int i = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const int tile = u / S, k0 = (u % S) * p.kups, k1 = min(p.kunits, k0 + p.kups);
            float acc[MTW][NT][4];
#pragma unroll
            for (int m = 0; m < MTW; ++m)
#pragma unroll
                for (int j = 0; j < NT; ++j) acc[m][j][0] = acc[m][j][1] = acc[m][j][2] = acc[m][j][3] = 0.f;
            for (int ku = k0; ku < k1; ++ku, ++i) {
                const int st = i % kTgStages;
                mbar_wait(&full[st], (i / kTgStages) & 1);
                const uint32_t wst = smem_u32(ring + st * kTgStage), xst = wst + kTgW;
#pragma unroll
                for (int ss = 0; ss < (p.dbg_load_only ? 0 : 2); ++ss) {
                    const int s = kg + 4 * ss;  // k16 step: k-block s / 4, 16-byte chunk pair 2(s % 4)
                    const int kb = s >> 2, cp = 2 * (s & 3);
                    uint32_t b[(NT + 1) / 2][4];
#pragma unroll
                    for (int jp = 0; jp < (NT + 1) / 2; ++jp) {
                        const int tok = 8 * (2 * jp + (mi >> 1)) + (lane & 7), ch = cp + (mi & 1);
                        ldsm_x4(xst + (kb * C::kXRows + tok) * 128 + ((ch ^ (tok & 7)) << 4), b[jp][0], b[jp][1],
                                b[jp][2], b[jp][3]);
                    }
#pragma unroll
                    for (int m = 0; m < MTW; ++m) {
                        const int row = rg * (128 / RG) + m * 16 + (mi & 1) * 8 + (lane & 7), ch = cp + (mi >> 1);
                        uint32_t a0, a1, a2, a3;
                        ldsm_x4(wst + (kb * 128 + row) * 128 + ((ch ^ (row & 7)) << 4), a0, a1, a2, a3);
#pragma unroll
                        for (int j = 0; j < NT; ++j)
                            mma16816(acc[m][j], a0, a1, a2, a3, b[j >> 1][2 * (j & 1)], b[j >> 1][2 * (j & 1) + 1]);
                    }
                }
                __syncwarp();
                if (lane == 0 && ku + 1 < k1) mbar_arrive(&empty[st]);
            }
            // the unit's last stage stays held: after every warp is done with its operands it
            // is the reduction scratch red [128 rows][kTgRS], released after the epilogue
            const int st_last = (i - 1) % kTgStages;
            float* red = reinterpret_cast<float*>(ring + st_last * kTgStage);
            named_sync(1, kTgWarps * 32);
            // ---- k-group partials -> red, summed in k-group order (deterministic)
#pragma unroll 1
            for (int r = 0; r < 4; ++r) {
                if (kg == r) {
#pragma unroll
                    for (int m = 0; m < MTW; ++m) {
                        const int rl = rg * (128 / RG) + m * 16 + g;
#pragma unroll
                        for (int j = 0; j < NT; ++j) {
                            const int tk = 8 * j + 2 * t;
                            float* r0 = red + rl * kTgRS + tk;
                            float* r8 = red + (rl + 8) * kTgRS + tk;
                            if (r == 0) {
                                r0[0] = acc[m][j][0];
                                r0[1] = acc[m][j][1];
                                r8[0] = acc[m][j][2];
                                r8[1] = acc[m][j][3];
                            } else {
                                r0[0] += acc[m][j][0];
                                r0[1] += acc[m][j][1];
                                r8[0] += acc[m][j][2];
                                r8[1] += acc[m][j][3];
                            }
                        }
                    }
                }
                named_sync(1, kTgWarps * 32);
            }
            if (S > 1) {
                // split partial -> workspace [tok][row]; the last-arriving split of the tile sums
                // all S in split order (every load in flight at once) and runs the epilogue
                float* w = p.ws + (size_t)u * (32 * 128);
                for (int e = tid; e < 128 * T; e += kTgWarps * 32) {
                    const int rl = e & 127, tok = e >> 7;
                    w[tok * 128 + rl] = red[rl * kTgRS + tok];
                }
                __threadfence();
                named_sync(1, kTgWarps * 32);
                if (tid == 0) {
                    const int prev = atomicAdd(p.cnt + tile, 1);
                    s_last = prev == S - 1;
                    if (s_last) p.cnt[tile] = 0;  // re-arm for the next launch
                }
                named_sync(1, kTgWarps * 32);
                if (!s_last) {
                    fence_proxy_async_smem();  // generic writes (red) before the next TMA into the stage
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[st_last]);
                    continue;
                }
                __threadfence();
                const float* w0 = p.ws + (size_t)tile * S * (32 * 128);
                for (int e = tid; e < 128 * T; e += kTgWarps * 32) {
                    const int rl = e & 127, tok = e >> 7;
                    float pv[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) pv[q] = q < S ? __ldcg(w0 + (size_t)q * (32 * 128) + tok * 128 + rl) : 0.f;
                    float v = 0.f;
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        if (q < S) v += pv[q];
                    red[rl * kTgRS + tok] = v;
                }
                named_sync(1, kTgWarps * 32);
            }
            // ---- epilogue of the tile (rows n = tile * 128 + rl, tokens < T)
            const int nb = tile * 128;
            switch (p.epi) {
            case EPI_SILU: {  // interleaved gate/up rows (2j, 2j+1) -> output column j
                for (int e = tid; e < 64 * T; e += kTgWarps * 32) {
                    const int pr = e & 63, tok = e >> 6, n = nb + 2 * pr;
                    if (n + 1 >= p.n_out) continue;
                    p.out[(size_t)tok * p.ldo + (n >> 1)] =
                        __float2bfloat16_rn(silu(red[2 * pr * kTgRS + tok]) * red[(2 * pr + 1) * kTgRS + tok]);
                }
                break;
            }
            case EPI_QKV: {
                const RopeEpi& Rp = p.rope;
                const int hd = Rp.hd, H = hd / 2, qd = Rp.hq * hd, kvd = Rp.hkv * hd;
                for (int e = tid; e < 64 * T; e += kTgWarps * 32) {
                    const int pi = e & 63, tok = e >> 6;
                    const int hl = pi / H, j = pi % H;  // head within the tile, pair index
                    const int f0 = nb + hl * hd;
                    if (f0 >= p.n_out) continue;
                    const int rl = hl * hd + j;
                    float x1 = red[rl * kTgRS + tok], x2 = red[(rl + H) * kTgRS + tok];
                    if (p.bias) {
                        x1 += __bfloat162float(p.bias[f0 + j]);
                        x2 += __bfloat162float(p.bias[f0 + j + H]);
                    }
                    const int sl = Rp.slot[tok];
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
                const bool amax = p.epi == EPI_F32 && p.amax;
                if (amax && tid < 32) key_s[tid] = 0ull;
                if (amax) named_sync(1, kTgWarps * 32);
                for (int e = tid; e < 128 * T; e += kTgWarps * 32) {
                    const int rl = e & 127, tok = e >> 7, n = nb + rl;
                    if (n >= p.n_out) continue;
                    float v = red[rl * kTgRS + tok];
                    const size_t o = (size_t)tok * p.ldo + n;
                    if (p.epi == EPI_F32) {
                        p.out_f32[o] = v;
                        if (amax) {
                            const unsigned long long k = argmax_key(v, n);
                            if (k) atomicMax(&key_s[tok], k);
                        }
                    } else {
                        if (p.epi == EPI_RESID) v += __bfloat162float(p.resid[(size_t)tok * p.ldr + n]);
                        else if (p.bias) v += __bfloat162float(p.bias[n]);
                        p.out[o] = __float2bfloat16_rn(v);
                    }
                }
                if (amax) {
                    named_sync(1, kTgWarps * 32);
                    if (tid < T && key_s[tid]) atomicMax(p.amax + tid, key_s[tid]);
                }
                break;
            }
            }
            named_sync(1, kTgWarps * 32);  // every warp is done with red: release the stage
            fence_proxy_async_smem();       // order red's generic writes before the next TMA write
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st_last]);
        }
    }
    // fused next pre-norm (decode steps): the last CTA normalises the updated residual rows
    if (p.post.w && grid_last_arriver(p.post.counter)) post_norm_rows(p.post, p.out, p.ldo);
}

template <int NT>
cudaError_t launch_nt(const CUtensorMap& tw, const CUtensorMap& tx, const TgemvParams& p, int grid,
                      cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(tgemv_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, TgCfg<NT>::kSmem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    return launch_k(tgemv_kernel<NT>, dim3(grid), dim3(TgCfg<NT>::kThreads), TgCfg<NT>::kSmem, st, tw, tx, p);
}

}  // namespace

int tgemv_max_tokens() { return 32; }

int tgemv_splits(int tiles, int kunits, int num_sms) {
    // K split minimising the makespan in waves of one CTA per SM, in stage units plus a fixed
    // cost per unit (ring fill + epilogue: ~2 stages; a split unit adds its workspace write,
    // fence and arrival atomic: ~6), units <= 4 waves (the workspace bound)
    int best = 1;
    long best_t = -1;
    for (int s = 1; s <= 8; ++s) {
        if (s > 1 && (kunits + s - 1) / s < 2) break;
        if (s > 1 && tiles * s > 4 * num_sms) break;
        const long waves = (long(tiles) * s + num_sms - 1) / num_sms;
        const long t = waves * ((kunits + s - 1) / s + (s > 1 ? 6 : 2));
        if (best_t < 0 || t < best_t) {
            best_t = t;
            best = s;
        }
    }
    return best;
}

cudaError_t tgemv_launch(const CUtensorMap& tmap_w, const CUtensorMap& tmap_x, TgemvParams p, int num_sms,
                         cudaStream_t stream) {
    if (p.T < 1 || p.T > 32 || p.K % 64 != 0) return cudaErrorInvalidValue;
    if (p.epi == EPI_QKV && (128 % p.rope.hd != 0)) return cudaErrorInvalidValue;
    p.kunits = (p.K / 64 + 1) / 2;
    if (p.splits < 1) p.splits = tgemv_splits(p.tiles, p.kunits, num_sms);
    p.kups = (p.kunits + p.splits - 1) / p.splits;
    p.splits = (p.kunits + p.kups - 1) / p.kups;  // no empty split
    if (p.splits > 1 && (!p.ws || !p.cnt)) return cudaErrorInvalidValue;
    const int grid = std::min(p.tiles * p.splits, std::max(1, num_sms));
    switch ((p.T + 7) / 8) {
    case 1: return launch_nt<1>(tmap_w, tmap_x, p, grid, stream);
    case 2: return launch_nt<2>(tmap_w, tmap_x, p, grid, stream);
    case 3: return launch_nt<3>(tmap_w, tmap_x, p, grid, stream);
    default: return launch_nt<4>(tmap_w, tmap_x, p, grid, stream);
    }
}

}  // namespace asb
