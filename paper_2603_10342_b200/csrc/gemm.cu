// tcgen05 GEMM for the SLM linear layers (K5 in SURVEY §2.3):
//   Y[tok][n] = sum_k X[tok][k] * W[n][k]   (+ bias / + residual / SiLU·mul / fp32)
//
// Replaces the simulated cost terms of the reference's executor
// (decode_step_duration_ms, /root/reference/proj/src/executor.cpp:207-220, and the
// prefill rate x length arithmetic, /root/reference/proj/src/engine.cpp:450-475).
//
// Structure (one CTA per SM, persistent over work units):
//   warp 0      : TMA producer   (A/B tiles -> smem ring, SWIZZLE_128B, mbarrier tx)
//   warp 1      : MMA issuer     (one elected lane, tcgen05.mma kind::f16, commit)
//   warps 2..5  : epilogue       (tcgen05.ld TMEM -> regs -> fused epilogue -> HBM)
// TMEM holds two BN-column fp32 accumulators so the epilogue of unit i overlaps the
// MMAs of unit i+1.
//
// Two operand orders:
//   normal (prefill, many tokens):  A = X (tokens, M = 128 rows/tile), B = W (BN = 256)
//   swap   (decode, <= 256 tokens): A = W (128 weight rows/tile),       B = X (BN = tokens)
//     plus split-K across CTAs (fp32 atomics into a workspace, finalised by
//     gemm_finalize_kernel) so a 9-tile projection still streams weights on all SMs.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "gemm.h"
#include "sm100.cuh"

namespace asb {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kThreads = 192;

template <int BN>
struct GemmCfg {
    static constexpr int kStages = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
    static constexpr int kBytesA = BM * BK * 2;
    static constexpr int kBytesB = BN * BK * 2;
    static constexpr int kStageBytes = kBytesA + kBytesB;
    static constexpr int kTmemCols = (2 * BN) <= 32 ? 32 : 2 * BN;  // power of two >= 32
    static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

__device__ __forceinline__ float silu(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

// Apply the epilogue to one output value pair-free path (all modes except SiLU).
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
        case EPI_ATOMIC:
            atomicAdd(p.ws + static_cast<size_t>(tok) * p.n_out + n, v);
            break;
        default:
            break;
        }
    }
};

// Work decomposition shared by the producer, MMA and epilogue roles.
//  classic : units (tile, split) strided over the persistent grid
//  stream-K: CTA b owns the contiguous range [b*W/grid, (b+1)*W/grid) of the flattened
//            (tile, k-block) space (W = tiles * k_blocks), so every CTA streams the same
//            number of k-blocks; tile boundaries inside a range flush through fp32 atomics.
struct Work {
    int tiles_m, k_blocks, units, splits, kbps, streamk, u;
    long long pos, hi;
    __device__ void init(const GemmParams& p, int tm_, int tn_, int kb) {
        tiles_m = tm_;
        k_blocks = kb;
        splits = p.splits;
        kbps = p.kb_per_split;
        streamk = p.streamk;
        units = tm_ * tn_ * p.splits;
        u = blockIdx.x;
        const long long total = static_cast<long long>(tm_) * tn_ * kb;
        pos = total * blockIdx.x / gridDim.x;
        hi = total * (blockIdx.x + 1) / gridDim.x;
    }
    __device__ bool next(int& tm, int& tn, int& kb0, int& kb1) {
        int tile;
        if (streamk) {
            if (pos >= hi) return false;
            tile = static_cast<int>(pos / k_blocks);
            kb0 = static_cast<int>(pos % k_blocks);
            kb1 = static_cast<int>(min(static_cast<long long>(k_blocks), kb0 + (hi - pos)));
            pos += kb1 - kb0;
        } else {
            if (u >= units) return false;
            const int split = u % splits;
            tile = u / splits;
            kb0 = split * kbps;
            kb1 = min(k_blocks, kb0 + kbps);
            u += gridDim.x;
        }
        tm = tile % tiles_m;
        tn = tile / tiles_m;
        return true;
    }
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmap_a,
                   const __grid_constant__ CUtensorMap tmap_b, const GemmParams p) {
    using C = GemmCfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
    uint8_t* smem_a = smem;
    uint8_t* smem_b = smem + C::kStages * C::kBytesA;
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
    uint64_t* empty_bar = full_bar + C::kStages;
    uint64_t* tfull_bar = empty_bar + C::kStages;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();

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
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc<C::kTmemCols>(tmem_slot);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int tiles_m = (p.M + BM - 1) / BM;
    const int tiles_n = (p.N + BN - 1) / BN;
    const int k_blocks = (p.K + BK - 1) / BK;

    if (warp == 0) {
        if (elect_one()) {
            // swap (decode): each weight tile is read by exactly one CTA -> evict-first; the
            // tiny activation operand is shared by all -> evict-last.  normal (prefill): a
            // weight tile is re-read by every M-tile in flight and the activation panel by
            // every N-tile, so both are kept (evict-last).
            const uint64_t pol_stream = p.swap ? policy_evict_first() : policy_evict_last();
            const uint64_t pol_keep = policy_evict_last();
            uint32_t stage = 0, phase = 0;
            Work w;
            w.init(p, tiles_m, tiles_n, k_blocks);
            int tm, tn, kb0, kb1;
            while (w.next(tm, tn, kb0, kb1)) {
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(&empty_bar[stage], phase ^ 1);
                    mbar_expect_tx(&full_bar[stage], C::kStageBytes);
                    tma_load_2d_hint(smem_a + stage * C::kBytesA, &tmap_a, &full_bar[stage],
                                     kb * BK, tm * BM, p.swap ? pol_stream : pol_keep);
                    tma_load_2d_hint(smem_b + stage * C::kBytesB, &tmap_b, &full_bar[stage],
                                     kb * BK, tn * BN, p.swap ? pol_keep : pol_stream);
                    if (++stage == C::kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
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
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t a_addr = smem_u32(smem_a + stage * C::kBytesA);
                    const uint32_t b_addr = smem_u32(smem_b + stage * C::kBytesB);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        const uint64_t ad = make_sw128_desc(a_addr + k * 32, 16, 1024);
                        const uint64_t bd = make_sw128_desc(b_addr + k * 32, 16, 1024);
                        umma_bf16(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
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
    } else {
        // Epilogue warps 2..5: TMEM lane quarter = warp % 4.
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
            tc_fence_after();
            const int m = tm * BM + row_in_tile;
            const uint32_t t_row = tmem_base + ((quarter * 32u) << 16) + ab * BN;
#pragma unroll 1
            for (int c = 0; c < BN; c += 32) {
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
                    // swap: D[m = weight row][n = token] -> Y[token][weight row]
#pragma unroll
                    for (int j = 0; j < 32; ++j) epi.store(n0 + j, m, __uint_as_float(r[j]));
                }
            }
            tc_fence_before();
            mbar_arrive(&tempty_bar[ab]);
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<C::kTmemCols>(tmem_base);
    }
}

// Split-K finalisation: ws (fp32 [tokens][n_out]) -> epilogue -> bf16/f32 out; zeroes ws.
__global__ void gemm_finalize_kernel(const GemmParams p) {
    const int cols = p.epi == EPI_SILU ? p.n_out / 2 : p.n_out;
    const size_t total = static_cast<size_t>(p.tokens) * cols;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int tok = static_cast<int>(i / cols);
        const int c = static_cast<int>(i % cols);
        float* wrow = p.ws + static_cast<size_t>(tok) * p.n_out;
        switch (p.epi) {
        case EPI_SILU: {
            const float g = wrow[2 * c], v = wrow[2 * c + 1];
            wrow[2 * c] = 0.f;
            wrow[2 * c + 1] = 0.f;
            p.out[static_cast<size_t>(tok) * p.ldo + c] = __float2bfloat16_rn(silu(g) * v);
            break;
        }
        case EPI_BF16: {
            float v = wrow[c];
            wrow[c] = 0.f;
            if (p.bias) v += __bfloat162float(p.bias[c]);
            p.out[static_cast<size_t>(tok) * p.ldo + c] = __float2bfloat16_rn(v);
            break;
        }
        case EPI_RESID: {
            float v = wrow[c];
            wrow[c] = 0.f;
            v += __bfloat162float(p.resid[static_cast<size_t>(tok) * p.ldr + c]);
            p.out[static_cast<size_t>(tok) * p.ldo + c] = __float2bfloat16_rn(v);
            break;
        }
        case EPI_F32: {
            float v = wrow[c];
            wrow[c] = 0.f;
            p.out_f32[static_cast<size_t>(tok) * p.ldo + c] = v;
            break;
        }
        default:
            break;
        }
    }
}

template <int BN>
cudaError_t launch_bn(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                      int num_sms, cudaStream_t stream) {
    using C = GemmCfg<BN>;
    static bool attr_set = false;  // per-process; harmless race (idempotent)
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(gemm_tn_kernel<BN>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::kSmemBytes);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int tiles = ((p.M + BM - 1) / BM) * ((p.N + BN - 1) / BN);
    int grid;
    if (p.streamk) {
        const long long work = static_cast<long long>(tiles) * ((p.K + BK - 1) / BK);
        grid = static_cast<int>(std::min<long long>(num_sms, std::max<long long>(1, work / 4)));
    } else {
        const int units = tiles * p.splits;
        grid = units < num_sms ? units : num_sms;
    }
    gemm_tn_kernel<BN><<<grid, kThreads, C::kSmemBytes, stream>>>(ta, tb, p);
    return cudaGetLastError();
}

}  // namespace

int gemm_pick_bn(int n) {
    if (n <= 32) return 32;
    if (n <= 64) return 64;
    if (n <= 128) return 128;
    return 256;
}

cudaError_t gemm_launch(const CUtensorMap& ta, const CUtensorMap& tb, GemmParams p, int bn,
                        int num_sms, cudaStream_t stream) {
    const int k_blocks = (p.K + BK - 1) / BK;
    if (p.streamk) {
        p.splits = 1;
        p.kb_per_split = k_blocks;
    } else if (p.splits <= 1) {
        p.splits = 1;
        p.kb_per_split = k_blocks;
    } else {
        p.kb_per_split = (k_blocks + p.splits - 1) / p.splits;
        p.splits = (k_blocks + p.kb_per_split - 1) / p.kb_per_split;
    }
    GemmParams kp = p;
    const bool split = p.splits > 1 || p.streamk;
    if (split) kp.epi = EPI_ATOMIC;
    cudaError_t e;
    switch (bn) {
    case 32: e = launch_bn<32>(ta, tb, kp, num_sms, stream); break;
    case 64: e = launch_bn<64>(ta, tb, kp, num_sms, stream); break;
    case 128: e = launch_bn<128>(ta, tb, kp, num_sms, stream); break;
    case 256: e = launch_bn<256>(ta, tb, kp, num_sms, stream); break;
    default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess || !split) return e;
    const int cols = p.epi == EPI_SILU ? p.n_out / 2 : p.n_out;
    const long total = static_cast<long>(p.tokens) * cols;
    int blocks = static_cast<int>((total + 255) / 256);
    if (blocks > 4 * num_sms) blocks = 4 * num_sms;
    if (blocks < 1) blocks = 1;
    gemm_finalize_kernel<<<blocks, 256, 0, stream>>>(p);
    return cudaGetLastError();
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
