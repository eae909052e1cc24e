// Persistent decode-step kernel ("megakernel"): one launch = one whole decode forward for
// T <= 16 single-token rows: embedding, L x (RMSNorm+QKV+RoPE+KV append | paged attention |
// O+residual | RMSNorm+gate/up+SiLU | down+residual), final RMSNorm + LM head + greedy argmax.
// It replaces, for decode-only steps, the ~5 launches per layer of the kernel-per-op path —
// the mu_D term of the reference's decode_step_duration_ms
// (/root/reference/proj/src/executor.cpp:207-220) on the AgentServe decode partition.
//
// Why: AgentServe runs decode on a small Green Context partition (16-64 SMs).  There a decode
// step is a weight stream (0.99 GB for Qwen2.5-0.5B) at the partition's per-SM bandwidth,
// but a kernel per op pays launch + pipeline-fill + reduction latency ~2-6 us per launch,
// ~50% of the step (profiles/r1_decode_partition.json).  Here the stream never stops:
//
//   warp 8  (weight producer): walks the CTA's share of every weight of the step in order
//            into an 8-stage smem ring.  A CTA owns whole 16-row slabs of a weight (full K);
//            a stage holds the 64-column chunk of up to 8 slabs (one 2 KiB cp.async.bulk each:
//            a 16x64 slab chunk is contiguous in the tile-packed layout).  Weights do not
//            depend on activations, so it runs ahead across layer/phase boundaries, bounded
//            only by ring space.  In attention phases it streams the CTA's K/V sub-blocks (TMA,
//            SWIZZLE_128B) once the QKV barrier has passed.
//   warp 9  (activation producer): after each phase barrier, TMA-loads the [32 x 64] slice
//            of the phase input (attn / act) belonging to each stage.  Pre-norm phases (QKV,
//            gate/up, LM head) instead read a normalised copy of x the consumers write to
//            shared memory once per phase (same rounding as rmsnorm_kernel).
//   warps 0-7 (consumers): legacy warp MMAs (m16n8k16; rows = weight rows, n = tokens), warp
//            w on slab w of the stage.  Slabs are owned whole, so there are no cross-CTA
//            reductions; the fused epilogues (bias + RoPE + paged K/V append with the QKV
//            rotate_half pairs owned by one CTA, residual, SiLU*up, fp32 logits + argmax keys)
//            run as soon as a group of 8 slabs has seen its last k-block.  Attention: split-KV
//            units, warp-MMA softmax as decode_attn.cu, last-arriver merge of the splits.
//
// Phases are separated by a grid barrier (one CTA per SM, cooperative launch); weight bytes
// of the next phase are already in flight while the barrier resolves.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>

#include "attn.h"
#include "decode_step.h"
#include "epi.cuh"
#include "sm100.cuh"
#include "warpmma.cuh"

namespace asb {

namespace {

constexpr int kCons = 8;                        // consumer warps
constexpr int kThreads = (kCons + 2) * 32;      // + weight producer + activation producer
constexpr int kStages = 8;
constexpr int kWBytes = 128 * 64 * 2;           // one packed weight chunk
constexpr int kXBytes = 32 * 64 * 2;            // activation slice [32 tokens][64]
constexpr int kStageBytes = kWBytes + kXBytes;  // a K+V sub-block (<= 16 KiB) uses the W part
constexpr int kTS = 32;                         // token stride of the tile buffer
constexpr int kRing = kStages * kStageBytes;
constexpr int kTile = 128 * kTS * 4;
constexpr int kHbuf = 32 * 1024;  // normalised x (KB x 2 KiB, d <= 1024) / attention warp merge
constexpr long long kTimeoutNs = 2000000000ll;  // trap instead of hanging the GPU

enum PhaseKind { PH_QKV = 0, PH_ATTN = 1, PH_O = 2, PH_GU = 3, PH_DOWN = 4, PH_LM = 5 };

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t cnt) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ float bf16cg(const __nv_bfloat16* p) {
    const unsigned short u = __ldcg(reinterpret_cast<const unsigned short*>(p));
    return __uint_as_float(static_cast<uint32_t>(u) << 16);
}

// mbarrier parity wait with a watchdog (a protocol bug traps instead of hanging the GPU)
__device__ __forceinline__ void mbar_wait_to(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    unsigned long long t0 = 0;
    while (true) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, 1000000;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        if (t0 == 0) t0 = gtime();
        else if (gtime() - t0 > kTimeoutNs) __trap();
    }
}

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_acquire_cta_shared(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta_shared(unsigned* p, unsigned v) {
    asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// Grid-barrier generation: one poller per CTA (consumer thread 0) on the global word, relaxed
// loads with back-off and one acquire fence on success (hundreds of acquire pollers on one L2
// line starve the arrivals); the producer warps poll the CTA's shared-memory copy instead.
__device__ __forceinline__ void wait_gen(const unsigned* gen, unsigned target) {
    const unsigned long long t0 = gtime();
    while (static_cast<int>(ld_relaxed(gen) - target) < 0) {
        __nanosleep(128);
        if (gtime() - t0 > kTimeoutNs) __trap();
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void wait_gen_cta(const unsigned* gen_s, unsigned target) {
    const unsigned long long t0 = gtime();
    while (static_cast<int>(ld_acquire_cta_shared(gen_s) - target) < 0) {
        __nanosleep(32);
        if (gtime() - t0 > kTimeoutNs) __trap();
    }
}

struct Gemv {
    const __nv_bfloat16* w;
    const __nv_bfloat16* norm;  // fused pre-norm over K, or null
    int N, K, KB, src, kind, layer;
    int units;  // work units: 16-row slabs, or (QKV) pairs of slabs j / j + hd/2 of one head
};

__device__ __forceinline__ int n_phases(const MkParams& p) { return 5 * p.L + 1; }
__device__ __forceinline__ int phase_kind(int k, const MkParams& p) { return k == 5 * p.L ? PH_LM : k % 5; }

__device__ __forceinline__ Gemv gemv_of(int k, const MkParams& p) {
    Gemv g{};
    const int kind = phase_kind(k, p);
    const int l = k / 5;
    g.kind = kind;
    g.layer = l;
    const int qd = p.hq * p.hd, kvd = p.hkv * p.hd;
    switch (kind) {
    case PH_QKV: g.w = p.layers[l].wqkv; g.norm = p.layers[l].attn_norm; g.N = qd + 2 * kvd; g.K = p.d; g.src = 0; break;
    case PH_O: g.w = p.layers[l].wo; g.norm = nullptr; g.N = p.d; g.K = qd; g.src = 1; break;
    case PH_GU: g.w = p.layers[l].wgu; g.norm = p.layers[l].mlp_norm; g.N = 2 * p.ffn; g.K = p.d; g.src = 0; break;
    case PH_DOWN: g.w = p.layers[l].wdown; g.norm = nullptr; g.N = p.d; g.K = p.ffn; g.src = 2; break;
    default: g.w = p.lm_head; g.norm = p.final_norm; g.N = p.vocab; g.K = p.d; g.src = 0; break;
    }
    g.KB = g.K / 64;
    g.units = kind == PH_QKV ? g.N / 32 : (g.N + 15) / 16;
    return g;
}

// this CTA's units [u0, u1) and its slabs: slab i (0 .. n_slabs-1) starts at weight row row0(i)
struct Share {
    int u0, u1, n_slabs;
};
__device__ __forceinline__ Share share_of(const Gemv& g, int G, int c) {
    Share sh;
    sh.u0 = static_cast<int>((static_cast<long long>(g.units) * c) / G);
    sh.u1 = static_cast<int>((static_cast<long long>(g.units) * (c + 1)) / G);
    sh.n_slabs = (sh.u1 - sh.u0) * (g.kind == PH_QKV ? 2 : 1);
    return sh;
}
__device__ __forceinline__ int slab_row0(const Gemv& g, const Share& sh, int hd, int i) {
    if (g.kind != PH_QKV) return 16 * (sh.u0 + i);
    const int spp = hd / 32;  // slabs per half head
    const int u = sh.u0 + i / 2, head = u / spp, c = u % spp;
    return head * hd + (i & 1) * (hd / 2) + 16 * c;
}

// attention unit u (item = (row, kv head), split) -> [s0, s0 + n) sub-blocks of 32 tokens
__device__ __forceinline__ void unit_range(const MkParams& p, int u, int& item, int& s0, int& n) {
    item = u / p.attn_spl;
    const int split = u % p.attn_spl;
    const int ctx = p.items[item / p.hkv].ctx_len;
    const int n_sub = (ctx + 31) / 32;
    const int sps = (n_sub + p.attn_spl - 1) / p.attn_spl;
    s0 = split * sps;
    n = max(0, min(n_sub, s0 + sps) - s0);
}

struct Smem {
    uint8_t* ring;
    float* tbuf;     // [128][kTS] finished rows of one slab group (also attention split merge)
    uint8_t* hbuf;   // pre-norm phases: normalised x, [KB][16 tokens][64] SWIZZLE_128B layout
    float* mrg;      // attention: [kCons][8][hd] (aliases hbuf)
    float* mls;      // [kCons][8][2]
    float* inv;      // [32]
    unsigned long long* keys;  // [32]
    uint64_t* full;
    uint64_t* empty;
    int* flag;
    unsigned* gen0;
    unsigned* gen_s;  // last grid-barrier generation this CTA's consumers observed
};

// ------------------------------------------------------------------ consumer pieces
// One slab chunk: rows 16 x 64 k of W at wsm (row-major, 128-byte rows), X slice at xsm
// ([tokens][64] bf16, SWIZZLE_128B rows).
template <int NT>
__device__ __forceinline__ void gemv_chunk(float (&acc)[NT][4], uint32_t wsm, uint32_t xsm, int lane) {
    const int gq = lane >> 2, t = lane & 3;
    const uint4 a0 = lds128(wsm + gq * 128 + 16 * t), a1 = lds128(wsm + gq * 128 + 64 + 16 * t);
    const uint4 b0 = lds128(wsm + (gq + 8) * 128 + 16 * t), b1 = lds128(wsm + (gq + 8) * 128 + 64 + 16 * t);
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        const int tok = 8 * j + gq;
        const uint4 x0 = lds128(xsm + tok * 128 + ((t ^ (tok & 7)) << 4));
        const uint4 x1 = lds128(xsm + tok * 128 + (((t + 4) ^ (tok & 7)) << 4));
        mma16816(acc[j], a0.x, b0.x, a0.y, b0.y, x0.x, x0.y);
        mma16816(acc[j], a0.z, b0.z, a0.w, b0.w, x0.z, x0.w);
        mma16816(acc[j], a1.x, b1.x, a1.y, b1.y, x1.x, x1.y);
        mma16816(acc[j], a1.z, b1.z, a1.w, b1.w, x1.z, x1.w);
    }
}

// epilogue of one finished slab group: tbuf row 16 s + j = weight row slab_row0(s) + j
__device__ void group_epilogue(const MkParams& p, const Gemv& g, const Share& sh, int s_first, int n_s,
                               const float* tbuf, unsigned long long* keys_s) {
    const int tid = threadIdx.x, T = p.T;
    switch (g.kind) {
    case PH_QKV: {
        // slab pairs (2i, 2i+1) of the group: rows j and j + hd/2 of one head
        RopeEpi R{p.pos, p.slot, p.cos_t, p.sin_t, p.q, p.k_pool, p.v_pool, p.hq, p.hkv, p.hd, g.layer, p.num_blocks};
        const int hd = p.hd, H = hd / 2, qd = p.hq * hd, kvd = p.hkv * hd;
        const __nv_bfloat16* bias = p.layers[g.layer].qkv_bias;
        for (int e = tid; e < (n_s / 2) * 16 * T; e += kCons * 32) {
            const int jj = e % 16, pi = (e / 16) % (n_s / 2), tok = e / (16 * (n_s / 2));
            const int r1 = slab_row0(g, sh, hd, s_first + 2 * pi) + jj;  // feature of the first half
            const int f0 = (r1 / hd) * hd, j = r1 - f0;
            float x1 = tbuf[(32 * pi + jj) * kTS + tok], x2 = tbuf[(32 * pi + 16 + jj) * kTS + tok];
            if (bias) {
                x1 += __bfloat162float(bias[f0 + j]);
                x2 += __bfloat162float(bias[f0 + j + H]);
            }
            const int sl = p.slot[tok];
            if (f0 >= qd + kvd) {
                __nv_bfloat16* v = p.v_pool + pool_off(R, sl, (f0 - qd - kvd) / hd);
                v[j] = __float2bfloat16_rn(x1);
                v[j + H] = __float2bfloat16_rn(x2);
                continue;
            }
            const int ps = p.pos[tok];
            float y1, y2;
            rope2(bf16r(x1), bf16r(x2), p.cos_t[(size_t)ps * H + j], p.sin_t[(size_t)ps * H + j], y1, y2);
            __nv_bfloat16* dst = f0 < qd ? p.q + ((size_t)tok * p.hq + f0 / hd) * hd
                                         : p.k_pool + pool_off(R, sl, (f0 - qd) / hd);
            dst[j] = __float2bfloat16_rn(y1);
            dst[j + H] = __float2bfloat16_rn(y2);
        }
        break;
    }
    case PH_O:
    case PH_DOWN: {
        // <= 8 elements per thread (128 rows x T <= 16): issue every residual load, then store
        const int n0 = slab_row0(g, sh, p.hd, s_first), R = 16 * n_s;
        float rv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = tid + u * kCons * 32, i = e % R, tok = e / R;
            rv[u] = (tok < T && n0 + i < g.N) ? bf16cg(p.x + (size_t)tok * p.d + n0 + i) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = tid + u * kCons * 32, i = e % R, tok = e / R;
            if (tok < T && n0 + i < g.N)
                p.x[(size_t)tok * p.d + n0 + i] = __float2bfloat16_rn(tbuf[i * kTS + tok] + rv[u]);
        }
        break;
    }
    case PH_GU: {
        const int n0 = slab_row0(g, sh, p.hd, s_first), R = 16 * n_s;
        for (int e = tid; e < (R / 2) * T; e += kCons * 32) {
            const int i = e % (R / 2), tok = e / (R / 2), n = n0 + 2 * i;
            if (n + 1 >= g.N) continue;
            p.act[(size_t)tok * p.ffn + (n >> 1)] =
                __float2bfloat16_rn(silu(tbuf[(2 * i) * kTS + tok]) * tbuf[(2 * i + 1) * kTS + tok]);
        }
        break;
    }
    default: {  // LM head: fp32 logits + per-token greedy keys (CTA max, then one global atomic)
        const int n0 = slab_row0(g, sh, p.hd, s_first), R = 16 * n_s;
        if (tid < 32) keys_s[tid] = 0ull;
        named_sync(2, kCons * 32);
        for (int e = tid; e < R * T; e += kCons * 32) {
            const int i = e % R, tok = e / R, n = n0 + i;
            if (n >= g.N) continue;
            const float v = tbuf[i * kTS + tok];
            p.logits[(size_t)tok * p.vocab + n] = v;
            const unsigned long long k = argmax_key(v, n);
            if (k) atomicMax(&keys_s[tok], k);
        }
        named_sync(2, kCons * 32);
        if (tid < T && keys_s[tid]) atomicMax(p.keys + tid, keys_s[tid]);
        break;
    }
    }
}

// pre-norm phases: hbuf = bf16(x * rms_inv(x) * norm_w) for the T rows (rows >= T zero), laid
// out like the TMA activation slices ([kb][16][64], chunk c of row t at (c ^ (t & 7)) * 16)
__device__ void stage_normed_x(const MkParams& p, const Gemv& g, Smem& sm) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    for (int tok = warp; tok < 16; tok += kCons) {
        const float iv = tok < p.T ? rms_inv_warp_cg(p.x + (size_t)tok * p.d, p.d, p.eps, lane) : 0.f;
        if (lane == 0) sm.inv[tok] = iv;
    }
    named_sync(1, kCons * 32);
    const int n16 = g.K / 8;  // 16-byte chunks per row
    for (int e = tid; e < 16 * n16; e += kCons * 32) {
        const int tok = e / n16, c = e % n16, kb = c / 8, cc = c % 8;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (tok < p.T) {
            const uint4 xv = ldcg128(p.x + (size_t)tok * p.d + 8 * c);
            const uint4 gm = *reinterpret_cast<const uint4*>(g.norm + 8 * c);
            const float iv = sm.inv[tok];
            v = make_uint4(rms_apply2(xv.x, gm.x, iv), rms_apply2(xv.y, gm.y, iv), rms_apply2(xv.z, gm.z, iv),
                           rms_apply2(xv.w, gm.w, iv));
        }
        *reinterpret_cast<uint4*>(sm.hbuf + kb * 2048 + tok * 128 + ((cc ^ (tok & 7)) << 4)) = v;
    }
    named_sync(1, kCons * 32);
}

// consumer side of one GEMV phase
template <int NT>
__device__ void gemv_phase(const MkParams& p, const Gemv& g, Smem& sm, uint32_t& pos) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const Share sh = share_of(g, p.G, blockIdx.x);
    if (sh.n_slabs == 0) return;
    if (g.norm) stage_normed_x(p, g, sm);
    const uint32_t ring = smem_u32(sm.ring), hb = smem_u32(sm.hbuf);
    for (int s_first = 0; s_first < sh.n_slabs; s_first += 8) {
        const int n_s = min(8, sh.n_slabs - s_first);
        float acc[NT][4];
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        for (int kb = 0; kb < g.KB; ++kb, ++pos) {
            const int st = pos % kStages;
            mbar_wait_to(&sm.full[st], (pos / kStages) & 1);
            const uint32_t wsm = ring + st * kStageBytes;
            if (warp < n_s)
                gemv_chunk<NT>(acc, wsm + warp * 2048, g.norm ? hb + kb * 2048 : wsm + kWBytes, lane);
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty[st]);
        }
        {
            const int gq = lane >> 2, t = lane & 3, ra = 16 * warp + gq;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                sm.tbuf[ra * kTS + 8 * j + 2 * t] = acc[j][0];
                sm.tbuf[ra * kTS + 8 * j + 2 * t + 1] = acc[j][1];
                sm.tbuf[(ra + 8) * kTS + 8 * j + 2 * t] = acc[j][2];
                sm.tbuf[(ra + 8) * kTS + 8 * j + 2 * t + 1] = acc[j][3];
            }
        }
        named_sync(1, kCons * 32);
        group_epilogue(p, g, sh, s_first, n_s, sm.tbuf, sm.keys);
        named_sync(1, kCons * 32);
    }
}

// consumer side of one attention phase (layer l)
template <int HD>
__device__ void attn_phase(const MkParams& p, Smem& sm, uint32_t& pos) {
    constexpr int NTD = HD / 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
    const int gq = lane >> 2, t = lane & 3;
    const int G = p.G, Gh = p.hq / p.hkv;
    const int n_units = p.T * p.hkv * p.attn_spl;
    const uint32_t ring = smem_u32(sm.ring);
    for (int u = blockIdx.x; u < n_units; u += G) {
        int item, s0, n_local;
        unit_range(p, u, item, s0, n_local);
        const int b = item / p.hkv, kvh = item % p.hkv;
        const DecodeItem it = p.items[b];
        uint32_t qa[HD / 16][2];
        {
            const __nv_bfloat16* qrow = p.q + (size_t)it.q_row * p.hq * HD + (size_t)(kvh * Gh + gq) * HD;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
                if (gq < Gh) {
                    qa[kk][0] = __ldcg(reinterpret_cast<const unsigned*>(qrow + kk * 16 + 2 * t));
                    qa[kk][1] = __ldcg(reinterpret_cast<const unsigned*>(qrow + kk * 16 + 2 * t + 8));
                } else {
                    qa[kk][0] = qa[kk][1] = 0u;
                }
            }
        }
        float o[NTD][4];
#pragma unroll
        for (int n = 0; n < NTD; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
        float m_run = -FLT_MAX, l_run = 0.f;
        for (int i = 0; i < n_local; ++i) {
            const uint32_t P = pos + i;
            if (static_cast<int>(P % kCons) != warp) continue;
            const int st = P % kStages;
            mbar_wait_to(&sm.full[st], (P / kStages) & 1);
            const uint32_t kt = ring + st * kStageBytes;
            const uint32_t vt = kt + 32 * HD * 2;
            float sacc[4][4];
#pragma unroll
            for (int n = 0; n < 4; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
#pragma unroll
                for (int np = 0; np < 2; ++np) {
                    const int mi = lane >> 3;
                    const int key = (2 * np + (mi >> 1)) * 8 + (lane & 7);
                    const int chunk = 2 * kk + (mi & 1);
                    uint32_t b0, b1, b2, b3;
                    ldsm_x4(kt + sw_off<HD>(key, chunk), b0, b1, b2, b3);
                    mma16816(sacc[2 * np], qa[kk][0], 0u, qa[kk][1], 0u, b0, b1);
                    mma16816(sacc[2 * np + 1], qa[kk][0], 0u, qa[kk][1], 0u, b2, b3);
                }
            }
            const int kbase = (s0 + i) * 32;
            float mx = m_run;
#pragma unroll
            for (int n = 0; n < 4; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const bool ok = kbase + 8 * n + 2 * t + e < it.ctx_len;
                    sacc[n][e] = ok ? sacc[n][e] * p.scale_log2 : -FLT_MAX;
                    mx = fmaxf(mx, sacc[n][e]);
                }
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float alpha = exp2f(m_run - mx);
            float psum = 0.f;
            uint32_t pa[2][2];
#pragma unroll
            for (int n = 0; n < 4; ++n) {
                const float p0 = sacc[n][0] == -FLT_MAX ? 0.f : exp2f(sacc[n][0] - mx);
                const float p1 = sacc[n][1] == -FLT_MAX ? 0.f : exp2f(sacc[n][1] - mx);
                const uint32_t pk = pack_bf16(p0, p1);
                psum += bf16_lo(pk) + bf16_hi(pk);
                pa[n >> 1][n & 1] = pk;
            }
            psum += __shfl_xor_sync(0xffffffffu, psum, 1);
            psum += __shfl_xor_sync(0xffffffffu, psum, 2);
            l_run = l_run * alpha + psum;
            m_run = mx;
#pragma unroll
            for (int n = 0; n < NTD; ++n) {
                o[n][0] *= alpha;
                o[n][1] *= alpha;
            }
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
                for (int dp = 0; dp < NTD / 2; ++dp) {
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
            if (lane == 0) mbar_arrive_cnt(&sm.empty[st], kCons);
        }
        pos += n_local;
        // ---- merge the 8 warps of this unit, write the split partial
        float* mw = sm.mrg + warp * 8 * HD;
        if (gq < Gh) {
#pragma unroll
            for (int n = 0; n < NTD; ++n) {
                mw[gq * HD + n * 8 + 2 * t] = o[n][0];
                mw[gq * HD + n * 8 + 2 * t + 1] = o[n][1];
            }
            if (t == 0) {
                sm.mls[(warp * 8 + gq) * 2] = m_run;
                sm.mls[(warp * 8 + gq) * 2 + 1] = l_run;
            }
        }
        named_sync(1, kCons * 32);
        const int split = u % p.attn_spl;
        for (int e = tid; e < Gh * HD; e += kCons * 32) {
            const int h = e / HD, dd = e % HD;
            float M = -FLT_MAX;
#pragma unroll
            for (int w = 0; w < kCons; ++w) M = fmaxf(M, sm.mls[(w * 8 + h) * 2]);
            float L = 0.f, O = 0.f;
#pragma unroll
            for (int w = 0; w < kCons; ++w) {
                const float lw = sm.mls[(w * 8 + h) * 2 + 1];
                if (lw == 0.f) continue;
                const float f = exp2f(sm.mls[(w * 8 + h) * 2] - M);
                L += lw * f;
                O += sm.mrg[(w * 8 + h) * HD + dd] * f;
            }
            const size_t slot = ((size_t)item * p.attn_spl + split) * Gh + h;
            __stcg(p.apart_o + slot * HD + dd, O);
            if (dd == 0) {
                __stcg(p.apart_ml + slot * 2, M);
                __stcg(p.apart_ml + slot * 2 + 1, L);
            }
        }
        __threadfence();
        named_sync(1, kCons * 32);
        if (tid == 0) {
            const int prev = atomicAdd(p.acnt + item, 1);
            const bool last = prev == p.attn_spl - 1;
            if (last) p.acnt[item] = 0;
            *sm.flag = last;
        }
        named_sync(1, kCons * 32);
        if (*sm.flag) {
            __threadfence();
            // merge the splits (decode_combine arithmetic, split order): every (m, l) load in
            // flight at once, per-head weights in smem, then every split's O load at once
            const int spl = p.attn_spl;
            float* wm = sm.tbuf;           // [Gh][spl] m, then the weights exp2(m - M)
            float* wl = sm.tbuf + 8 * 16;  // [Gh][spl] l
            float* li = wl + 8 * 16;       // [Gh] L
            for (int i = tid; i < Gh * spl; i += kCons * 32) {
                const int h = i / spl, sp = i % spl;
                const size_t sl = ((size_t)item * spl + sp) * Gh + h;
                wm[i] = __ldcg(p.apart_ml + sl * 2);
                wl[i] = __ldcg(p.apart_ml + sl * 2 + 1);
            }
            named_sync(1, kCons * 32);
            if (tid < Gh) {
                float M = -FLT_MAX;
                for (int sp = 0; sp < spl; ++sp) M = fmaxf(M, wm[tid * spl + sp]);
                float L = 0.f;
                for (int sp = 0; sp < spl; ++sp) {
                    const float ls = wl[tid * spl + sp];
                    const float w = ls == 0.f ? 0.f : exp2f(wm[tid * spl + sp] - M);
                    wm[tid * spl + sp] = w;
                    L += ls * w;
                }
                li[tid] = L;
            }
            named_sync(1, kCons * 32);
            for (int e = tid; e < Gh * HD; e += kCons * 32) {
                const int h = e / HD, dd = e % HD;
                float po[16];
#pragma unroll
                for (int sp = 0; sp < 16; ++sp)
                    po[sp] = sp < spl ? __ldcg(p.apart_o + (((size_t)item * spl + sp) * Gh + h) * HD + dd) : 0.f;
                float O = 0.f;
#pragma unroll
                for (int sp = 0; sp < 16; ++sp)
                    if (sp < spl && wm[h * spl + sp] != 0.f) O += po[sp] * wm[h * spl + sp];
                p.attn[(size_t)it.q_row * p.hq * HD + (kvh * Gh + h) * HD + dd] = __float2bfloat16_rn(O / li[h]);
            }
        }
        named_sync(1, kCons * 32);
    }
}

// grid barrier among the consumer warps of all CTAs (arrivals: p.bar[0]; generation: p.bar[32],
// its own 128-byte line)
__device__ __forceinline__ void grid_sync(const MkParams& p, Smem& sm, unsigned& gen) {
    fence_proxy_async_global();  // generic-proxy stores -> TMA readers on other SMs
    __threadfence();
    named_sync(1, kCons * 32);
    ++gen;
    if (threadIdx.x == 0) {
        if (atomicAdd(p.bar, 1u) == static_cast<unsigned>(p.G) - 1) {
            p.bar[0] = 0;
            __threadfence();
            st_release(p.bar + 32, gen);
        } else {
            wait_gen(p.bar + 32, gen);
        }
        st_release_cta_shared(sm.gen_s, gen);
    }
    named_sync(1, kCons * 32);
}

template <int NT, int HD>
__global__ void __launch_bounds__(kThreads, 1)
    decode_step_kernel(const __grid_constant__ MkMaps maps, const MkParams p) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    uint8_t* base = smem_raw + (((raw + 1023) & ~1023u) - raw);
    Smem sm;
    sm.ring = base;
    sm.tbuf = reinterpret_cast<float*>(base + kRing);
    sm.hbuf = base + kRing + kTile;
    sm.mrg = reinterpret_cast<float*>(sm.hbuf);
    sm.mls = reinterpret_cast<float*>(sm.hbuf + kHbuf);
    sm.inv = sm.mls + kCons * 16;
    sm.keys = reinterpret_cast<unsigned long long*>(sm.inv + 32);
    sm.full = reinterpret_cast<uint64_t*>(sm.keys + 32);
    sm.empty = sm.full + kStages;
    sm.flag = reinterpret_cast<int*>(sm.empty + kStages);
    sm.gen0 = reinterpret_cast<unsigned*>(sm.flag + 1);
    sm.gen_s = sm.gen0 + 1;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&sm.full[s], 2);       // weight/KV producer + activation producer
            mbar_init(&sm.empty[s], kCons);  // every consumer warp (attention: owner x 8)
        }
        fence_barrier_init();
        *sm.gen0 = ld_acquire(p.bar + 32);
        *sm.gen_s = *sm.gen0;
    }
    __syncthreads();
    const unsigned gen0 = *sm.gen0;
    const int K = n_phases(p);

    if (warp == kCons) {
        // ------------------------------------------------------------ weight / KV producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            uint32_t pos = 0;
            for (int k = 0; k < K; ++k) {
                if (phase_kind(k, p) == PH_ATTN) {
                    wait_gen_cta(sm.gen_s, gen0 + k + 1);  // the QKV phase appended this step's K/V
                    fence_proxy_async_global();
                    const int l = k / 5;
                    const int n_units = p.T * p.hkv * p.attn_spl;
                    for (int u = blockIdx.x; u < n_units; u += p.G) {
                        int item, s0, n;
                        unit_range(p, u, item, s0, n);
                        const int kvh = item % p.hkv;
                        const int32_t* table = p.tables + p.items[item / p.hkv].table_off;
                        for (int i = 0; i < n; ++i, ++pos) {
                            const int st = pos % kStages;
                            mbar_wait_to(&sm.empty[st], ((pos / kStages) & 1) ^ 1);
                            mbar_expect_tx(&sm.full[st], 2 * 32 * HD * 2);
                            const int j = s0 + i;
                            const int blk = table[j >> 1];
                            const int row = ((l * p.num_blocks + blk) * p.hkv + kvh) * kBlockTokens + (j & 1) * 32;
                            uint8_t* kd = sm.ring + st * kStageBytes;
                            uint8_t* vd = kd + 32 * HD * 2;
#pragma unroll
                            for (int h = 0; h < HD / 64; ++h) {
                                tma_load_2d_hint(kd + h * (32 * 128), &maps.k32, &sm.full[st], h * 64, row, pol);
                                tma_load_2d_hint(vd + h * (32 * 128), &maps.v32, &sm.full[st], h * 64, row, pol);
                            }
                        }
                    }
                    continue;
                }
                const Gemv g = gemv_of(k, p);
                const Share sh = share_of(g, p.G, blockIdx.x);
                for (int s_first = 0; s_first < sh.n_slabs; s_first += 8) {
                    const int n_s = min(8, sh.n_slabs - s_first);
                    const __nv_bfloat16* src[8];
                    for (int i = 0; i < n_s; ++i) {
                        const int r0 = slab_row0(g, sh, p.hd, s_first + i);
                        src[i] = g.w + ((size_t)(r0 >> 7) * g.KB * 128 + (r0 & 127)) * 64;
                    }
                    for (int kb = 0; kb < g.KB; ++kb, ++pos) {
                        const int st = pos % kStages;
                        mbar_wait_to(&sm.empty[st], ((pos / kStages) & 1) ^ 1);
                        mbar_expect_tx(&sm.full[st], n_s * 2048);
                        for (int i = 0; i < n_s; ++i)
                            bulk_g2s(sm.ring + st * kStageBytes + i * 2048, src[i] + (size_t)kb * 8192, 2048,
                                     &sm.full[st], pol);
                    }
                }
            }
        }
        return;
    }
    if (warp == kCons + 1) {
        // ------------------------------------------------------------ activation producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_last();
            uint32_t pos = 0;
            for (int k = 0; k < K; ++k) {
                if (phase_kind(k, p) == PH_ATTN) {
                    const int n_units = p.T * p.hkv * p.attn_spl;
                    for (int u = blockIdx.x; u < n_units; u += p.G) {
                        int item, s0, n;
                        unit_range(p, u, item, s0, n);
                        for (int i = 0; i < n; ++i, ++pos) {
                            const int st = pos % kStages;
                            mbar_wait_to(&sm.empty[st], ((pos / kStages) & 1) ^ 1);
                            mbar_arrive(&sm.full[st]);
                        }
                    }
                    continue;
                }
                const Gemv g = gemv_of(k, p);
                const Share sh = share_of(g, p.G, blockIdx.x);
                const int n_pos = ((sh.n_slabs + 7) / 8) * g.KB;
                if (g.norm) {  // consumers stage the normalised x themselves
                    for (int i = 0; i < n_pos; ++i, ++pos) {
                        const int st = pos % kStages;
                        mbar_wait_to(&sm.empty[st], ((pos / kStages) & 1) ^ 1);
                        mbar_arrive(&sm.full[st]);
                    }
                    continue;
                }
                if (n_pos == 0) continue;
                wait_gen_cta(sm.gen_s, gen0 + k + 1);  // the phase before produced this input
                fence_proxy_async_global();
                const CUtensorMap* m = g.src == 1 ? &maps.attn : &maps.act;
                for (int i = 0; i < n_pos; ++i, ++pos) {
                    const int st = pos % kStages;
                    mbar_wait_to(&sm.empty[st], ((pos / kStages) & 1) ^ 1);
                    mbar_expect_tx(&sm.full[st], kXBytes);
                    tma_load_2d_hint(sm.ring + st * kStageBytes + kWBytes, m, &sm.full[st], (i % g.KB) * 64, 0, pol);
                }
            }
        }
        return;
    }

    // ---------------------------------------------------------------- consumers
    unsigned gen = gen0;
    uint32_t pos = 0;
    {
        // embedding rows (tile-packed table) and the argmax accumulators
        const int tid = threadIdx.x;
        for (int tok = blockIdx.x; tok < p.T; tok += p.G) {
            const long long R = p.tok[tok];
            const int kb = p.d / 64;
            for (int i = tid; i < p.d / 8; i += kCons * 32) {
                const int col = 8 * i;
                const __nv_bfloat16* src = p.embed + ((R >> 7) * kb + col / 64) * 8192 + (R & 127) * 64 + (col & 63);
                *reinterpret_cast<uint4*>(p.x + (size_t)tok * p.d + col) = *reinterpret_cast<const uint4*>(src);
            }
        }
        if (blockIdx.x == 0 && tid < p.T) p.keys[tid] = 0ull;
    }
    grid_sync(p, sm, gen);
    for (int k = 0; k < K; ++k) {
        if (p.dbg && threadIdx.x == 0 && k < kMkDbgSlots - 1) p.dbg[blockIdx.x * kMkDbgSlots + k] = gtime();
        if (phase_kind(k, p) == PH_ATTN) {
            attn_phase<HD>(p, sm, pos);
        } else {
            gemv_phase<NT>(p, gemv_of(k, p), sm, pos);
        }
        if (k + 1 < K) grid_sync(p, sm, gen);
    }
    if (p.dbg && threadIdx.x == 0) p.dbg[blockIdx.x * kMkDbgSlots + kMkDbgSlots - 1] = gtime();
}

template <int NT, int HD>
cudaError_t launch_t(const MkMaps& maps, const MkParams& p, cudaStream_t st) {
    const int smem = decode_step_smem_bytes(HD);
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(decode_step_kernel<NT, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeCooperative;
    a[0].val.cooperative = 1;
    cfg.attrs = a;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, decode_step_kernel<NT, HD>, maps, p);
}

}  // namespace

int decode_step_smem_bytes(int hd) {
    (void)hd;
    return 1024 + kRing + kTile + kHbuf + kCons * 16 * 4 + 32 * 4 + 32 * 8 + 2 * kStages * 8 + 16;
}

cudaError_t decode_step_launch(const MkMaps& maps, const MkParams& p, cudaStream_t stream) {
    if (p.T < 1 || p.T > kMkMaxRows || p.G < 1 || (p.hq / p.hkv) > 8) return cudaErrorInvalidValue;
    const bool two = p.T > 8;
    if (p.hd == 64) return two ? launch_t<2, 64>(maps, p, stream) : launch_t<1, 64>(maps, p, stream);
    if (p.hd == 128) return two ? launch_t<2, 128>(maps, p, stream) : launch_t<1, 128>(maps, p, stream);
    return cudaErrorInvalidValue;
}

}  // namespace asb
