// Device runtime behind the asb_* C ABI (include/agentserve_b200.h): model weights,
// paged KV pool + host block allocator (with the reference KvCacheRegistry protocol),
// execution lanes and the ragged-batch SLM forward.
//
// The forward is the work the reference simulates at its two seams:
//   decode step  -> decode_step_duration_ms   (/root/reference/proj/src/executor.cpp:84-97)
//   prefill unit -> remaining / rate           (/root/reference/proj/src/engine.cpp:450-475)
// Numerics contract (restated by oracle/forward.c): bf16 storage of x / h / qkv / q / k / v /
// attn / act, fp32 accumulation, single rounding after bias / residual / SiLU·mul epilogues.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <cstdio>
#include <vector>

#include "../../include/agentserve_b200.h"
#include "attn.h"
#include "ew.h"
#include "gemm.h"
#include "launch.cuh"
#include "json.hpp"
#include "runtime.h"
#include "sm100.cuh"

using asb::kBlockTokens;
using nlohmann::json;

namespace asb {

thread_local std::string g_err;

struct AsbError : std::runtime_error {
    asb_status st;
    AsbError(asb_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

[[noreturn]] void fail(asb_status s, const std::string& m) { throw AsbError(s, m); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        fail(ASB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    }
}

template <typename Fn>
asb_status guarded(Fn&& fn) {
    try {
        fn();
        return ASB_OK;
    } catch (const AsbError& e) {
        g_err = e.what();
        return e.st;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ASB_ERR_INVALID_ARGUMENT;
    }
}

// ------------------------------------------------------------------ model spec
static uint64_t fnv1a(const std::string& s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (unsigned char c : s) {
        h ^= c;
        h *= 0x00000100000001b3ull;
    }
    return h;
}
static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
uint64_t substream_state(uint64_t seed, const std::string& name) { return mix64(seed ^ fnv1a(name)); }

ModelSpec spec_preset(const std::string& name) {
    ModelSpec s;
    s.name = name;
    if (name == "tiny") {
        s.layers = 2; s.d = 256; s.hq = 4; s.hkv = 2; s.hd = 64; s.ffn = 704; s.vocab = 4096;
        s.tied = true; s.qkv_bias = false; s.theta = 10000.0; s.eps = 1e-6f;
    } else if (name == "qwen2.5-0.5b") {
        s.layers = 24; s.d = 896; s.hq = 14; s.hkv = 2; s.hd = 64; s.ffn = 4864; s.vocab = 151936;
        s.tied = true; s.qkv_bias = true; s.theta = 1000000.0; s.eps = 1e-6f;
    } else if (name == "llama3.2-3b") {
        s.layers = 28; s.d = 3072; s.hq = 24; s.hkv = 8; s.hd = 128; s.ffn = 8192; s.vocab = 128256;
        s.tied = true; s.qkv_bias = false; s.theta = 500000.0; s.eps = 1e-5f;
        s.rope_llama3 = true; s.rope_factor = 32.0; s.rope_lo = 1.0; s.rope_hi = 4.0; s.rope_orig = 8192;
    } else if (name == "qwen2.5-7b") {
        s.layers = 28; s.d = 3584; s.hq = 28; s.hkv = 4; s.hd = 128; s.ffn = 18944; s.vocab = 152064;
        s.tied = false; s.qkv_bias = true; s.theta = 1000000.0; s.eps = 1e-6f;
    } else if (name == "llama3.1-8b") {
        s.layers = 32; s.d = 4096; s.hq = 32; s.hkv = 8; s.hd = 128; s.ffn = 14336; s.vocab = 128256;
        s.tied = false; s.qkv_bias = false; s.theta = 500000.0; s.eps = 1e-5f;
        s.rope_llama3 = true; s.rope_factor = 8.0; s.rope_lo = 1.0; s.rope_hi = 4.0; s.rope_orig = 8192;
    } else {
        fail(ASB_ERR_VALIDATION, "unknown model preset '" + name + "'");
    }
    return s;
}

ModelSpec parse_spec(const std::string& text) {
    if (text.empty() || text[0] != '{') return spec_preset(text);
    json j;
    try {
        j = json::parse(text);
    } catch (const json::exception& e) {
        fail(ASB_ERR_VALIDATION, std::string("model spec is not JSON: ") + e.what());
    }
    ModelSpec s = j.contains("preset") ? spec_preset(j["preset"].get<std::string>()) : ModelSpec{};
    if (!j.contains("preset")) s.name = j.value("name", std::string("custom"));
    s.layers = j.value("layers", s.layers);
    s.d = j.value("d_model", s.d);
    s.hq = j.value("n_heads", s.hq);
    s.hkv = j.value("n_kv_heads", s.hkv);
    s.hd = j.value("head_dim", s.hd);
    s.ffn = j.value("ffn", s.ffn);
    s.vocab = j.value("vocab", s.vocab);
    s.tied = j.value("tied", s.tied);
    s.qkv_bias = j.value("qkv_bias", s.qkv_bias);
    s.theta = j.value("rope_theta", s.theta);
    s.eps = j.value("rms_eps", s.eps);
    return s;
}

void validate_spec(const ModelSpec& s) {
    if (s.layers < 1 || s.d < 64 || s.hq < 1 || s.hkv < 1 || s.vocab < 2 || s.ffn < 64)
        fail(ASB_ERR_VALIDATION, "model spec: non-positive dimension");
    if (s.hd != 64 && s.hd != 128) fail(ASB_ERR_VALIDATION, "model spec: head_dim must be 64 or 128");
    if (s.hq % s.hkv != 0 || s.hq / s.hkv > 8)
        fail(ASB_ERR_VALIDATION, "model spec: n_heads must be a multiple of n_kv_heads, group <= 8");
    if (s.d % 64 || s.ffn % 64 || (s.hq * s.hd) % 64)
        fail(ASB_ERR_VALIDATION, "model spec: d_model, ffn and n_heads*head_dim must be multiples of 64");
}

// RoPE inverse frequencies (double), Llama-3 wavelength scaling when requested.
std::vector<double> rope_inv_freq(const ModelSpec& s) {
    const int half = s.hd / 2;
    std::vector<double> f(half);
    for (int i = 0; i < half; ++i) {
        double inv = 1.0 / std::pow(s.theta, (2.0 * i) / s.hd);
        if (s.rope_llama3) {
            const double lo_wl = s.rope_orig / s.rope_lo, hi_wl = s.rope_orig / s.rope_hi;
            const double wl = 2.0 * M_PI / inv;
            if (wl > lo_wl) {
                inv = inv / s.rope_factor;
            } else if (wl >= hi_wl) {
                const double smooth = (s.rope_orig / wl - s.rope_lo) / (s.rope_hi - s.rope_lo);
                inv = (1.0 - smooth) * inv / s.rope_factor + smooth * inv;
            }
        }
        f[i] = inv;
    }
    return f;
}

// ------------------------------------------------------------------ weights
static void* dmalloc(size_t bytes, std::vector<void*>& track) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    track.push_back(p);
    return p;
}

// Weights are stored tile-packed, [N/128][K/64][128 rows][64 cols]: one 128x64 TMA box is a
// contiguous 16 KiB chunk, so streaming a weight tile is a run of long sequential HBM reads
// instead of 128 strided 128-byte pieces.
static void weight_maps(Weight& w) {
    if (!make_tmap_packed(&w.map_b256, w.ptr, w.rows_pad, w.cols, 2) ||
        !make_tmap_packed(&w.map_a128, w.ptr, w.rows_pad, w.cols, 1) ||
        !make_tmap_packed(&w.map_a128k2, w.ptr, w.rows_pad, w.cols, 1, 2))
        fail(ASB_ERR_CUDA, "cuTensorMapEncodeTiled failed for a weight");
}

}  // namespace asb

using namespace asb;

// =================================================================== model
struct asb_model {
    ModelSpec spec;
    int device = 0;
    int num_sms = 148;
    uint64_t seed = 0;
    int max_ctx = 0;
    std::vector<void*> allocs;
    Weight embed, lm_head;
    __nv_bfloat16* final_norm = nullptr;
    struct Layer {
        __nv_bfloat16 *attn_norm, *mlp_norm, *qkv_bias;
        Weight qkv, o, gate_up, down;
    };
    std::vector<Layer> layers;
    float *cos_t = nullptr, *sin_t = nullptr;

    ~asb_model() {
        cudaSetDevice(device);
        for (void* p : allocs) cudaFree(p);
    }
};

namespace {

// vectors (norms, biases): row-major
void fill(const asb_model* m, __nv_bfloat16* dst, const std::string& name, int64_t rows, int cols,
          int row_mult, int row_off, float offset, float amp) {
    cuda_check(init_weights(dst, substream_state(m->seed, name), rows, cols, row_mult, row_off, 0, offset,
                            amp, nullptr),
               "init_weights");
}
// matrices: tile-packed; source row r -> logical row r*row_mult + row_off of w
void fillw(const asb_model* m, const Weight& w, const std::string& name, int64_t rows, int row_mult,
           int row_off) {
    cuda_check(init_weights(w.ptr, substream_state(m->seed, name), rows, w.cols, row_mult, row_off,
                            w.cols / 64, 0.f, 0.034641016f, nullptr),
               "init_weights");
}

constexpr float kAmpW = 0.034641016f;  // uniform amplitude with std 0.02
constexpr float kAmpB = 0.1f;
constexpr float kAmpN = 0.1f;

}  // namespace

// =================================================================== kv
struct asb_kv {
    asb_model* m = nullptr;
    int nb = 0;
    __nv_bfloat16* pool = nullptr;  // interleaved K|V pages (attn.h)
    __nv_bfloat16 *k_pool = nullptr, *v_pool = nullptr;  // pool, pool + one page (element views)
    CUtensorMap tk, tv;      // box 64 rows (prefill attention)
    CUtensorMap tkv;         // whole K|V block per box (decode attention)
    std::vector<int> free_list;  // LIFO: back() is handed out next
    struct Sess {
        std::vector<int32_t> blocks;
        int len = 0;
        int prefix = 0;
        bool sealed = false;
    };
    std::map<uint32_t, Sess> sess;

    ~asb_kv() {
        cudaSetDevice(m->device);
        cudaFree(pool);
    }
    Sess& get(uint32_t s) { return sess[s]; }
    void ensure(Sess& s, int new_len) {
        const int need = (new_len + kBlockTokens - 1) / kBlockTokens;
        while (static_cast<int>(s.blocks.size()) < need) {
            if (free_list.empty())
                fail(ASB_ERR_INFEASIBLE, "KV pool exhausted (" + std::to_string(nb) + " blocks)");
            s.blocks.push_back(free_list.back());
            free_list.pop_back();
        }
    }
};

// =================================================================== lane
struct asb_lane {
    asb_model* m = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int max_T = 0, max_segs = 0, max_tbl = 0, max_pitems = 0, max_splits = 16;
    int max_ditems = 0;  // decode-attention rows: single-token rows + admitted-chunk tokens
    __nv_bfloat16 *x, *h, *qkv, *q, *attn, *act, *hl;
    float *logits, *part_o, *part_ml, *ppart_o, *ppart_ml;
    int* dcnt = nullptr;  // decode-attention split arrival counters [rows][hkv] (self-resetting)
    int* post_cnt = nullptr;  // grid arrival counter of the fused post-norm (self-resetting)
    float* tg_ws = nullptr;   // tgemv split partials [4 * SMs units][32][128] fp32
    int* tg_cnt = nullptr;    // tgemv per-tile split arrival counters (self-resetting)
    // split merge inside the decode-attention kernel (last-arriving split) instead of a
    // combine launch; ASB_ATTN_COMBINE=1 selects the separate combine kernel
    bool attn_fused_merge = std::getenv("ASB_ATTN_COMBINE") == nullptr;
    unsigned long long* attn_dbg = nullptr;  // ASB_ATTN_TIMELINE=1: decode-attention CTA stamps
    CUtensorMap map_x[8];
    bool pdl = std::getenv("ASB_NO_PDL") == nullptr;  // programmatic dependent launch
    unsigned long long* dbg_times = nullptr;  // ASB_GEMM_TIMELINE: per-CTA stamps of the last GEMM
    size_t ppart_rows = 0;
    int32_t* d_meta = nullptr;
    int32_t* h_meta = nullptr;
    unsigned long long* d_out = nullptr;  // per logit row argmax_key (fused into the LM head)
    unsigned long long* h_out = nullptr;
    size_t meta_ints = 0;
    std::vector<void*> allocs;
    // tensor maps of GEMM inputs: [0] box 128 (normal A), [1..4] box 32/64/128/256 (swap B)
    CUtensorMap map_h[8], map_attn[8], map_act[8], map_hl[8], map_q;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_switch = nullptr;  // orders a rebound stream after the old one (set_stream)
    bool launched = false;
    int last_logit_rows = 0;
    // per-category kernel timing (asb_lane_profile / asb_lane_stats)
    struct Mark {
        cudaEvent_t a, b;
        int cat;
        double units;
    };
    bool prof = false;
    std::vector<Mark> marks;
    std::vector<cudaEvent_t> pool;
    double st_ms[ASB_STAT_COUNT] = {}, st_units[ASB_STAT_COUNT] = {};
    int64_t st_n[ASB_STAT_COUNT] = {};
    int sms = 0;  // SMs of the partition the lane's stream runs on (0: whole device)
    int64_t n_launch = 0, h2d = 0, d2h = 0;
    int n_sms() const { return sms > 0 ? sms : m->num_sms; }

    cudaEvent_t take_event() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        cuda_check(cudaEventCreate(&e), "event");
        return e;
    }
    template <typename Fn>
    void timed(int cat, double units, Fn&& fn) {
        if (!prof) {
            fn();
            return;
        }
        Mark m{take_event(), take_event(), cat, units};
        cuda_check(cudaEventRecord(m.a, stream), "event");
        fn();
        cuda_check(cudaEventRecord(m.b, stream), "event");
        marks.push_back(m);
    }
    void resolve_marks() {
        for (auto& m : marks) {
            float ms = 0.f;
            if (cudaEventSynchronize(m.b) == cudaSuccess && cudaEventElapsedTime(&ms, m.a, m.b) == cudaSuccess) {
                st_ms[m.cat] += ms;
                st_units[m.cat] += m.units;
                st_n[m.cat] += 1;
            }
            pool.push_back(m.a);
            pool.push_back(m.b);
        }
        marks.clear();
    }

    ~asb_lane() {
        cudaSetDevice(m->device);
        if (launched) cudaStreamSynchronize(stream);
        if (ev_switch) cudaEventDestroy(ev_switch);
        for (void* p : allocs) cudaFree(p);
        if (h_meta) cudaFreeHost(h_meta);
        if (h_out) cudaFreeHost(h_out);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (auto& m : marks) {
            cudaEventDestroy(m.a);
            cudaEventDestroy(m.b);
        }
        for (auto e : pool) cudaEventDestroy(e);
        if (own_stream && stream) cudaStreamDestroy(stream);
    }
};

namespace {

// [0] box 128 rows (normal-path A), [1..4] box 32/64/128/256 (swap-path B), [5..6] k-pair
// boxes of 32/64 rows (swap-path B with two k-blocks per stage), [7] k-pair box of 16 rows
// (tgemv at <= 16 tokens)
constexpr int kActMaps = 8;
constexpr int kDItemInts = int(sizeof(DecodeItem) / 4);  // DecodeItem slots in the meta block
void act_maps(CUtensorMap* maps, const void* base, int rows, int cols) {
    const int boxes[5] = {128, 32, 64, 128, 256};
    for (int i = 0; i < 5; ++i)
        if (!make_tmap_bf16(&maps[i], base, rows, cols, cols, boxes[i]))
            fail(ASB_ERR_CUDA, "cuTensorMapEncodeTiled failed for an activation");
    if (!make_tmap_act_kpair(&maps[5], base, rows, cols, 32) || !make_tmap_act_kpair(&maps[6], base, rows, cols, 64) ||
        !make_tmap_act_kpair(&maps[7], base, rows, cols, 16))
        fail(ASB_ERR_CUDA, "cuTensorMapEncodeTiled failed for an activation (k-pair)");
}

int swap_map_index(int bn) { return bn == 32 ? 1 : bn == 64 ? 2 : bn == 128 ? 3 : 4; }

// The X operand of a linear layer: TMA maps for the tcgen05 paths, the raw rows for the
// small-batch dgemv path, which can also apply the layer's RMSNorm on the fly (norm_w) and
// gather its rows (rows, the LM-head logit rows).
struct XIn {
    const CUtensorMap* maps;
    const __nv_bfloat16* ptr;
    int ld;
    const __nv_bfloat16* norm_w = nullptr;
    const int32_t* rows = nullptr;
    float eps = 0.f;
};

// Small-batch decode path for this linear?  dgemv wins where the launch is latency-bound
// (few weight bytes); above ~24 MB of weights the tcgen05 swap-AB kernel already streams at
// ~6 TB/s (profiles/r1_gemm_bench_dgemv.json).  ASB_NO_DGEMV=1: tcgen05 everywhere.
bool use_dgemv(int T, const Weight& w, int num_sms) {
    static const bool off = std::getenv("ASB_NO_DGEMV") && std::atoi(std::getenv("ASB_NO_DGEMV")) != 0;
    const double bytes = 2.0 * double(w.rows) * w.cols;
    // Measured crossover: in isolation dgemv wins while each SM of the partition streams
    // <= ~160 KB of the weight (profiles/r1_gemm_bench_partitions.json), but inside a decode
    // step on <= 32 SMs the all-tcgen05 chain is faster (1.71 vs 1.78 ms at 16 SMs, 1.31 vs
    // 1.32 at 32): dgemv's two 8-warp CTAs fill an SM's registers, so the next PDL launch
    // cannot become resident and prefetch its weights; from 64 SMs up dgemv wins (1.02 vs
    // 1.10 ms at 64, 0.84 vs 0.97 at 148; scripts/step_launches.py --level=L, B=2).
    const double per_sm = bytes / num_sms;
    return !off && T <= 16 && num_sms > 32 && per_sm <= 160e3;
}

// tgemv split workspace of a lane: units <= 4 waves of one CTA per SM (tgemv_splits)
constexpr int kTgMaxUnits = 4 * 160;
constexpr int kTgMaxTiles = 4096;
void tgemv_buffers(asb_lane* L) {
    if (L->tg_ws) return;
    L->tg_ws = static_cast<float*>(dmalloc(size_t(kTgMaxUnits) * 32 * 128 * 4, L->allocs));
    L->tg_cnt = static_cast<int*>(dmalloc(size_t(kTgMaxTiles) * 4, L->allocs));
    cuda_check(cudaMemset(L->tg_cnt, 0, size_t(kTgMaxTiles) * 4), "tgemv counters");
}

// Decode (swap) linear on tgemv (TMA ring + warp MMAs) instead of the tcgen05 swap-AB kernel?
// Measured per path, model and partition size (profiles/r2_decode_linear_paths.txt): tgemv
// wins at <= 16 tokens on weights >= 16 MB with K >= 2048 on Green Context partitions
// (1.1-1.6x at 16-64 SMs for the 3B/8B projections) and, on the full device, where the weight
// has enough 128-row tiles for one whole wave (no K split); the tcgen05 kernel keeps 17-32
// tokens (tgemv is MMA-issue bound there: 256 m16n8k16 per 32 KiB stage) and the small 0.5B
// projections.  ASB_NO_TGEMV=1: never (A/B baseline); ASB_TGEMV=1: every T <= 32 linear.
bool use_tgemv(int T, const Weight& w, int num_sms, int epi) {
    static const int mode = std::getenv("ASB_NO_TGEMV") && std::atoi(std::getenv("ASB_NO_TGEMV")) != 0 ? 0
                            : std::getenv("ASB_TGEMV") && std::atoi(std::getenv("ASB_TGEMV")) != 0     ? 2
                                                                                                        : 1;
    if (mode == 0 || T > 32) return false;
    if (mode == 2) return true;
    const double bytes = 2.0 * double(w.rows) * w.cols;
    const int tiles = w.rows_pad / 128;
    if (T <= 16) return bytes >= 16e6 && w.cols >= 2048 && (num_sms <= 120 || tiles * 5 >= num_sms * 4);
    // 17-32 tokens (decode steps carrying an admitted-resume chunk): only the fused QKV projection
    // on a 40-72 SM partition, where the tcgen05 kernel splits its few tiles over clusters
    // (1.17-1.28x there; the other projections stay on tcgen05, profiles/r2_tgemv_17_32.txt)
    return epi == EPI_QKV && bytes >= 16e6 && num_sms >= 40 && num_sms <= 72 && tiles < num_sms;
}

// Y[T][n_out] = X[T][k] . W^T with the path chosen by T (path 2 = dgemv, 3 = tgemv, 1 = tcgen05
// swap-AB, 0 = tcgen05 normal).
void linear(asb_lane* L, const XIn& xin, const Weight& w, int T, int epi,
            __nv_bfloat16* out, int ldo, const __nv_bfloat16* bias, const __nv_bfloat16* resid,
            float* out_f32, int force_path = -1, int force_splits = 0,
            unsigned long long* amax = nullptr, const RopeEpi* rope = nullptr, const PostNorm* post = nullptr) {
    const CUtensorMap* xmaps = xin.maps;
    if (force_path == 2 || (force_path < 0 && use_dgemv(T, w, L->n_sms()))) {
        DgemvParams d{};
        d.w = w.ptr;
        d.rows_pad = w.rows_pad;
        d.x = xin.ptr;
        d.x_rows = xin.rows;
        d.ldx = xin.ld;
        d.T = T;
        d.n_out = w.rows;
        d.K = w.cols;
        d.norm_w = xin.norm_w;
        d.eps = xin.eps;
        d.epi = epi;
        d.out = out;
        d.out_f32 = out_f32;
        d.ldo = ldo;
        d.bias = bias;
        d.resid = resid;
        d.ldr = ldo;
        if (rope) d.rope = *rope;
        d.amax = amax;
        if (post) d.post = *post;
        L->n_launch += 1;
        const double units = 2.0 * (double(w.rows) * w.cols + double(T) * w.cols) +
                             double(T) * w.rows * (epi == EPI_F32 ? 4.0 : 2.0);
        cudaError_t e = cudaSuccess;
        L->timed(ASB_STAT_DECODE_GEMM, units, [&] { e = dgemv_launch(d, L->n_sms(), L->stream); });
        cuda_check(e, "dgemv launch");
        return;
    }
    if (xin.norm_w || xin.rows) fail(ASB_ERR_INVALID_ARGUMENT, "fused norm / row gather needs the dgemv path");
    if (force_path == 3 || (force_path < 0 && use_tgemv(T, w, L->n_sms(), epi))) {
        if (T > 32) fail(ASB_ERR_INVALID_ARGUMENT, "tgemv takes <= 32 tokens");
        tgemv_buffers(L);
        TgemvParams d{};
        d.T = T;
        d.n_out = w.rows;
        d.K = w.cols;
        d.tiles = w.rows_pad / 128;
        d.splits = force_splits;
        d.epi = epi;
        d.out = out;
        d.out_f32 = out_f32;
        d.ldo = ldo;
        d.bias = bias;
        d.resid = resid;
        d.ldr = ldo;
        if (rope) d.rope = *rope;
        d.amax = amax;
        if (post) d.post = *post;
        d.ws = L->tg_ws;
        d.cnt = L->tg_cnt;
        static const bool tg_load_only = std::getenv("ASB_DEBUG_SKIP") &&
                                         std::string(std::getenv("ASB_DEBUG_SKIP")).find("tgmath") != std::string::npos;
        d.dbg_load_only = tg_load_only ? 1 : 0;
        if (d.tiles > kTgMaxTiles || (force_splits > 1 && d.tiles * force_splits > kTgMaxUnits))
            fail(ASB_ERR_INVALID_ARGUMENT, "tgemv: work units exceed the split workspace");
        L->n_launch += 1;
        const double units = 2.0 * (double(w.rows) * w.cols + double(T) * w.cols) +
                             double(T) * w.rows * (epi == EPI_F32 ? 4.0 : 2.0);
        cudaError_t e = cudaSuccess;
        L->timed(ASB_STAT_DECODE_GEMM, units,
                 [&] { e = tgemv_launch(w.map_a128k2, xmaps[T <= 16 ? 7 : 5], d, L->n_sms(), L->stream); });
        cuda_check(e, "tgemv launch");
        return;
    }
    GemmParams p{};
    p.amax = amax;
    if (post) p.post = *post;
    if (rope) p.rope = *rope;
    p.tokens = T;
    p.n_out = w.rows;
    p.K = w.cols;
    p.epi = epi;
    p.out = out;
    p.out_f32 = out_f32;
    p.ldo = ldo;
    p.bias = bias;
    p.resid = resid;
    p.ldr = ldo;
    p.dbg_times = L->dbg_times;
    static const bool no_epi = std::getenv("ASB_GEMM_NO_EPI") != nullptr;  // timing ablation only
    p.dbg_no_epi = no_epi ? 1 : 0;
    static const bool pull = std::getenv("ASB_GEMM_PULL_REDUCE") != nullptr;  // A/B: DSMEM-load reduce
    p.reduce_pull = pull ? 1 : 0;
    const int num_sms = L->n_sms();
    L->n_launch += 1;
    const bool swap = force_path >= 0 ? force_path == 1 : T <= 256;
    cudaError_t e = cudaSuccess;
    // algorithmic work: swap (decode) path is weight-streaming -> bytes; normal -> flops
    const double units = swap ? 2.0 * (double(w.rows) * w.cols + double(T) * w.cols) +
                                    double(T) * w.rows * (epi == EPI_F32 ? 4.0 : 2.0)
                              : 2.0 * T * double(w.rows) * w.cols;
    const bool pdl = tl_pdl;
    L->timed(swap ? ASB_STAT_DECODE_GEMM : ASB_STAT_PREFILL_GEMM, units, [&] {
    if (swap) {
        const int bn = gemm_pick_bn(T);
        p.swap = 1;
        p.a_packed = 1;
        p.w_packed = w.ptr;
        p.w_kblocks = w.cols / 64;
        // L2 prefetch-ahead of the weight stream: measured slower (+5-8% per decode step at
        // 16-148 SMs, profiles/r1_gemm_l2_prefetch_ab.txt), off unless ASB_GEMM_L2PF=<units>
        static const int l2pf = std::getenv("ASB_GEMM_L2PF") ? std::atoi(std::getenv("ASB_GEMM_L2PF")) : 0;
        p.l2_pf = l2pf;
        p.M = w.rows;
        p.N = T;
        const int tiles = (w.rows + 127) / 128;
        // BN <= 64: two k-blocks per pipeline stage (32 KiB weight requests; ASB_GEMM_KP=1 off)
        static const bool kp1 = std::getenv("ASB_GEMM_KP") && std::atoi(std::getenv("ASB_GEMM_KP")) == 1;
        const int kp = (bn <= 64 && !kp1) ? 2 : 1;
        const int kb = ((w.cols + 63) / 64 + kp - 1) / kp;
        // fewer weight tiles than SMs: split K over an S-CTA cluster per tile (DSMEM reduce)
        static const int env_splits = std::getenv("ASB_GEMM_SPLITS") ? std::atoi(std::getenv("ASB_GEMM_SPLITS")) : 0;
        p.splits = gemm_cluster_splits(tiles, kb, bn, num_sms, L->stream, force_splits ? force_splits : env_splits, kp);
        e = kp == 2 ? gemm_launch(w.map_a128k2, xmaps[bn == 32 ? 5 : 6], p, bn, num_sms, L->stream, pdl, 2)
                    : gemm_launch(w.map_a128, xmaps[swap_map_index(bn)], p, bn, num_sms, L->stream, pdl);
    } else {
        p.swap = 0;
        p.b_packed = 1;
        p.M = T;
        p.N = w.rows;
        // BN by wave quantisation: the tile count that fills whole waves of the persistent
        // grid best.  A 128x128 UMMA reads as many operand bytes from smem per flop as the SMEM
        // pipe delivers, so BN = 128 only wins by a wide fill margin at d >= 2048 (3B/7B/8B:
        // 1016-1081 TF/s with it vs 1174-1226 with BN = 256 at C3-C5, profiles/r2_prefill_bn.txt)
        // and by a small one for the 0.5B shapes; ASB_PREFILL_BN forces
        const int tm = (T + 127) / 128;
        const int t256 = tm * ((w.rows + 255) / 256), t128 = tm * ((w.rows + 127) / 128);
        auto fill = [&](int tiles) {
            const int waves = (tiles + num_sms - 1) / num_sms;
            return double(tiles) / (double(waves) * num_sms);
        };
        static const int bn_env = std::getenv("ASB_PREFILL_BN") ? std::atoi(std::getenv("ASB_PREFILL_BN")) : 0;
        const int bn = bn_env == 128 || bn_env == 256 ? bn_env : (fill(t128) * (w.cols <= 1024 ? 0.96 : 0.75) > fill(t256) ? 128 : 256);
        p.splits = 1;
        // normal path: B = W.  bn==128 reuses the box-128 weight map.
        e = gemm_launch(xmaps[0], bn == 256 ? w.map_b256 : w.map_a128, p, bn, num_sms, L->stream, pdl);
    }
    });
    cuda_check(e, "gemm launch");
}

}  // namespace

extern "C" {

const char* asb_last_error(void) { return g_err.c_str(); }

const char* asb_status_name(asb_status s) {
    switch (s) {
    case ASB_OK: return "ok";
    case ASB_ERR_INVALID_ARGUMENT: return "invalid_argument";
    case ASB_ERR_VALIDATION: return "validation_error";
    case ASB_ERR_PROTOCOL: return "protocol_error";
    case ASB_ERR_IO: return "io_error";
    case ASB_ERR_NO_DATA: return "no_data";
    case ASB_ERR_INFEASIBLE: return "infeasible";
    case ASB_ERR_CUDA: return "cuda_error";
    }
    return "unknown";
}

void asb_string_free(char* s) { delete[] s; }

const char* asb_build_info(void) { return "sm_100a;agentserve_b200 r1"; }

asb_status asb_model_create(const char* model, uint64_t seed, int device, int max_context,
                            asb_model** out) {
    if (!model || !out) {
        g_err = "null argument";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        ModelSpec s = parse_spec(model);
        validate_spec(s);
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= device)
            fail(ASB_ERR_CUDA, "no CUDA device " + std::to_string(device));
        cuda_check(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
        if (prop.major != 10)
            fail(ASB_ERR_CUDA, std::string("device is not sm_100 (") + prop.name + ")");
        auto m = std::make_unique<asb_model>();
        m->spec = s;
        m->device = device;
        m->num_sms = prop.multiProcessorCount;
        m->seed = seed;
        m->max_ctx = max_context > 0 ? max_context : 16384;
        auto mk = [&](int rows, int cols) {
            Weight w;
            w.rows = rows;
            w.rows_pad = (rows + 127) / 128 * 128;
            w.cols = cols;
            w.ptr = static_cast<__nv_bfloat16*>(dmalloc(size_t(w.rows_pad) * cols * 2, m->allocs));
            cuda_check(cudaMemset(w.ptr, 0, size_t(w.rows_pad) * cols * 2), "memset weight");
            return w;
        };
        auto vec = [&](int n) {
            return static_cast<__nv_bfloat16*>(dmalloc(size_t(n) * 2, m->allocs));
        };
        const int qd = s.hq * s.hd, kvd = s.hkv * s.hd;
        m->embed = mk(s.vocab, s.d);
        fillw(m.get(), m->embed, "embed", s.vocab, 1, 0);
        weight_maps(m->embed);
        if (s.tied) {
            m->lm_head = m->embed;
        } else {
            m->lm_head = mk(s.vocab, s.d);
            fillw(m.get(), m->lm_head, "lm_head", s.vocab, 1, 0);
            weight_maps(m->lm_head);
        }
        m->final_norm = vec(s.d);
        fill(m.get(), m->final_norm, "final_norm", 1, s.d, 1, 0, 1.f, kAmpN);
        for (int l = 0; l < s.layers; ++l) {
            asb_model::Layer ly{};
            const std::string p = "L" + std::to_string(l) + "/";
            ly.attn_norm = vec(s.d);
            fill(m.get(), ly.attn_norm, p + "attn_norm", 1, s.d, 1, 0, 1.f, kAmpN);
            ly.mlp_norm = vec(s.d);
            fill(m.get(), ly.mlp_norm, p + "mlp_norm", 1, s.d, 1, 0, 1.f, kAmpN);
            ly.qkv = mk(qd + 2 * kvd, s.d);
            fillw(m.get(), ly.qkv, p + "q", qd, 1, 0);
            fillw(m.get(), ly.qkv, p + "k", kvd, 1, qd);
            fillw(m.get(), ly.qkv, p + "v", kvd, 1, qd + kvd);
            weight_maps(ly.qkv);
            ly.qkv_bias = nullptr;
            if (s.qkv_bias) {
                ly.qkv_bias = vec(qd + 2 * kvd);
                fill(m.get(), ly.qkv_bias, p + "q_bias", 1, qd, 1, 0, 0.f, kAmpB);
                fill(m.get(), ly.qkv_bias + qd, p + "k_bias", 1, kvd, 1, 0, 0.f, kAmpB);
                fill(m.get(), ly.qkv_bias + qd + kvd, p + "v_bias", 1, kvd, 1, 0, 0.f, kAmpB);
            }
            ly.o = mk(s.d, qd);
            fillw(m.get(), ly.o, p + "o", s.d, 1, 0);
            weight_maps(ly.o);
            // gate/up interleaved: row 2j = gate_j, row 2j+1 = up_j (SiLU·mul epilogue pairs)
            ly.gate_up = mk(2 * s.ffn, s.d);
            fillw(m.get(), ly.gate_up, p + "gate", s.ffn, 2, 0);
            fillw(m.get(), ly.gate_up, p + "up", s.ffn, 2, 1);
            weight_maps(ly.gate_up);
            ly.down = mk(s.d, s.ffn);
            fillw(m.get(), ly.down, p + "down", s.d, 1, 0);
            weight_maps(ly.down);
            m->layers.push_back(ly);
        }
        // RoPE tables
        const int half = s.hd / 2;
        std::vector<double> inv = rope_inv_freq(s);
        std::vector<float> c(size_t(m->max_ctx) * half), sn(size_t(m->max_ctx) * half);
        for (int pos = 0; pos < m->max_ctx; ++pos)
            for (int i = 0; i < half; ++i) {
                const double a = pos * inv[i];
                c[size_t(pos) * half + i] = static_cast<float>(std::cos(a));
                sn[size_t(pos) * half + i] = static_cast<float>(std::sin(a));
            }
        m->cos_t = static_cast<float*>(dmalloc(c.size() * 4, m->allocs));
        m->sin_t = static_cast<float*>(dmalloc(sn.size() * 4, m->allocs));
        cuda_check(cudaMemcpy(m->cos_t, c.data(), c.size() * 4, cudaMemcpyHostToDevice), "copy rope");
        cuda_check(cudaMemcpy(m->sin_t, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice), "copy rope");
        cuda_check(cudaDeviceSynchronize(), "weight init");
        *out = m.release();
    });
}

asb_status asb_model_describe(const asb_model* m, char** out_json) {
    if (!m || !out_json) {
        g_err = "null argument";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        const ModelSpec& s = m->spec;
        json j = {{"name", s.name},       {"layers", s.layers},     {"d_model", s.d},
                  {"n_heads", s.hq},      {"n_kv_heads", s.hkv},    {"head_dim", s.hd},
                  {"ffn", s.ffn},         {"vocab", s.vocab},       {"tied", s.tied},
                  {"qkv_bias", s.qkv_bias}, {"rope_theta", s.theta}, {"rms_eps", s.eps},
                  {"rope_llama3", s.rope_llama3}, {"rope_factor", s.rope_factor},
                  {"rope_lo", s.rope_lo}, {"rope_hi", s.rope_hi}, {"rope_orig", s.rope_orig},
                  {"seed", m->seed},      {"num_sms", m->num_sms},  {"max_context", m->max_ctx},
                  {"block_tokens", kBlockTokens}};
        const std::string t = j.dump();
        char* o = new char[t.size() + 1];
        std::memcpy(o, t.c_str(), t.size() + 1);
        *out_json = o;
    });
}

void asb_model_free(asb_model* m) { delete m; }

int asb_kv_block_tokens(void) { return kBlockTokens; }

asb_status asb_kv_create(asb_model* m, int num_blocks, asb_kv** out) {
    if (!m || !out || num_blocks < 1) {
        g_err = "invalid argument";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        cuda_check(cudaSetDevice(m->device), "cudaSetDevice");
        auto kv = std::make_unique<asb_kv>();
        kv->m = m;
        kv->nb = num_blocks;
        const ModelSpec& s = m->spec;
        const size_t pages = size_t(s.layers) * num_blocks * s.hkv;
        const size_t elems = pages * kKvPageRows * s.hd;
        cuda_check(cudaMalloc(&kv->pool, elems * 2), "cudaMalloc KV pool");
        // zeroed so that masked tail rows of a partial block are finite
        cuda_check(cudaMemset(kv->pool, 0, elems * 2), "memset");
        kv->k_pool = kv->pool;
        kv->v_pool = kv->pool + size_t(kBlockTokens) * s.hd;
        const long rows = long(pages) * kKvPageRows;
        if (rows >= (1l << 31)) fail(ASB_ERR_VALIDATION, "KV pool too large for 32-bit TMA rows");
        // [64 rows][64 cols] boxes of the K pages (row = page*128 + t on the k_pool view) and the
        // V pages (the same row index on the v_pool view, one page further) for prefill
        // attention; one box per whole block, K and V together, for decode attention
        if (!make_tmap_bf16(&kv->tk, kv->k_pool, int(rows), s.hd, s.hd, kBlockTokens) ||
            !make_tmap_bf16(&kv->tv, kv->v_pool, int(rows - kBlockTokens), s.hd, s.hd, kBlockTokens) ||
            !make_tmap_kv_sub(&kv->tkv, kv->pool, long(pages), s.hd, kBlockTokens, kBlockTokens))
            fail(ASB_ERR_CUDA, "cuTensorMapEncodeTiled failed for the KV pool");
        kv->free_list.reserve(num_blocks);
        for (int b = num_blocks - 1; b >= 0; --b) kv->free_list.push_back(b);
        cuda_check(cudaDeviceSynchronize(), "kv init");
        *out = kv.release();
    });
}

void asb_kv_free(asb_kv* kv) { delete kv; }

int asb_kv_free_blocks(const asb_kv* kv) { return kv ? int(kv->free_list.size()) : -1; }

asb_status asb_kv_begin_write(asb_kv* kv, uint32_t session) {
    if (!kv) return ASB_ERR_INVALID_ARGUMENT;
    kv->get(session).sealed = false;
    return ASB_OK;
}

asb_status asb_kv_commit(asb_kv* kv, uint32_t session, int new_prefix) {
    if (!kv) return ASB_ERR_INVALID_ARGUMENT;
    return guarded([&] {
        auto& s = kv->get(session);
        if (new_prefix < s.prefix)
            fail(ASB_ERR_PROTOCOL, "kv commit shrinks session " + std::to_string(session) +
                                       " prefix from " + std::to_string(s.prefix) + " to " +
                                       std::to_string(new_prefix));
        s.prefix = new_prefix;
        s.sealed = true;
    });
}

asb_status asb_kv_append(asb_kv* kv, uint32_t session, int tokens) {
    if (!kv) return ASB_ERR_INVALID_ARGUMENT;
    return guarded([&] {
        auto& s = kv->get(session);
        if (!s.sealed)
            fail(ASB_ERR_PROTOCOL, "decode append on unsealed KV entry for session " +
                                       std::to_string(session));
        s.prefix += tokens;
    });
}

int asb_kv_sealed(const asb_kv* kv, uint32_t session) {
    if (!kv) return 0;
    auto it = kv->sess.find(session);
    return it != kv->sess.end() && it->second.sealed ? 1 : 0;
}

asb_status asb_kv_require_sealed(const asb_kv* kv, uint32_t session) {
    if (!kv) return ASB_ERR_INVALID_ARGUMENT;
    if (!asb_kv_sealed(kv, session)) {
        g_err = "decode step on unsealed KV entry for session " + std::to_string(session);
        return ASB_ERR_PROTOCOL;
    }
    return ASB_OK;
}

int asb_kv_prefix(const asb_kv* kv, uint32_t session) {
    if (!kv) return -1;
    auto it = kv->sess.find(session);
    return it == kv->sess.end() ? 0 : it->second.prefix;
}

int asb_kv_length(const asb_kv* kv, uint32_t session) {
    if (!kv) return -1;
    auto it = kv->sess.find(session);
    return it == kv->sess.end() ? 0 : it->second.len;
}

asb_status asb_kv_block_table(const asb_kv* kv, uint32_t session, int32_t* out, int cap, int* n) {
    if (!kv || !n) return ASB_ERR_INVALID_ARGUMENT;
    auto it = kv->sess.find(session);
    const int cnt = it == kv->sess.end() ? 0 : int(it->second.blocks.size());
    *n = cnt;
    if (out)
        for (int i = 0; i < std::min(cap, cnt); ++i) out[i] = it->second.blocks[i];
    return ASB_OK;
}

asb_status asb_kv_release(asb_kv* kv, uint32_t session) {
    if (!kv) return ASB_ERR_INVALID_ARGUMENT;
    auto it = kv->sess.find(session);
    if (it == kv->sess.end()) return ASB_OK;
    // return blocks in reverse so a re-allocation hands them out in the same order
    for (auto b = it->second.blocks.rbegin(); b != it->second.blocks.rend(); ++b)
        kv->free_list.push_back(*b);
    kv->sess.erase(it);
    return ASB_OK;
}

asb_status asb_kv_read_token(const asb_kv* kv, uint32_t session, int position, uint16_t* k_out,
                             uint16_t* v_out) {
    if (!kv || !k_out || !v_out) return ASB_ERR_INVALID_ARGUMENT;
    return guarded([&] {
        auto it = kv->sess.find(session);
        if (it == kv->sess.end() || position < 0 || position >= it->second.len)
            fail(ASB_ERR_INVALID_ARGUMENT, "position not written for session");
        const ModelSpec& s = kv->m->spec;
        const int blk = it->second.blocks[position / kBlockTokens];
        const int off = position % kBlockTokens;
        cuda_check(cudaSetDevice(kv->m->device), "cudaSetDevice");
        for (int l = 0; l < s.layers; ++l)
            for (int h = 0; h < s.hkv; ++h) {
                const size_t src =
                    (((size_t(l) * kv->nb + blk) * s.hkv + h) * kKvPageRows + off) * s.hd;
                const size_t dst = (size_t(l) * s.hkv + h) * s.hd;
                cuda_check(cudaMemcpy(k_out + dst, kv->k_pool + src, s.hd * 2, cudaMemcpyDeviceToHost), "copy");
                cuda_check(cudaMemcpy(v_out + dst, kv->v_pool + src, s.hd * 2, cudaMemcpyDeviceToHost), "copy");
            }
    });
}

asb_status asb_lane_create(asb_model* m, int max_tokens, int max_segments, void* stream,
                           asb_lane** out) {
    if (!m || !out || max_tokens < 1 || max_segments < 1) {
        g_err = "invalid argument";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        cuda_check(cudaSetDevice(m->device), "cudaSetDevice");
        auto L = std::make_unique<asb_lane>();
        L->m = m;
        const ModelSpec& s = m->spec;
        L->max_T = max_tokens;
        // the fused last-arriver merge sums at most 16 split partials (decode_attn.cu): clamp
        if (const char* e = std::getenv("ASB_DECODE_MAX_SPLITS")) L->max_splits = std::min(16, std::max(1, std::atoi(e)));
        L->max_segs = std::min(max_segments, max_tokens);
        L->max_tbl = L->max_segs * ((m->max_ctx + kBlockTokens - 1) / kBlockTokens);
        L->max_pitems = max_tokens / prefill_tokens_per_tile(s.hq, s.hkv) + L->max_segs;
        if (stream) {
            L->stream = static_cast<cudaStream_t>(stream);
        } else {
            cuda_check(cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking), "stream");
            L->own_stream = true;
        }
        const int T = max_tokens;
        const int qd = s.hq * s.hd, kvd = s.hkv * s.hd;
        auto bf = [&](size_t n) { return static_cast<__nv_bfloat16*>(dmalloc(n * 2, L->allocs)); };
        L->x = bf(size_t(T) * s.d);
        L->h = bf(size_t(T) * s.d);
        L->qkv = bf(size_t(T) * (qd + 2 * kvd));
        L->q = bf(size_t(T) * qd);
        L->attn = bf(size_t(T) * qd);
        L->act = bf(size_t(T) * s.ffn);
        L->hl = bf(size_t(L->max_segs) * s.d);
        L->logits = static_cast<float*>(dmalloc(size_t(L->max_segs) * s.vocab * 4, L->allocs));
        if (std::getenv("ASB_GEMM_TIMELINE"))
            L->dbg_times = static_cast<unsigned long long*>(dmalloc(148 * 8 * 8, L->allocs));
        // decode-attention items: one per single-token row, ceil(n * G / 8) per short segment (the
        // admitted resume chunk of a decode step, its tokens' columns packed 8 per item); split
        // partials per (item, kv head, column)
        L->max_ditems = std::min(T, L->max_segs + 32);
        const int dec_rows = L->max_ditems;
        L->part_o = static_cast<float*>(
            dmalloc(size_t(dec_rows) * s.hkv * 8 * L->max_splits * s.hd * 4, L->allocs));
        L->part_ml = static_cast<float*>(
            dmalloc(size_t(dec_rows) * s.hkv * 8 * L->max_splits * 2 * 4, L->allocs));
        L->dcnt = static_cast<int*>(dmalloc(size_t(dec_rows) * s.hkv * 4, L->allocs));
        L->post_cnt = static_cast<int*>(dmalloc(64, L->allocs));
        tgemv_buffers(L.get());
        cuda_check(cudaMemset(L->post_cnt, 0, 64), "counters");
        cuda_check(cudaMemset(L->dcnt, 0, size_t(dec_rows) * s.hkv * 4), "counters");
        {
            if (std::getenv("ASB_ATTN_TIMELINE")) {
                L->attn_dbg = static_cast<unsigned long long*>(dmalloc(1024 * 8 * 8, L->allocs));
                cuda_check(cudaMemset(L->attn_dbg, 0, 1024 * 8 * 8), "attn dbg");
            }
        }
        // split-KV partials for small prefill grids (resume chunks): <= 4096 rows of 128 queries
        L->ppart_rows = size_t(4096) * 256 / 4;
        L->ppart_o = static_cast<float*>(dmalloc(L->ppart_rows * s.hd * 4, L->allocs));
        L->ppart_ml = static_cast<float*>(dmalloc(L->ppart_rows * 2 * 4, L->allocs));
        L->meta_ints = size_t(3) * T + L->max_segs + L->max_tbl + kDItemInts * size_t(L->max_ditems) +
                       4 * size_t(L->max_pitems) + 64 +
                       4 * (size_t(L->max_pitems) + 512) + 4;  // prefill work units + combine list
        L->d_meta = static_cast<int32_t*>(dmalloc(L->meta_ints * 4, L->allocs));
        cuda_check(cudaMallocHost(&L->h_meta, L->meta_ints * 4), "cudaMallocHost");
        L->d_out = static_cast<unsigned long long*>(dmalloc(size_t(L->max_segs) * 8, L->allocs));
        cuda_check(cudaMallocHost(&L->h_out, size_t(L->max_segs) * 8), "cudaMallocHost");
        act_maps(L->map_h, L->h, T, s.d);
        act_maps(L->map_x, L->x, T, s.d);
        act_maps(L->map_attn, L->attn, T, qd);
        act_maps(L->map_act, L->act, T, s.ffn);
        act_maps(L->map_hl, L->hl, L->max_segs, s.d);
        {
            const int G = s.hq / s.hkv;
            if (!make_tmap_bf16_3d(&L->map_q, L->q, s.hd, s.hq, T, G, prefill_tokens_per_tile(s.hq, s.hkv)))
                fail(ASB_ERR_CUDA, "cuTensorMapEncodeTiled failed for q");
        }
        cuda_check(cudaEventCreate(&L->ev0), "event");
        cuda_check(cudaEventCreate(&L->ev1), "event");
        cuda_check(cudaDeviceSynchronize(), "lane init");
        *out = L.release();
    });
}

void asb_lane_free(asb_lane* lane) { delete lane; }

// Rebind without draining: the lane's in-flight forward (if any) keeps running on the old
// partition; the new stream is ordered after it by an event (device-side wait, no host
// block), so the lane's next launch still sees its previous one complete.  Cost: one event
// record + one stream wait, a few microseconds ("< 50 us per rebinding").
asb_status asb_lane_set_stream(asb_lane* lane, void* stream) {
    if (!lane || !stream) return ASB_ERR_INVALID_ARGUMENT;
    cudaStream_t ns = static_cast<cudaStream_t>(stream);
    if (ns == lane->stream) return ASB_OK;
    return guarded([&] {
        if (lane->launched) {
            if (!lane->ev_switch)
                cuda_check(cudaEventCreateWithFlags(&lane->ev_switch, cudaEventDisableTiming), "event");
            cuda_check(cudaEventRecord(lane->ev_switch, lane->stream), "rebind record");
            cuda_check(cudaStreamWaitEvent(ns, lane->ev_switch, 0), "rebind wait");
        }
        if (lane->own_stream) {
            // an owned stream is only replaced once; its pending work completes asynchronously
            cuda_check(cudaStreamDestroy(lane->stream), "stream destroy");
        }
        lane->own_stream = false;
        lane->stream = ns;
    });
}

void* asb_lane_stream(const asb_lane* lane) { return lane ? lane->stream : nullptr; }

int asb_lane_query(const asb_lane* lane) {
    if (!lane || !lane->launched) return 1;
    return cudaEventQuery(lane->ev1) == cudaSuccess ? 1 : 0;
}

asb_status asb_lane_wait(asb_lane* lane) {
    if (!lane) return ASB_ERR_INVALID_ARGUMENT;
    if (!lane->launched) return ASB_OK;
    return guarded([&] { cuda_check(cudaEventSynchronize(lane->ev1), "lane wait"); });
}

float asb_lane_last_ms(const asb_lane* lane) {
    if (!lane || !lane->launched) return -1.f;
    float ms = -1.f;
    if (cudaEventElapsedTime(&ms, lane->ev0, lane->ev1) != cudaSuccess) return -1.f;
    return ms;
}

asb_status asb_forward(asb_lane* L, asb_kv* kv, const asb_segment* segs, int n_segs,
                       const int32_t* tokens) {
    if (!L || !kv || !segs || !tokens || n_segs < 1) {
        g_err = "invalid argument";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        asb_model* m = L->m;
        const ModelSpec& s = m->spec;
        if (kv->m != m) fail(ASB_ERR_INVALID_ARGUMENT, "kv belongs to another model");
        if (n_segs > L->max_segs) fail(ASB_ERR_INVALID_ARGUMENT, "too many segments for lane");
        int T = 0;
        for (int i = 0; i < n_segs; ++i) {
            if (segs[i].n_tokens < 1) fail(ASB_ERR_INVALID_ARGUMENT, "segment with no tokens");
            T += segs[i].n_tokens;
        }
        if (T > L->max_T) fail(ASB_ERR_INVALID_ARGUMENT, "batch exceeds lane max_tokens");
        cuda_check(cudaSetDevice(m->device), "cudaSetDevice");
        // previous launch must be done before the pinned staging is reused
        if (L->launched) cuda_check(cudaEventSynchronize(L->ev1), "lane reuse");

        // ---- host metadata ------------------------------------------------------------
        int32_t* hm = L->h_meta;
        int32_t* h_tok = hm;
        int32_t* h_pos = h_tok + T;
        int32_t* h_slot = h_pos + T;
        int32_t* h_lrows = h_slot + T;
        int n_logit = 0;
        std::vector<int32_t> tbl;
        std::vector<DecodeItem> ditems;
        double dattn_seg_bytes = 0.0;  // algorithmic decode-attention bytes: each session's K/V once
        std::vector<PrefillItem> pitems;
        int max_ctx = 0, max_pblocks = 0;
        int row = 0;
        // Validate and size every segment before touching the registry: a failure (context
        // limit, pool exhaustion, table overflow) leaves every length, block list and the
        // free list exactly as they were.
        {
            std::map<uint32_t, int> grow;  // session -> tokens this call appends
            int64_t tbl_need = 0, blocks_need = 0;
            for (int i = 0; i < n_segs; ++i) {
                const auto it = kv->sess.find(segs[i].session);
                const int len0 = it == kv->sess.end() ? 0 : it->second.len;
                const int start = len0 + grow[segs[i].session];
                if (start + segs[i].n_tokens > m->max_ctx)
                    fail(ASB_ERR_INFEASIBLE, "session " + std::to_string(segs[i].session) +
                                                  " exceeds max_context");
                grow[segs[i].session] += segs[i].n_tokens;
                tbl_need += (start + segs[i].n_tokens + kBlockTokens - 1) / kBlockTokens;
            }
            if (tbl_need > L->max_tbl) fail(ASB_ERR_INVALID_ARGUMENT, "block tables exceed lane");
            for (const auto& [sid, n] : grow) {
                const auto it = kv->sess.find(sid);
                const int len0 = it == kv->sess.end() ? 0 : it->second.len;
                const int have = it == kv->sess.end() ? 0 : int(it->second.blocks.size());
                blocks_need += std::max(0, (len0 + n + kBlockTokens - 1) / kBlockTokens - have);
            }
            if (blocks_need > int64_t(kv->free_list.size()))
                fail(ASB_ERR_INFEASIBLE, "KV pool exhausted (" + std::to_string(kv->nb) + " blocks)");
        }
        for (int i = 0; i < n_segs; ++i) {
            const asb_segment& g = segs[i];
            auto& ss = kv->get(g.session);
            const int start = ss.len;
            kv->ensure(ss, start + g.n_tokens);  // cannot fail: sized above
            const int toff = int(tbl.size());
            tbl.insert(tbl.end(), ss.blocks.begin(), ss.blocks.end());
            for (int t = 0; t < g.n_tokens; ++t) {
                const int p = start + t;
                h_tok[row + t] = tokens[row + t];
                h_pos[row + t] = p;
                h_slot[row + t] = ss.blocks[p / kBlockTokens] * kBlockTokens + p % kBlockTokens;
            }
            // A short segment (<= kChunkAsDecode tokens: the admitted resume chunk riding in a
            // decode step) goes through the decode-attention kernel as a token group: token t
            // attends keys 0..start+t (its causal prefix), and its (token, head) columns are
            // packed 8 per item, so each K/V block is read once per 8 columns instead of a
            // small, latency-bound prefill-attention launch (+ combine) per layer.
            // DecodeItem.pad = the first position this forward writes for the row's session:
            // blocks from there on are read only after the QKV kernel (PDL wait).
            // ASB_CHUNK_AS_DECODE=0: chunks through prefill attention; =2: one item per token
            // (the unpacked form, for the ablation).
            static const int chunk_dec = std::getenv("ASB_CHUNK_AS_DECODE")
                                             ? std::atoi(std::getenv("ASB_CHUNK_AS_DECODE")) : 1;
            constexpr int kChunkAsDecode = 16;
            const int G = s.hq / s.hkv;
            const int n_dit = chunk_dec == 2 ? g.n_tokens : (g.n_tokens * G + 7) / 8;
            if (g.n_tokens == 1 || (chunk_dec && g.n_tokens <= kChunkAsDecode &&
                                    int(ditems.size()) + n_dit <= L->max_ditems)) {
                if (chunk_dec == 2) {
                    for (int t = 0; t < g.n_tokens; ++t)
                        ditems.push_back(DecodeItem{row + t, start + t + 1, toff, start, 0, G});
                } else {
                    for (int c0 = 0; c0 < g.n_tokens * G; c0 += 8)
                        ditems.push_back(DecodeItem{row, start + 1, toff, start, c0, g.n_tokens * G});
                }
                max_ctx = std::max(max_ctx, start + g.n_tokens);
                dattn_seg_bytes += double(start + g.n_tokens) * s.hkv * s.hd * 2 * 2;  // K/V read once per session
            } else {
                const int tpt = prefill_tokens_per_cta(s.hq, s.hkv);
                for (int q0 = 0; q0 < g.n_tokens; q0 += tpt)
                    pitems.push_back(PrefillItem{row + q0, start + q0, std::min(tpt, g.n_tokens - q0), toff});
                max_pblocks = std::max(max_pblocks, (start + g.n_tokens + kBlockTokens - 1) / kBlockTokens);
            }
            if (g.want_logits) h_lrows[n_logit++] = row + g.n_tokens - 1;
            ss.len = start + g.n_tokens;
            row += g.n_tokens;
        }
        if (int(tbl.size()) > L->max_tbl) fail(ASB_ERR_INVALID_ARGUMENT, "block tables exceed lane");
        int32_t* h_tbl = h_lrows + L->max_segs;
        std::memcpy(h_tbl, tbl.data(), tbl.size() * 4);
        int32_t* h_ditems = h_tbl + L->max_tbl;
        std::memcpy(h_ditems, ditems.data(), ditems.size() * sizeof(DecodeItem));
        int32_t* h_pitems = h_ditems + kDItemInts * L->max_ditems;
        std::memcpy(h_pitems, pitems.data(), pitems.size() * sizeof(PrefillItem));
        // prefill work units (one wave, long causal items split; ASB_PREFILL_UNITS=0 off), int4-aligned
        static const bool units_off = std::getenv("ASB_PREFILL_UNITS") && std::atoi(std::getenv("ASB_PREFILL_UNITS")) == 0;
        static const bool psplit_forced = std::getenv("ASB_PREFILL_SPLITS") != nullptr;
        std::vector<int4> punits, pcomb;
        if (!units_off && !psplit_forced && !pitems.empty())
            prefill_units(pitems.data(), int(pitems.size()), s.hkv, L->n_sms(), L->ppart_rows, punits, pcomb);
        const size_t units_off_ints = (size_t(h_pitems - hm) + 4 * pitems.size() + 3) & ~size_t(3);
        std::memcpy(hm + units_off_ints, punits.data(), punits.size() * sizeof(int4));
        std::memcpy(hm + units_off_ints + 4 * punits.size(), pcomb.data(), pcomb.size() * sizeof(int4));
        const size_t used = units_off_ints + 4 * (punits.size() + pcomb.size());

        cudaStream_t st = L->stream;
        // ASB_GRAPH_PROBE=1 (measurement only): capture this forward -- meta H2D, every kernel,
        // ids D2H -- into a CUDA graph and replay it, so ev0..ev1 times the graph-launched step
        // against the stream-launched one (capture + instantiate happen before ev0).
        static const bool graph_probe = std::getenv("ASB_GRAPH_PROBE") && std::atoi(std::getenv("ASB_GRAPH_PROBE")) == 1;
        const bool capture = graph_probe && !L->prof && !L->attn_dbg;
        if (capture) cuda_check(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "graph capture");
        else cuda_check(cudaEventRecord(L->ev0, st), "event");
        cuda_check(cudaMemcpyAsync(L->d_meta, hm, used * 4, cudaMemcpyHostToDevice, st), "meta H2D");
        L->h2d += int64_t(used) * 4;
        const int32_t* d_tok = L->d_meta;
        const int32_t* d_pos = d_tok + T;
        const int32_t* d_slot = d_pos + T;
        const int32_t* d_lrows = d_slot + T;
        const int32_t* d_tbl = d_lrows + L->max_segs;
        const DecodeItem* d_ditems = reinterpret_cast<const DecodeItem*>(d_tbl + L->max_tbl);
        const PrefillItem* d_pitems =
            reinterpret_cast<const PrefillItem*>(d_tbl + L->max_tbl + kDItemInts * L->max_ditems);
        const int4* d_units = reinterpret_cast<const int4*>(L->d_meta + units_off_ints);
        const int4* d_comb = d_units + punits.size();

        // ---- forward -----------------------------------------------------------------------
        const int qd = s.hq * s.hd, kvd = s.hkv * s.hd;
        AttnShape as{};
        as.hq = s.hq;
        as.hkv = s.hkv;
        as.hd = s.hd;
        as.num_blocks = kv->nb;
        as.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(double(s.hd)));
        {
            static const bool load_only = std::getenv("ASB_DEBUG_SKIP") &&
                                          std::string(std::getenv("ASB_DEBUG_SKIP")).find("attnmath") != std::string::npos;
            as.dbg_load_only = load_only ? 1 : 0;
            static const bool no_prewait = std::getenv("ASB_ATTN_PREWAIT") && std::atoi(std::getenv("ASB_ATTN_PREWAIT")) == 0;
            as.no_prewait = no_prewait ? 1 : 0;
        }
        if (L->attn_dbg) {
            cuda_check(cudaMemsetAsync(L->attn_dbg, 0, 1024 * 8 * 8, L->stream), "attn dbg");
            as.dbg = L->attn_dbg;
        }
        // algorithmic work per layer: decode attention streams every context token's K and V
        // once; prefill attention is 4*hd flops per (query, key<=query) pair per head.
        double dattn_bytes = 0.0, pattn_flops = 0.0;
        static const int psplit_env = std::getenv("ASB_PREFILL_SPLITS") ? std::atoi(std::getenv("ASB_PREFILL_SPLITS")) : 0;
        int psplits = pitems.empty() ? 1
                                     : prefill_splits(int(pitems.size()), s.hkv, max_pblocks, L->n_sms(), L->ppart_rows);
        if (psplit_env > 0 && !pitems.empty())  // timing experiments: force the split count
            psplits = std::max(1, std::min({psplit_env, 32, int(L->ppart_rows / (pitems.size() * s.hkv * 256))}));
        dattn_bytes = dattn_seg_bytes;
        for (const auto& it : pitems)
            pattn_flops += 4.0 * s.hd * s.hq *
                           (double(it.n_q) * it.q_pos0 + double(it.n_q) * (it.n_q + 1) / 2.0);
        if (L->prof && !L->marks.empty()) L->resolve_marks();
        cudaEvent_t fwd_a = L->prof ? L->take_event() : nullptr;
        if (fwd_a) cuda_check(cudaEventRecord(fwd_a, st), "event");
        PdlScope pdl_scope(L->pdl && !L->prof);
        {
            // the fused QKV epilogue needs q/k/v regions aligned to the 128-row weight tiles
            // ASB_DEBUG_SKIP=attn,norm,...: timing ablation only (outputs are garbage)
            static const std::string skip_list = std::getenv("ASB_DEBUG_SKIP") ? std::getenv("ASB_DEBUG_SKIP") : "";
            auto skip = [&](const char* what) {
                return !skip_list.empty() && ("," + skip_list + ",").find("," + std::string(what) + ",") != std::string::npos;
            };
            const bool fuse_qkv = (qd % 128 == 0) && (kvd % 128 == 0) && (s.hd == 64 || s.hd == 128) &&
                                  std::getenv("ASB_NO_QKV_FUSION") == nullptr;
            // Small batches (decode steps) take the dgemv path where it wins; its QKV / gate-up /
            // LM-head launches apply the preceding RMSNorm themselves (no norm launch).
            const bool dg_qkv = use_dgemv(T, m->layers[0].qkv, L->n_sms()),
                       dg_gu = use_dgemv(T, m->layers[0].gate_up, L->n_sms());
            const bool dg_lm = n_logit > 0 && use_dgemv(n_logit, m->lm_head, L->n_sms());
            // Pre-norms of tcgen05 linears: layer 0's in the embedding kernel; on small decode
            // batches the others in the residual GEMM before them (its last CTA normalises the
            // updated rows, PostNorm) -- no separate norm launches.
            // (one CTA normalises all T rows: worth a launch only while T x d is small -- at
            // Llama-3.1-8B B=64 it costs 3.5 ms per step; Qwen2.5-0.5B B=2: -1%)
            const bool post_ok = int64_t(T) * s.d <= 16 * 1024 && std::getenv("ASB_NO_POST_NORM") == nullptr;
            const bool post_attn = !dg_qkv && post_ok, post_mlp = !dg_gu && post_ok;
            const bool post_final = n_logit > 0 && !dg_lm && n_logit <= 256 && post_ok;
            cuda_check(embed(d_tok, m->embed.ptr, L->x, T, s.d, st, dg_lm ? L->d_out : nullptr, n_logit,
                             dg_qkv ? nullptr : m->layers[0].attn_norm, L->h, s.eps),
                       "embed");
            // non-GEMM kernels of this forward (linear() counts its own launches): embed; per layer
            // the unfused norms, the unfused RoPE/append, decode attention (split merge fused) and
            // prefill attention (+ its split combine); final norm and argmax when not fused
            L->n_launch += 1 + int64_t(s.layers - 1) * ((dg_qkv || post_attn) ? 0 : 1) +
                           int64_t(s.layers) * ((dg_gu || post_mlp ? 0 : 1) + (fuse_qkv ? 0 : 1) +
                                                (ditems.empty() ? 0 : 1) + (pitems.empty() ? 0
                                                 : !punits.empty() ? (pcomb.empty() ? 1 : 2)
                                                                   : (psplits > 1 ? 2 : 1)));
            if (n_logit > 0 && !dg_lm) L->n_launch += (post_final ? 0 : 1) + (n_logit <= 256 ? 0 : 1);
            PostNorm pn_attn{}, pn_mlp{}, pn_final{};
            if (post_mlp || post_attn || post_final) {
                pn_attn = PostNorm{nullptr, L->h, nullptr, T, s.d, s.eps, L->post_cnt, nullptr};
                pn_mlp = pn_attn;
                pn_final = PostNorm{m->final_norm, L->hl, d_lrows, n_logit, s.d, s.eps, L->post_cnt, L->d_out};
            }
            const XIn x_attn{L->map_attn, L->attn, qd};
            const XIn x_act{L->map_act, L->act, s.ffn};
            for (int l = 0; l < s.layers; ++l) {
                const auto& ly = m->layers[l];
                as.layer = l;
                const XIn xa = dg_qkv ? XIn{nullptr, L->x, s.d, ly.attn_norm, nullptr, s.eps}
                                      : XIn{L->map_h, L->h, s.d};
                const XIn xm = dg_gu ? XIn{nullptr, L->x, s.d, ly.mlp_norm, nullptr, s.eps}
                                     : XIn{L->map_h, L->h, s.d};
                if (!dg_qkv && l > 0 && !post_attn && !skip("norm"))
                    cuda_check(rmsnorm(L->x, nullptr, ly.attn_norm, L->h, T, s.d, s.eps, st), "rmsnorm");
                if (skip("qkv")) {
                } else if (fuse_qkv) {
                    // QKV GEMM with bias, RoPE and the paged K/V append fused into its epilogue
                    RopeEpi re{d_pos, d_slot, m->cos_t, m->sin_t, L->q, kv->k_pool, kv->v_pool,
                               s.hq, s.hkv, s.hd, l, kv->nb};
                    linear(L, xa, ly.qkv, T, EPI_QKV, nullptr, qd + 2 * kvd, ly.qkv_bias, nullptr, nullptr,
                           -1, 0, nullptr, &re);
                } else {
                    linear(L, xa, ly.qkv, T, EPI_BF16, L->qkv, qd + 2 * kvd, ly.qkv_bias, nullptr, nullptr);
                    cuda_check(rope_append(L->qkv, d_pos, d_slot, m->cos_t, m->sin_t, L->q, kv->k_pool,
                                           kv->v_pool, T, s.hq, s.hkv, s.hd, l, kv->nb, st),
                               "rope_append");
                }
                if (!ditems.empty() && !skip("attn"))
                    L->timed(ASB_STAT_DECODE_ATTN, dattn_bytes, [&] {
                        cuda_check(decode_attention(kv->tkv, L->q, d_ditems, int(ditems.size()),
                                                    max_ctx, d_tbl, L->attn, L->part_o, L->part_ml,
                                                    L->dcnt, L->max_splits, L->n_sms(), as, st),
                                   "decode attention");
                    });
                if (!pitems.empty())
                    L->timed(ASB_STAT_PREFILL_ATTN, pattn_flops, [&] {
                        if (!punits.empty())
                            cuda_check(prefill_attention_units(L->map_q, kv->tk, kv->tv, d_pitems, d_units,
                                                               int(punits.size()), d_comb, int(pcomb.size()), d_tbl,
                                                               L->attn, L->ppart_o, L->ppart_ml, as, st),
                                       "prefill attention (units)");
                        else
                            cuda_check(prefill_attention(L->map_q, kv->tk, kv->tv, d_pitems, int(pitems.size()),
                                                         max_pblocks, psplits, d_tbl, L->attn, L->ppart_o,
                                                         L->ppart_ml, as, st),
                                       "prefill attention");
                    });
                pn_mlp.w = post_mlp ? ly.mlp_norm : nullptr;
                if (!skip("o"))
                    linear(L, x_attn, ly.o, T, EPI_RESID, L->x, s.d, nullptr, L->x, nullptr, -1, 0, nullptr, nullptr,
                           post_mlp ? &pn_mlp : nullptr);
                if (!dg_gu && !post_mlp && !skip("norm"))
                    cuda_check(rmsnorm(L->x, nullptr, ly.mlp_norm, L->h, T, s.d, s.eps, st), "rmsnorm");
                if (!skip("gate_up")) linear(L, xm, ly.gate_up, T, EPI_SILU, L->act, s.ffn, nullptr, nullptr, nullptr);
                // the residual GEMM closing the layer prepares the next pre-norm (next layer's
                // attention norm, or the final norm of the LM-head rows after the last layer)
                const bool last = l + 1 == s.layers;
                const PostNorm* pn = nullptr;
                if (!last && post_attn) {
                    pn_attn.w = m->layers[l + 1].attn_norm;
                    pn = &pn_attn;
                } else if (last && post_final) {
                    pn = &pn_final;
                }
                if (!skip("down"))
                    linear(L, x_act, ly.down, T, EPI_RESID, L->x, s.d, nullptr, L->x, nullptr, -1, 0, nullptr, nullptr, pn);
            }
            if (n_logit > 0) {
                // greedy sample fused into the LM head epilogue (<= 256 rows): the argmax keys are
                // zeroed by the final norm (or, on the dgemv path, by the embedding kernel, and the
                // LM head normalises and gathers its rows itself); the GEMM atomicMax-es into them
                const bool fused_argmax = n_logit <= 256;
                if (dg_lm) {
                    XIn xl{nullptr, L->x, s.d, m->final_norm, d_lrows, s.eps};
                    linear(L, xl, m->lm_head, n_logit, EPI_F32, nullptr, s.vocab, nullptr, nullptr, L->logits, -1, 0,
                           L->d_out);
                } else {
                    if (!post_final)
                        cuda_check(rmsnorm(L->x, d_lrows, m->final_norm, L->hl, n_logit, s.d, s.eps, st,
                                           fused_argmax ? L->d_out : nullptr), "final norm");
                    linear(L, XIn{L->map_hl, L->hl, s.d}, m->lm_head, n_logit, EPI_F32, nullptr, s.vocab, nullptr,
                           nullptr, L->logits, -1, 0, fused_argmax ? L->d_out : nullptr);
                    if (!fused_argmax)
                        cuda_check(argmax_rows(L->logits, n_logit, s.vocab, s.vocab, L->d_out, st), "argmax");
                }
                cuda_check(cudaMemcpyAsync(L->h_out, L->d_out, n_logit * 8, cudaMemcpyDeviceToHost, st),
                           "ids D2H");
                L->d2h += int64_t(n_logit) * 8;
            }
        }
        if (fwd_a) {
            cudaEvent_t fwd_b = L->take_event();
            cuda_check(cudaEventRecord(fwd_b, st), "event");
            L->marks.push_back(asb_lane::Mark{fwd_a, fwd_b, ASB_STAT_FORWARD, double(T)});
        }
        if (capture) {
            cudaGraph_t g = nullptr;
            cudaGraphExec_t ge = nullptr;
            cuda_check(cudaStreamEndCapture(st, &g), "graph end capture");
            cuda_check(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
            cuda_check(cudaEventRecord(L->ev0, st), "event");
            cuda_check(cudaGraphLaunch(ge, st), "graph launch");
            cuda_check(cudaGraphExecDestroy(ge), "graph destroy");  // deferred until the launch completes
            cuda_check(cudaGraphDestroy(g), "graph destroy");
        }
        cuda_check(cudaEventRecord(L->ev1, st), "event");
        L->launched = true;
        L->last_logit_rows = n_logit;
    });
}

static unsigned long long g_timeline[148 * 8];

asb_status asb_debug_gemm_timeline(asb_lane* L, unsigned long long* out, int n) {
    if (!out) return ASB_ERR_INVALID_ARGUMENT;
    if (!L) {  // last asb_debug_gemm call
        std::memcpy(out, g_timeline, size_t(std::min(n, 148 * 8)) * 8);
        return ASB_OK;
    }
    if (!L->dbg_times) return ASB_ERR_INVALID_ARGUMENT;
    return guarded([&] {
        cuda_check(cudaStreamSynchronize(L->stream), "timeline");
        cuda_check(cudaMemcpy(out, L->dbg_times, size_t(std::min(n, 148 * 8)) * 8, cudaMemcpyDeviceToHost), "timeline");
    });
}

asb_status asb_debug_attn_timeline(asb_lane* L, unsigned long long* out, int n) {
    if (!L || !out) return ASB_ERR_INVALID_ARGUMENT;
    return guarded([&] {
        if (!L->attn_dbg) fail(ASB_ERR_NO_DATA, "lane created without ASB_ATTN_TIMELINE=1");
        cuda_check(cudaStreamSynchronize(L->stream), "sync");
        cuda_check(cudaMemcpy(out, L->attn_dbg, std::min<size_t>(1024 * 8, size_t(n)) * 8, cudaMemcpyDeviceToHost),
                   "timeline");
    });
}

asb_status asb_lane_set_sms(asb_lane* L, int sms) {
    if (!L || sms < 0) return ASB_ERR_INVALID_ARGUMENT;
    L->sms = sms;
    return ASB_OK;
}

asb_status asb_lane_counters(asb_lane* L, int64_t* launches, int64_t* h2d_bytes, int64_t* d2h_bytes,
                             int reset) {
    if (!L) return ASB_ERR_INVALID_ARGUMENT;
    if (launches) *launches = L->n_launch;
    if (h2d_bytes) *h2d_bytes = L->h2d;
    if (d2h_bytes) *d2h_bytes = L->d2h;
    if (reset) L->n_launch = L->h2d = L->d2h = 0;
    return ASB_OK;
}

asb_status asb_lane_profile(asb_lane* L, int enable) {
    if (!L) return ASB_ERR_INVALID_ARGUMENT;
    L->prof = enable != 0;
    return ASB_OK;
}

asb_status asb_lane_stats(asb_lane* L, int cat, double* ms, double* units, int64_t* launches,
                          int reset) {
    if (!L || cat < 0 || cat >= ASB_STAT_COUNT) return ASB_ERR_INVALID_ARGUMENT;
    return guarded([&] {
        if (L->launched) cuda_check(cudaEventSynchronize(L->ev1), "lane stats");
        L->resolve_marks();
        if (ms) *ms = L->st_ms[cat];
        if (units) *units = L->st_units[cat];
        if (launches) *launches = L->st_n[cat];
        if (reset) {
            L->st_ms[cat] = 0.0;
            L->st_units[cat] = 0.0;
            L->st_n[cat] = 0;
        }
    });
}

asb_status asb_lane_fetch(asb_lane* L, int32_t* out_next, int n, float* out_logits) {
    if (!L) return ASB_ERR_INVALID_ARGUMENT;
    return guarded([&] {
        if (!L->launched) fail(ASB_ERR_NO_DATA, "nothing launched on this lane");
        cuda_check(cudaEventSynchronize(L->ev1), "lane fetch");
        if (n > L->last_logit_rows) fail(ASB_ERR_INVALID_ARGUMENT, "more ids requested than produced");
        if (out_next)
            for (int i = 0; i < n; ++i) out_next[i] = argmax_key_index(L->h_out[i]);
        if (out_logits)
            cuda_check(cudaMemcpy(out_logits, L->logits, size_t(n) * L->m->spec.vocab * 4,
                                  cudaMemcpyDeviceToHost),
                       "logits D2H");
    });
}

asb_status asb_prefill_launch(asb_lane* lane, asb_kv* kv, uint32_t session, const int32_t* tokens,
                              int n) {
    asb_segment g{session, n, 1};
    return asb_forward(lane, kv, &g, 1, tokens);
}

asb_status asb_decode_launch(asb_lane* lane, asb_kv* kv, const uint32_t* sessions,
                             const int32_t* in_tokens, int batch, int64_t chunk_session,
                             const int32_t* chunk_tokens, int chunk_n) {
    std::vector<asb_segment> segs;
    std::vector<int32_t> toks;
    for (int i = 0; i < batch; ++i) {
        segs.push_back(asb_segment{sessions[i], 1, 1});
        toks.push_back(in_tokens[i]);
    }
    if (chunk_session >= 0 && chunk_n > 0) {
        segs.push_back(asb_segment{static_cast<uint32_t>(chunk_session), chunk_n, 1});
        toks.insert(toks.end(), chunk_tokens, chunk_tokens + chunk_n);
    }
    if (segs.empty()) {
        g_err = "decode step needs at least one stream or an admitted chunk";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    return asb_forward(lane, kv, segs.data(), int(segs.size()), toks.data());
}

// Back-to-back timing of one linear layer: weights packed once into enough copies to exceed
// L2 (cycled, so each launch streams from HBM as in a real step); `reps` launches with PDL,
// bracketed by CUDA events: average microseconds per launch.  num_sms = 0: all.
asb_status asb_debug_gemm_bench(const void* x, const void* w, void* out, int tokens, int n_out, int k,
                                int epi, int force_path, int reps, int num_sms, void* stream,
                                float* us_per_launch) {
    if (!us_per_launch || reps < 1) {
        g_err = "invalid argument";
        return ASB_ERR_INVALID_ARGUMENT;
    }
    return guarded([&] {
        // enough packed copies to exceed the 126 MB L2, cycled, so every launch streams from HBM
        const size_t wbytes = size_t((n_out + 127) / 128 * 128) * k * 2;
        const int copies = int(std::min<size_t>(256, (size_t(320) << 20) / wbytes + 1));
        std::vector<Weight> Ws(copies);
        for (auto& W : Ws) {
            W.rows = n_out;
            W.rows_pad = (n_out + 127) / 128 * 128;
            W.cols = k;
            cuda_check(cudaMalloc(&W.ptr, wbytes), "packed w");
            cuda_check(cudaMemset(W.ptr, 0, wbytes), "packed w");
            cuda_check(pack_weights(static_cast<const __nv_bfloat16*>(w), W.ptr, n_out, k, nullptr), "pack");
            weight_maps(W);
        }
        CUtensorMap xm[8];
        act_maps(xm, x, tokens, k);
        asb_model fake;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, dev), "props");
        fake.device = dev;
        fake.num_sms = num_sms > 0 ? num_sms : prop.multiProcessorCount;
        asb_lane tmp;
        tmp.m = &fake;
        if (stream) tmp.stream = static_cast<cudaStream_t>(stream);
        else cuda_check(cudaStreamCreateWithFlags(&tmp.stream, cudaStreamNonBlocking), "stream");
        const int ldo = epi == EPI_SILU ? n_out / 2 : n_out;
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        auto run = [&](int n) {
            PdlScope pdl(true);
            for (int i = 0; i < n; ++i)
                linear(&tmp, XIn{xm, static_cast<const __nv_bfloat16*>(x), k}, Ws[i % copies], tokens, epi,
                       static_cast<__nv_bfloat16*>(out), ldo, nullptr,
                       epi == EPI_RESID ? static_cast<const __nv_bfloat16*>(out) : nullptr,
                       epi == EPI_F32 ? static_cast<float*>(out) : nullptr, force_path, 0);
        };
        run(3);
        cuda_check(cudaEventRecord(e0, tmp.stream), "event");
        run(reps);
        cuda_check(cudaEventRecord(e1, tmp.stream), "event");
        cuda_check(cudaEventSynchronize(e1), "bench sync");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        *us_per_launch = 1000.f * ms / reps;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        if (!stream) cudaStreamDestroy(tmp.stream);
        tmp.stream = nullptr;
        for (auto& W : Ws) cudaFree(W.ptr);
        tmp.m = &fake;
    });
}

asb_status asb_debug_gemm(const void* x, const void* w, const void* bias, const void* resid,
                          void* out, int tokens, int n_out, int k, int epi, int force_path,
                          int splits, void* stream) {
    return guarded([&] {
        Weight W;
        W.rows = n_out;
        W.rows_pad = (n_out + 127) / 128 * 128;
        W.cols = k;
        cuda_check(cudaMalloc(&W.ptr, size_t(W.rows_pad) * k * 2), "packed w");
        cuda_check(cudaMemset(W.ptr, 0, size_t(W.rows_pad) * k * 2), "packed w");
        cuda_check(pack_weights(static_cast<const __nv_bfloat16*>(w), W.ptr, n_out, k,
                                static_cast<cudaStream_t>(stream)), "pack");
        weight_maps(W);
        CUtensorMap xm[8];
        act_maps(xm, x, tokens, k);
        asb_lane tmp;  // only stream and sms are used by linear()
        asb_model fake;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceProp prop;
        cuda_check(cudaGetDeviceProperties(&prop, dev), "props");
        fake.device = dev;
        fake.num_sms = prop.multiProcessorCount;
        tmp.m = &fake;
        tmp.stream = static_cast<cudaStream_t>(stream);
        const int ldo = epi == EPI_SILU ? n_out / 2 : n_out;
        if (std::getenv("ASB_GEMM_TIMELINE")) {
            cuda_check(cudaMalloc(&tmp.dbg_times, 148 * 8 * 8), "timeline");
            cuda_check(cudaMemset(tmp.dbg_times, 0, 148 * 8 * 8), "timeline");
        }
        linear(&tmp, XIn{xm, static_cast<const __nv_bfloat16*>(x), k}, W, tokens, epi,
               static_cast<__nv_bfloat16*>(out), ldo,
               static_cast<const __nv_bfloat16*>(bias), static_cast<const __nv_bfloat16*>(resid),
               epi == EPI_F32 ? static_cast<float*>(out) : nullptr, force_path, splits);
        cuda_check(cudaStreamSynchronize(tmp.stream), "debug gemm");
        if (tmp.dbg_times) {
            cuda_check(cudaMemcpy(g_timeline, tmp.dbg_times, sizeof(g_timeline), cudaMemcpyDeviceToHost), "timeline");
            cudaFree(tmp.dbg_times);
            tmp.dbg_times = nullptr;
        }
        cudaFree(W.ptr);
        tmp.allocs.clear();
        fake.allocs.clear();
        tmp.m = &fake;
        tmp.stream = nullptr;
        tmp.launched = false;
    });
}

}  // extern "C"
