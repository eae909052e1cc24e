/*
 * CPU fp32 forward oracle for the AgentServe SLM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs as the checker; never linked into or called by the
 * product (paper_2603_10342_b200/libagentserve_b200.so).
 *
 * PARITY STATUS: the reference (/root/reference/proj, agentsim) contains NO forward pass:
 * SPEC.md:9 lists "actual model inference and KV tensors" as out of scope and the simulator
 * replaces the forward with decode_step_duration_ms (src/executor.cpp:84-97) and a prefill
 * rate (src/engine.cpp:450-475).  The paper's real system extended llama.cpp,
 * which is not vendored and has no pinned version.  Logits / greedy ids / KV VALUES are
 * therefore "parity unpinned" against the reference: this file restates public Llama-3 /
 * Qwen2 decoder math (RMSNorm, RoPE rotate_half, GQA causal softmax attention, SwiGLU, tied
 * or untied LM head, greedy argmax with lowest index on ties) at the same bf16 rounding
 * points as the device path.  What IS pinned to the reference: the splitmix64 named
 * sub-stream generator used for weights and token ids (src/rng.hpp:14-60, restated below and
 * checked against the compiled reference in tests), and — through oracle/_ref — every
 * scheduling decision and KV prefix length.  The decoder math itself is pinned to an
 * independent public implementation instead: tests/test_oracle_pin_hf.py runs these weights
 * (fo_tensor) through transformers 5.5.0's Llama / Qwen2 modelling code in fp32 and bounds
 * the logit difference at 1% (measured 0.3-0.5%; a wrong RoPE theta, Llama-3 frequency
 * scaling or KV-head grouping exceeds it).
 *
 * Numerics contract (identical on device):
 *   x0 = embed[tok]                                   (bf16)
 *   h  = bf16(x * (1/sqrt(mean(x^2) + eps)) * w)      (fp32 math, one rounding)
 *   qkv= bf16(h . W^T + b)
 *   q,k= bf16(rotate_half RoPE with fp32 cos/sin table built in double)
 *   attn = bf16(softmax(q.k^T / sqrt(hd)) . v)        (fp32 softmax)
 *   x  = bf16(x + attn . Wo^T)
 *   a  = bf16(silu(h2 . Wg^T) * (h2 . Wu^T))          (gate/up never rounded)
 *   x  = bf16(x + a . Wd^T)
 *   logits = rmsnorm(x_last) . Wlm^T (fp32); next = argmax (lowest index on ties)
 * Weights: element i of tensor <name> = bf16(offset + t * (amp / 2^23)),
 *   t = (int)(splitmix64 draw i+1 of substream(seed, name) >> 40) - 2^23.
 */
#include "forward.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define KAMP_W 0.034641016f
#define KAMP_B 0.1f
#define KAMP_N 0.1f

static uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

static uint64_t fnv1a(const char* s) {
    uint64_t h = 0xcbf29ce484222325ull;
    for (; *s; ++s) {
        h ^= (unsigned char)*s;
        h *= 0x00000100000001b3ull;
    }
    return h;
}

uint64_t fo_substream(uint64_t seed, const char* name) { return mix64(seed ^ fnv1a(name)); }

uint64_t fo_next_u64(uint64_t* state) {
    *state += 0x9e3779b97f4a7c15ull;
    return mix64(*state);
}

uint64_t fo_uniform_int(uint64_t* state, uint64_t n) {
    return (uint64_t)(((__uint128_t)fo_next_u64(state) * n) >> 64);
}

static inline float bf16r(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u) {
        u &= 0xffff0000u;
    } else {
        u += 0x7fffu + ((u >> 16) & 1u);
        u &= 0xffff0000u;
    }
    memcpy(&f, &u, 4);
    return f;
}

static inline uint16_t bf16bits(float f) {
    uint32_t u;
    f = bf16r(f);
    memcpy(&u, &f, 4);
    return (uint16_t)(u >> 16);
}

static float gen_value(uint64_t state0, int64_t i, float offset, float amp_scaled) {
    uint64_t u = mix64(state0 + (uint64_t)(i + 1) * 0x9e3779b97f4a7c15ull);
    int32_t t = (int32_t)(u >> 40) - 8388608;
    volatile float prod = (float)t * amp_scaled; /* no FMA contraction */
    return bf16r(offset + prod);
}

uint16_t fo_weight_bits(uint64_t seed, const char* name, int64_t index, float offset, float amp) {
    return bf16bits(gen_value(fo_substream(seed, name), index, offset, amp * (1.0f / 8388608.0f)));
}

static float* gen_tensor(uint64_t seed, const char* name, int64_t n, float offset, float amp) {
    float* p = (float*)malloc((size_t)n * sizeof(float));
    uint64_t s0 = fo_substream(seed, name);
    float a = amp * (1.0f / 8388608.0f);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) p[i] = gen_value(s0, i, offset, a);
    return p;
}

typedef struct {
    float *attn_norm, *mlp_norm, *wq, *wk, *wv, *bq, *bk, *bv, *wo, *wg, *wu, *wd;
} fo_layer;

struct fo_model {
    fo_spec s;
    int n_layers; /* may be truncated for large shapes (stated by the caller) */
    int max_ctx;
    float *embed, *lm_head, *final_norm;
    fo_layer* layers;
    float *cos_t, *sin_t;
};

struct fo_session {
    int len;
    float* k; /* [layer][pos][hkv][hd] */
    float* v;
    int cap;
};

fo_model* fo_create(const fo_spec* spec, uint64_t seed, int max_ctx, int n_layers_limit) {
    fo_model* m = (fo_model*)calloc(1, sizeof(fo_model));
    m->s = *spec;
    m->n_layers = (n_layers_limit > 0 && n_layers_limit < spec->layers) ? n_layers_limit : spec->layers;
    m->max_ctx = max_ctx;
    const fo_spec* s = spec;
    const int qd = s->hq * s->hd, kvd = s->hkv * s->hd;
    char name[64];
    m->embed = gen_tensor(seed, "embed", (int64_t)s->vocab * s->d, 0.f, KAMP_W);
    m->lm_head = s->tied ? m->embed : gen_tensor(seed, "lm_head", (int64_t)s->vocab * s->d, 0.f, KAMP_W);
    m->final_norm = gen_tensor(seed, "final_norm", s->d, 1.f, KAMP_N);
    m->layers = (fo_layer*)calloc((size_t)m->n_layers, sizeof(fo_layer));
    for (int l = 0; l < m->n_layers; ++l) {
        fo_layer* L = &m->layers[l];
#define G(field, nm, n, off, amp)                      \
    snprintf(name, sizeof name, "L%d/%s", l, nm);      \
    L->field = gen_tensor(seed, name, (int64_t)(n), off, amp);
        G(attn_norm, "attn_norm", s->d, 1.f, KAMP_N);
        G(mlp_norm, "mlp_norm", s->d, 1.f, KAMP_N);
        G(wq, "q", (int64_t)qd * s->d, 0.f, KAMP_W);
        G(wk, "k", (int64_t)kvd * s->d, 0.f, KAMP_W);
        G(wv, "v", (int64_t)kvd * s->d, 0.f, KAMP_W);
        if (s->qkv_bias) {
            G(bq, "q_bias", qd, 0.f, KAMP_B);
            G(bk, "k_bias", kvd, 0.f, KAMP_B);
            G(bv, "v_bias", kvd, 0.f, KAMP_B);
        }
        G(wo, "o", (int64_t)s->d * qd, 0.f, KAMP_W);
        G(wg, "gate", (int64_t)s->ffn * s->d, 0.f, KAMP_W);
        G(wu, "up", (int64_t)s->ffn * s->d, 0.f, KAMP_W);
        G(wd, "down", (int64_t)s->d * s->ffn, 0.f, KAMP_W);
#undef G
    }
    /* RoPE table: double math, float storage (same formula as the device runtime) */
    const int half = s->hd / 2;
    double* inv = (double*)malloc(sizeof(double) * half);
    for (int i = 0; i < half; ++i) {
        double f = 1.0 / pow(s->theta, (2.0 * i) / s->hd);
        if (s->rope_llama3) {
            const double lo_wl = s->rope_orig / s->rope_lo, hi_wl = s->rope_orig / s->rope_hi;
            const double wl = 2.0 * M_PI / f;
            if (wl > lo_wl) {
                f = f / s->rope_factor;
            } else if (wl >= hi_wl) {
                const double smooth = (s->rope_orig / wl - s->rope_lo) / (s->rope_hi - s->rope_lo);
                f = (1.0 - smooth) * f / s->rope_factor + smooth * f;
            }
        }
        inv[i] = f;
    }
    m->cos_t = (float*)malloc(sizeof(float) * (size_t)max_ctx * half);
    m->sin_t = (float*)malloc(sizeof(float) * (size_t)max_ctx * half);
    for (int p = 0; p < max_ctx; ++p)
        for (int i = 0; i < half; ++i) {
            const double a = p * inv[i];
            m->cos_t[(size_t)p * half + i] = (float)cos(a);
            m->sin_t[(size_t)p * half + i] = (float)sin(a);
        }
    free(inv);
    return m;
}

void fo_free(fo_model* m) {
    if (!m) return;
    for (int l = 0; l < m->n_layers; ++l) {
        fo_layer* L = &m->layers[l];
        free(L->attn_norm); free(L->mlp_norm); free(L->wq); free(L->wk); free(L->wv);
        free(L->bq); free(L->bk); free(L->bv); free(L->wo); free(L->wg); free(L->wu); free(L->wd);
    }
    free(m->layers);
    if (!m->s.tied) free(m->lm_head);
    free(m->embed);
    free(m->final_norm);
    free(m->cos_t);
    free(m->sin_t);
    free(m);
}

const float* fo_tensor(const fo_model* m, int layer, const char* name, int64_t* n) {
    const fo_spec* s = &m->s;
    const int64_t qd = (int64_t)s->hq * s->hd, kvd = (int64_t)s->hkv * s->hd, d = s->d, f = s->ffn;
    if (!strcmp(name, "embed")) { *n = (int64_t)s->vocab * d; return m->embed; }
    if (!strcmp(name, "lm_head")) { *n = (int64_t)s->vocab * d; return m->lm_head; }
    if (!strcmp(name, "final_norm")) { *n = d; return m->final_norm; }
    if (layer < 0 || layer >= m->n_layers) return NULL;
    const fo_layer* L = &m->layers[layer];
    if (!strcmp(name, "attn_norm")) { *n = d; return L->attn_norm; }
    if (!strcmp(name, "mlp_norm")) { *n = d; return L->mlp_norm; }
    if (!strcmp(name, "q")) { *n = qd * d; return L->wq; }
    if (!strcmp(name, "k")) { *n = kvd * d; return L->wk; }
    if (!strcmp(name, "v")) { *n = kvd * d; return L->wv; }
    if (!strcmp(name, "q_bias")) { *n = qd; return L->bq; }
    if (!strcmp(name, "k_bias")) { *n = kvd; return L->bk; }
    if (!strcmp(name, "v_bias")) { *n = kvd; return L->bv; }
    if (!strcmp(name, "o")) { *n = d * qd; return L->wo; }
    if (!strcmp(name, "gate")) { *n = f * d; return L->wg; }
    if (!strcmp(name, "up")) { *n = f * d; return L->wu; }
    if (!strcmp(name, "down")) { *n = d * f; return L->wd; }
    return NULL;
}

fo_session* fo_session_new(fo_model* m) {
    fo_session* s = (fo_session*)calloc(1, sizeof(fo_session));
    s->cap = m->max_ctx;
    const size_t n = (size_t)m->n_layers * m->max_ctx * m->s.hkv * m->s.hd;
    s->k = (float*)calloc(n, sizeof(float));
    s->v = (float*)calloc(n, sizeof(float));
    return s;
}

void fo_session_free(fo_session* s) {
    if (!s) return;
    free(s->k);
    free(s->v);
    free(s);
}

int fo_session_len(const fo_session* s) { return s->len; }

static void rmsnorm_rows(const float* x, const float* w, float* y, int n, int d, float eps) {
#pragma omp parallel for schedule(static)
    for (int r = 0; r < n; ++r) {
        const float* xr = x + (size_t)r * d;
        float ss = 0.f;
        for (int i = 0; i < d; ++i) ss += xr[i] * xr[i];
        const float inv = 1.0f / sqrtf(ss / (float)d + eps);
        for (int i = 0; i < d; ++i) {
            volatile float a = xr[i] * inv;
            y[(size_t)r * d + i] = bf16r(a * w[i]);
        }
    }
}

/* y[r][o] = sum_k x[r][k] * W[o][k]  (fp32 accumulation; the k-sum is vectorised, so its
 * association order is the SIMD reduction's, not left-to-right -- a difference of a few fp32
 * ulps, far below the bf16 rounding applied to every output).  Blocks of 16 weight rows stay
 * in L2 while all activation rows stream past them. */
static void matmul(const float* x, const float* W, float* y, int n, int k, int o) {
    const int JB = 16;
#pragma omp parallel for schedule(dynamic)
    for (int jb = 0; jb < o; jb += JB) {
        const int je = jb + JB < o ? jb + JB : o;
        for (int r = 0; r < n; ++r) {
            const float* xr = x + (size_t)r * k;
            for (int j = jb; j < je; ++j) {
                const float* wr = W + (size_t)j * k;
                float acc = 0.f;
#pragma omp simd reduction(+ : acc)
                for (int i = 0; i < k; ++i) acc += xr[i] * wr[i];
                y[(size_t)r * o + j] = acc;
            }
        }
    }
}

int fo_forward(fo_model* m, fo_session* S, const int32_t* tokens, int n, float* logits_out) {
    const fo_spec* s = &m->s;
    const int d = s->d, qd = s->hq * s->hd, kvd = s->hkv * s->hd, hd = s->hd, half = hd / 2;
    const int G = s->hq / s->hkv;
    const int start = S->len;
    float* x = (float*)malloc(sizeof(float) * (size_t)n * d);
    float* h = (float*)malloc(sizeof(float) * (size_t)n * d);
    float* q = (float*)malloc(sizeof(float) * (size_t)n * qd);
    float* kk = (float*)malloc(sizeof(float) * (size_t)n * kvd);
    float* vv = (float*)malloc(sizeof(float) * (size_t)n * kvd);
    float* at = (float*)malloc(sizeof(float) * (size_t)n * qd);
    float* t1 = (float*)malloc(sizeof(float) * (size_t)n * (d > s->ffn ? d : s->ffn));
    float* g = (float*)malloc(sizeof(float) * (size_t)n * s->ffn);
    float* u = (float*)malloc(sizeof(float) * (size_t)n * s->ffn);
    for (int r = 0; r < n; ++r) memcpy(x + (size_t)r * d, m->embed + (size_t)tokens[r] * d, sizeof(float) * d);
    const float scale = (float)(1.0 / sqrt((double)hd));
    for (int l = 0; l < m->n_layers; ++l) {
        const fo_layer* L = &m->layers[l];
        rmsnorm_rows(x, L->attn_norm, h, n, d, s->eps);
        matmul(h, L->wq, q, n, d, qd);
        matmul(h, L->wk, kk, n, d, kvd);
        matmul(h, L->wv, vv, n, d, kvd);
        for (int r = 0; r < n; ++r) {
            for (int i = 0; i < qd; ++i) q[(size_t)r * qd + i] = bf16r(q[(size_t)r * qd + i] + (s->qkv_bias ? L->bq[i] : 0.f));
            for (int i = 0; i < kvd; ++i) {
                kk[(size_t)r * kvd + i] = bf16r(kk[(size_t)r * kvd + i] + (s->qkv_bias ? L->bk[i] : 0.f));
                vv[(size_t)r * kvd + i] = bf16r(vv[(size_t)r * kvd + i] + (s->qkv_bias ? L->bv[i] : 0.f));
            }
            const int pos = start + r;
            const float* ct = m->cos_t + (size_t)pos * half;
            const float* st = m->sin_t + (size_t)pos * half;
            for (int hh = 0; hh < s->hq + s->hkv; ++hh) {
                float* v = hh < s->hq ? q + (size_t)r * qd + hh * hd : kk + (size_t)r * kvd + (hh - s->hq) * hd;
                for (int j = 0; j < half; ++j) {
                    const float x1 = v[j], x2 = v[j + half];
                    volatile float a = x1 * ct[j], b = x2 * st[j], c = x2 * ct[j], e = x1 * st[j];
                    v[j] = bf16r(a - b);
                    v[j + half] = bf16r(c + e);
                }
            }
            float* kdst = S->k + (((size_t)l * m->max_ctx + pos) * kvd);
            float* vdst = S->v + (((size_t)l * m->max_ctx + pos) * kvd);
            memcpy(kdst, kk + (size_t)r * kvd, sizeof(float) * kvd);
            memcpy(vdst, vv + (size_t)r * kvd, sizeof(float) * kvd);
        }
        /* causal attention over the session cache */
#pragma omp parallel for collapse(2) schedule(dynamic)
        for (int r = 0; r < n; ++r) {
            for (int hh = 0; hh < s->hq; ++hh) {
                const int kvh = hh / G;
                const int ctx = start + r + 1;
                const float* qr = q + (size_t)r * qd + hh * hd;
                float* sc = (float*)malloc(sizeof(float) * ctx);
                float mx = -INFINITY;
                for (int t = 0; t < ctx; ++t) {
                    const float* kr = S->k + (((size_t)l * m->max_ctx + t) * kvd) + kvh * hd;
                    float a = 0.f;
                    for (int i = 0; i < hd; ++i) a += qr[i] * kr[i];
                    sc[t] = a * scale;
                    if (sc[t] > mx) mx = sc[t];
                }
                float sum = 0.f;
                for (int t = 0; t < ctx; ++t) {
                    sc[t] = expf(sc[t] - mx);
                    sum += sc[t];
                }
                float* o = at + (size_t)r * qd + hh * hd;
                for (int i = 0; i < hd; ++i) o[i] = 0.f;
                for (int t = 0; t < ctx; ++t) {
                    const float* vr = S->v + (((size_t)l * m->max_ctx + t) * kvd) + kvh * hd;
                    const float p = sc[t] / sum;
                    for (int i = 0; i < hd; ++i) o[i] += p * vr[i];
                }
                for (int i = 0; i < hd; ++i) o[i] = bf16r(o[i]);
                free(sc);
            }
        }
        matmul(at, L->wo, t1, n, qd, d);
        for (size_t i = 0; i < (size_t)n * d; ++i) x[i] = bf16r(x[i] + t1[i]);
        rmsnorm_rows(x, L->mlp_norm, h, n, d, s->eps);
        matmul(h, L->wg, g, n, d, s->ffn);
        matmul(h, L->wu, u, n, d, s->ffn);
        for (size_t i = 0; i < (size_t)n * s->ffn; ++i) {
            const float gg = g[i];
            volatile float sl = gg / (1.0f + expf(-gg));
            g[i] = bf16r(sl * u[i]);
        }
        matmul(g, L->wd, t1, n, s->ffn, d);
        for (size_t i = 0; i < (size_t)n * d; ++i) x[i] = bf16r(x[i] + t1[i]);
    }
    S->len = start + n;
    /* logits of the last row */
    float* hl = (float*)malloc(sizeof(float) * d);
    rmsnorm_rows(x + (size_t)(n - 1) * d, m->final_norm, hl, 1, d, s->eps);
    float* lg = logits_out ? logits_out : (float*)malloc(sizeof(float) * s->vocab);
    matmul(hl, m->lm_head, lg, 1, d, s->vocab);
    int best = 0;
    for (int i = 1; i < s->vocab; ++i)
        if (lg[i] > lg[best]) best = i;
    if (!logits_out) free(lg);
    free(hl); free(x); free(h); free(q); free(kk); free(vv); free(at); free(t1); free(g); free(u);
    return best;
}

void fo_read_kv(const fo_model* m, const fo_session* S, int pos, uint16_t* k_out, uint16_t* v_out) {
    const int kvd = m->s.hkv * m->s.hd;
    for (int l = 0; l < m->n_layers; ++l) {
        const float* kr = S->k + (((size_t)l * m->max_ctx + pos) * kvd);
        const float* vr = S->v + (((size_t)l * m->max_ctx + pos) * kvd);
        for (int i = 0; i < kvd; ++i) {
            k_out[(size_t)l * kvd + i] = bf16bits(kr[i]);
            v_out[(size_t)l * kvd + i] = bf16bits(vr[i]);
        }
    }
}
