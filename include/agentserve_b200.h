/*
 * agentserve_b200 — device seam of the AgentServe serving hot path on B200 (sm_100a).
 *
 * The reference (AgentServe's agentsim, /root/reference/proj) stands the SLM forward pass
 * in with a throughput model at three C++ seams; each asb_* entry point below replaces one:
 *
 *   asb_kv_*        <- KvCacheRegistry::{begin_write,commit,append_decode_tokens,
 *                      require_sealed,prefix}      (/root/reference/proj/src/executor.hpp:47-71)
 *                      plus the device paged KV pool it now owns (block tables, append).
 *   asb_forward /
 *   asb_decode_launch <- decode_step_duration_ms   (/root/reference/proj/src/executor.hpp:76-77,
 *                      executor.cpp:84-97): one continuous-batching decode step, B single-token
 *                      rows + <= resume_chunk_tokens rows of an admitted resume
 *                      (engine.cpp:295-339).
 *   asb_prefill_launch <- prefill rate x length     (/root/reference/proj/src/engine.cpp:442-477).
 *   asb_slots_*     <- SlotSet::{select_slot,rebind} (/root/reference/proj/src/executor.hpp:20-42):
 *                      pre-created CUDA Green Context SM partitions with per-partition streams.
 *
 * Conventions mirror agentsim.h: status returns, thread-local asb_last_error(), opaque
 * single-owner handles, caller-owned buffers, no exceptions across the ABI, heap strings
 * freed with asb_string_free.  Launches are asynchronous on the lane's stream; completion
 * is observed with asb_lane_query / asb_lane_wait, results read with asb_lane_fetch.
 * There is no CPU fallback: on a host without a usable sm_100 device every device call
 * fails with ASB_ERR_CUDA.
 */
#ifndef AGENTSERVE_B200_H
#define AGENTSERVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef enum asb_status {
    ASB_OK = 0,
    ASB_ERR_INVALID_ARGUMENT = 1,
    ASB_ERR_VALIDATION = 2,
    ASB_ERR_PROTOCOL = 3, /* KV read-only-handoff violations, as AGSV_ERR_PROTOCOL */
    ASB_ERR_IO = 4,
    ASB_ERR_NO_DATA = 5,
    ASB_ERR_INFEASIBLE = 6, /* e.g. KV pool exhausted, slot level beyond the device */
    ASB_ERR_CUDA = 7        /* device / driver failure (no sm_100 device, launch error) */
} asb_status;

typedef struct asb_model asb_model;
typedef struct asb_kv asb_kv;
typedef struct asb_lane asb_lane;
typedef struct asb_slots asb_slots;

const char* asb_last_error(void);
const char* asb_status_name(asb_status s);
void asb_string_free(char* s);
/* Library build string: "sm_100a;<git-ish version>". */
const char* asb_build_info(void);

/* --- model --------------------------------------------------------------------------------
 * model: "tiny" | "qwen2.5-0.5b" | "llama3.2-3b" | "qwen2.5-7b" | "llama3.1-8b", or a JSON
 * object {"layers":..,"d_model":..,"n_heads":..,"n_kv_heads":..,"head_dim":..,"ffn":..,
 * "vocab":..,"tied":..,"qkv_bias":..,"rope_theta":..,"rms_eps":..}.
 * Weights are random-init bf16 from named splitmix64 sub-streams of `seed`
 * (bit-identical to oracle/forward.c).  max_context bounds the RoPE table. */
asb_status asb_model_create(const char* model, uint64_t seed, int device, int max_context,
                            asb_model** out);
asb_status asb_model_describe(const asb_model* m, char** out_json);
void asb_model_free(asb_model* m);

/* --- paged KV cache ------------------------------------------------------------------------
 * Pool of num_blocks blocks of 64 tokens, all layers.  Block ids are handed out by a
 * deterministic LIFO free list (initially 0,1,2,...). */
asb_status asb_kv_create(asb_model* m, int num_blocks, asb_kv** out);
void asb_kv_free(asb_kv* kv);
int asb_kv_block_tokens(void);
int asb_kv_free_blocks(const asb_kv* kv);
/* reference registry protocol (executor.cpp:43-82) */
asb_status asb_kv_begin_write(asb_kv* kv, uint32_t session);
asb_status asb_kv_commit(asb_kv* kv, uint32_t session, int new_prefix);
asb_status asb_kv_append(asb_kv* kv, uint32_t session, int tokens);
asb_status asb_kv_require_sealed(const asb_kv* kv, uint32_t session);
int asb_kv_sealed(const asb_kv* kv, uint32_t session);
int asb_kv_prefix(const asb_kv* kv, uint32_t session);
/* physical tokens written to the pool for the session (== prefix at every commit) */
int asb_kv_length(const asb_kv* kv, uint32_t session);
asb_status asb_kv_block_table(const asb_kv* kv, uint32_t session, int32_t* out, int cap, int* n);
/* release a finished session's blocks back to the free list */
asb_status asb_kv_release(asb_kv* kv, uint32_t session);
/* copy one token's K and V (all layers, [layer][kv_head][head_dim] bf16 bits) to host */
asb_status asb_kv_read_token(const asb_kv* kv, uint32_t session, int position, uint16_t* k_out,
                             uint16_t* v_out);

/* --- execution lanes -----------------------------------------------------------------------
 * A lane = one stream + its activation workspace + pinned staging.  Decode and prefill run
 * on separate lanes so they can co-run on disjoint SM partitions.  stream may be NULL (the
 * lane creates its own) or a cudaStream_t (e.g. from asb_slots_bind). */
asb_status asb_lane_create(asb_model* m, int max_tokens, int max_segments, void* stream,
                           asb_lane** out);
void asb_lane_free(asb_lane* lane);
asb_status asb_lane_set_stream(asb_lane* lane, void* stream);
void* asb_lane_stream(const asb_lane* lane);
/* 1 when the last launch has completed, 0 when still running */
int asb_lane_query(const asb_lane* lane);
asb_status asb_lane_wait(asb_lane* lane);
/* device time of the last launch in ms (valid once complete) */
float asb_lane_last_ms(const asb_lane* lane);

typedef struct asb_segment {
    uint32_t session;   /* KV owner; tokens are appended at the session's current length */
    int32_t n_tokens;   /* 1 = decode row, > 1 = prefill / resume chunk rows */
    int32_t want_logits;/* 1: produce next-token id (and optionally logits) for its last row */
} asb_segment;

/* One ragged forward: rows of all segments, in order, through every layer.  tokens is a
 * host array of sum(n_tokens) ids (copied H2D inside the launch).  Asynchronous. */
asb_status asb_forward(asb_lane* lane, asb_kv* kv, const asb_segment* segs, int n_segs,
                       const int32_t* tokens);
/* After completion: next-token ids (one per want_logits segment, in order) and, when
 * out_logits != NULL, fp32 logits [n][vocab].  Blocks until the launch completes. */
asb_status asb_lane_fetch(asb_lane* lane, int32_t* out_next, int n, float* out_logits);

/* Kernel timing inside the lane: CUDA events on the lane's stream around every launch of a
 * category, with the algorithmic work of that launch (bytes for HBM-bound categories,
 * FLOPs for tensor-bound ones).  Used by bench.py for the live roofline. */
enum {
    ASB_STAT_DECODE_ATTN = 0,  /* units: K/V bytes streamed */
    ASB_STAT_PREFILL_ATTN = 1, /* units: FLOPs */
    ASB_STAT_DECODE_GEMM = 2,  /* units: weight + activation bytes (swap-AB path) */
    ASB_STAT_PREFILL_GEMM = 3, /* units: FLOPs */
    ASB_STAT_FORWARD = 4,      /* whole forward; units: tokens */
    ASB_STAT_DECODE_STEP = 5,  /* reserved (the persistent decode-step kernel was removed) */
    ASB_STAT_COUNT = 6
};
asb_status asb_lane_profile(asb_lane* lane, int enable);
/* SMs available to the lane's current stream (green-context partition); sizes persistent
 * GEMM grids and split-K.  0 = whole device. */
asb_status asb_lane_set_sms(asb_lane* lane, int sms);
/* kernels launched and host<->device bytes moved by the lane since the last reset */
asb_status asb_lane_counters(asb_lane* lane, int64_t* launches, int64_t* h2d_bytes,
                             int64_t* d2h_bytes, int reset);
asb_status asb_lane_stats(asb_lane* lane, int category, double* ms, double* units,
                          int64_t* launches, int reset);

/* Convenience forms named after the reference seams. */
asb_status asb_prefill_launch(asb_lane* lane, asb_kv* kv, uint32_t session, const int32_t* tokens,
                              int n);
asb_status asb_decode_launch(asb_lane* lane, asb_kv* kv, const uint32_t* sessions,
                             const int32_t* in_tokens, int batch, int64_t chunk_session,
                             const int32_t* chunk_tokens, int chunk_n);

/* --- Green Context slot manager ------------------------------------------------------------
 * Pre-creates, for every decode level 1..levels-1, a (decode, prefill) pair of green
 * contexts with level*granularity and the complementary SMs, each with its own stream,
 * plus the full-device pair for level == levels (shared).  Rebind = pick another pair. */
asb_status asb_slots_create(int device, int levels, int granularity_sms, asb_slots** out);
void asb_slots_free(asb_slots* s);
int asb_slots_levels(const asb_slots* s);
int asb_slots_green(const asb_slots* s); /* 1 when real green contexts back the levels */
asb_status asb_slots_bind(asb_slots* s, int decode_level, void** decode_stream,
                          void** prefill_stream);
asb_status asb_slots_sm_counts(const asb_slots* s, int decode_level, int* decode_sms,
                               int* prefill_sms);

/* --- debug / test hooks (used by tests/, not by the engine) --------------------------------*/
/* Y[tokens][n_out] = X[tokens][k] . W[n_out][k]^T on device pointers; epi: 0 bf16(+bias),
 * 1 +resid, 2 silu-mul (interleaved rows), 3 fp32.  force_path: -1 auto, 0 normal, 1 swap,
 * 2 small-batch dgemv (tokens <= 32). */
/* ASB_GEMM_TIMELINE=1: per-CTA globaltimer stamps (start, MMA done, epilogue done, exit) of the
 * lane's most recent GEMM launch, [148][4] ns. */
asb_status asb_debug_gemm_timeline(asb_lane* lane, unsigned long long* out, int n);
/* ASB_ATTN_TIMELINE=1 at lane creation: per-CTA globaltimer stamps [1024][8] of the last decode
 * attention launch of the lane's most recent forward (entry, after pdl wait, first K/V
 * sub-block, consumers done, partial written, exit). */
asb_status asb_debug_attn_timeline(asb_lane* lane, unsigned long long* out, int n);
asb_status asb_debug_gemm(const void* x, const void* w, const void* bias, const void* resid,
                          void* out, int tokens, int n_out, int k, int epi, int force_path,
                          int splits, void* stream);
/* Average device time of `reps` back-to-back launches of one linear layer (weights packed
 * once into copies that exceed L2, PDL on); force_path 2 = small-batch dgemv.  stream: e.g. a
 * green-context stream from asb_slots_bind (NULL: a new full-device stream); num_sms: the SMs
 * that stream owns (0: the whole device). */
asb_status asb_debug_gemm_bench(const void* x, const void* w, void* out, int tokens, int n_out, int k,
                                int epi, int force_path, int reps, int num_sms, void* stream,
                                float* us_per_launch);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* AGENTSERVE_B200_H */
