/* CPU fp32 forward oracle — TEST INFRASTRUCTURE ONLY (see oracle/forward.c header). */
#ifndef AGENTSERVE_FORWARD_ORACLE_H
#define AGENTSERVE_FORWARD_ORACLE_H
#include <stdint.h>

typedef struct fo_spec {
    int layers, d, hq, hkv, hd, ffn, vocab;
    int tied, qkv_bias;
    double theta;
    float eps;
    int rope_llama3;
    double rope_factor, rope_lo, rope_hi, rope_orig;
} fo_spec;

typedef struct fo_model fo_model;
typedef struct fo_session fo_session;

fo_model* fo_create(const fo_spec* spec, uint64_t seed, int max_ctx, int n_layers_limit);
void fo_free(fo_model* m);
/* bf16 bits of a named weight tensor element (same generator as the device init) */
uint16_t fo_weight_bits(uint64_t seed, const char* name, int64_t index, float offset, float amp);
/* Read-only view of a generated weight tensor (fp32 holding bf16 values): name is one of
 * embed, lm_head, final_norm, or a per-layer attn_norm, mlp_norm, q, k, v, q_bias, k_bias,
 * v_bias, o, gate, up, down; *n receives the element count.  NULL if absent. */
const float* fo_tensor(const fo_model* m, int layer, const char* name, int64_t* n);
fo_session* fo_session_new(fo_model* m);
void fo_session_free(fo_session* s);
int fo_session_len(const fo_session* s);
/* Append n tokens; logits (fp32 [vocab]) of the last row into logits_out (nullable).
 * Returns the greedy next id (lowest index on ties). */
int fo_forward(fo_model* m, fo_session* s, const int32_t* tokens, int n, float* logits_out);
/* bf16 bits of K and V at one position: [layer][kv_head][head_dim] each */
void fo_read_kv(const fo_model* m, const fo_session* s, int pos, uint16_t* k_out, uint16_t* v_out);
/* splitmix64 named sub-stream helpers (rng.hpp restatement) */
uint64_t fo_substream(uint64_t seed, const char* name);
uint64_t fo_next_u64(uint64_t* state);
uint64_t fo_uniform_int(uint64_t* state, uint64_t n);

#endif
