// Persistent decode-step kernel: one launch runs a whole decode forward (all layers + LM head
// + greedy sample) for <= 16 single-token decode rows.  See decode_step.cu.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "attn.h"

namespace asb {

struct MkLayer {
    const __nv_bfloat16* wqkv;  // tile-packed [(hq+2hkv)hd / 128][d/64][128][64]
    const __nv_bfloat16* wo;    // [d/128][hq*hd/64][128][64]
    const __nv_bfloat16* wgu;   // [2ffn/128][d/64][128][64], rows interleaved gate/up
    const __nv_bfloat16* wdown; // [d/128][ffn/64][128][64]
    const __nv_bfloat16* attn_norm;
    const __nv_bfloat16* mlp_norm;
    const __nv_bfloat16* qkv_bias;  // or null
};

struct MkParams {
    const MkLayer* layers;  // device array [L]
    int L, d, hq, hkv, hd, ffn, vocab;
    float eps, scale_log2;
    int T;           // decode rows (<= 16), row t = DecodeItem t
    int G;           // grid size (CTAs, one per SM of the partition)
    int attn_spl;    // attention splits per (row, kv head)
    const int32_t* tok;
    const int32_t* pos;
    const int32_t* slot;
    const DecodeItem* items;
    const int32_t* tables;
    const __nv_bfloat16* embed;    // tile-packed embedding table [vocab_pad/128][d/64][128][64]
    const __nv_bfloat16* lm_head;  // tile-packed (== embed when tied)
    const __nv_bfloat16* final_norm;
    __nv_bfloat16* x;     // [T][d] residual stream
    __nv_bfloat16* q;     // [T][hq][hd] rotated queries
    __nv_bfloat16* attn;  // [T][hq][hd]
    __nv_bfloat16* act;   // [T][ffn]
    float* logits;        // [T][vocab]
    unsigned long long* keys;  // [T] greedy argmax keys
    __nv_bfloat16* k_pool;
    __nv_bfloat16* v_pool;
    int num_blocks;
    const float* cos_t;
    const float* sin_t;
    // synchronisation and workspaces (zero-initialised, self-resetting)
    unsigned* bar;      // [0] arrivals, [32] generation (separate 128-byte lines)
    int* tile_cnt;      // [max weight tiles]
    float* ws;          // [G][2][128][32] split-tile partials
    float* apart_o;     // [T*hkv*attn_spl][G_heads][hd]
    float* apart_ml;    // [T*hkv*attn_spl][G_heads][2]
    int* acnt;          // [T*hkv]
    unsigned long long* dbg;  // optional: [G][kMkDbgSlots] globaltimer at each phase start
};
constexpr int kMkDbgSlots = 256;

// Activation tensor maps (bf16 [rows][cols], box [32 rows][64 cols], SWIZZLE_128B) for the
// three GEMV inputs and the K/V pool maps with 32-row boxes (decode attention's tk32/tv32).
struct MkMaps {
    CUtensorMap x, attn, act, k32, v32;
};

constexpr int kMkMaxRows = 16;
int decode_step_smem_bytes(int hd);
// Grid = p.G CTAs launched cooperatively (all co-resident or the launch fails).
cudaError_t decode_step_launch(const MkMaps& maps, const MkParams& p, cudaStream_t stream);

}  // namespace asb
