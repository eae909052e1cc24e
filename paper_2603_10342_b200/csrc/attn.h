#pragma once
#include <vector>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace asb {

// Paged KV cache geometry.  One bf16 pool, laid out
//   [layer][block][kv_head][K: kBlockTokens rows | V: kBlockTokens rows][head_dim]
// so one KV block of one head is a contiguous 64 x head_dim K tile followed by its V tile
// (8 or 16 KiB each): a single TMA box each for prefill attention, one box for both in decode.
constexpr int kBlockTokens = 64;

// One prefill-attention work item: up to prefill_tokens_per_cta() query tokens of one
// segment; the CTA's 2 x 128 MMA rows are those tokens x the G query heads of one KV head
// (two Q tiles of prefill_tokens_per_tile() tokens each).
struct PrefillItem {
    int q_row0;     // first token row in the q / out buffers
    int q_pos0;     // absolute position of that token
    int n_q;        // valid query tokens (<= 2 * 128 / G)
    int table_off;  // offset of this segment's block table in the batch table array
};

// One decode-attention item: up to 8 (token, query head) columns of one KV head's MMA N tile.
// The columns of a token group (n tokens of one session at consecutive rows / positions:
// a decode row is n = 1, an admitted resume chunk n <= 16) are numbered c = token * G + head;
// an item takes columns col0 .. col0 + 7 of its group, so a chunk's tokens share each K/V block
// read (G = 3: 16 tokens in 6 items instead of 16 single-token rows).
struct DecodeItem {
    int q_row;      // row in q / out of the group's first token
    int ctx_len;    // keys the first token attends (positions 0..ctx_len-1, its own included);
                    // token j of the group attends ctx_len + j
    int table_off;  // block table offset
    int pad;        // first position of the session written by this forward (its blocks are
                    // read only after the QKV kernel: PDL wait); ctx_len - 1 for a decode row
    int col0;       // first column of this item within its group
    int ncols;      // columns of the group (n * G); columns >= ncols are padding
};

// KV pool page layout: [layer][block][kv_head][K rows 0..63 | V rows 0..63][hd] bf16 -- the K and
// V pages of one (block, head) are adjacent, so a decode sub-block (32 tokens of K and of V)
// is one 16 KiB (hd 128) TMA request; kKvPageRows rows separate consecutive (block, head) pages.
constexpr int kKvPageRows = 2 * kBlockTokens;

struct AttnShape {
    int hq, hkv, hd;
    int num_blocks;   // blocks per layer in the pool
    int layer;        // layer index (selects the pool slice)
    float scale_log2; // log2(e) / sqrt(hd)
    unsigned long long* dbg = nullptr;  // decode attention: per-CTA globaltimer stamps [cta][8]
    int dbg_load_only = 0;  // decode attention timing ablation: consumers skip the math
    int no_prewait = 0;     // decode attention: wait for the previous kernel before any block
                            // (ASB_ATTN_PREWAIT=0; default streams blocks older than this step first)
};

// grid = (items, hkv, splits).  Split-KV over gridDim.z when the grid is small (resume
// chunks): partials part_o [items*hkv*splits*256][hd] fp32 and part_ml [..][2], merged by a
// combine kernel.  tmap_q is the 3-D map [T][hq][hd] with box [tokens_per_tile][G][64].
int prefill_tokens_per_tile(int hq, int hkv);
int prefill_tokens_per_cta(int hq, int hkv);
int prefill_splits(int n_items, int hkv, int max_blocks, int num_sms, size_t ws_rows);
// Work-unit form (one wave; only items longer than the per-CTA page budget split).  units[u] =
// (item, first page, pages, partial slot or -1); comb[c] = (item, first slot, slots).
// prefill_units returns 0 when the uniform path should be used instead.
int prefill_units(const PrefillItem* items, int n_items, int hkv, int num_sms, size_t ws_rows,
                  std::vector<int4>& units, std::vector<int4>& comb);
cudaError_t prefill_attention_units(const CUtensorMap& tmap_q, const CUtensorMap& tmap_k,
                                    const CUtensorMap& tmap_v, const PrefillItem* items, const int4* units,
                                    int n_units, const int4* comb, int n_comb, const int32_t* tables,
                                    __nv_bfloat16* out, float* part_o, float* part_ml, const AttnShape& s,
                                    cudaStream_t stream);
cudaError_t prefill_attention(const CUtensorMap& tmap_q, const CUtensorMap& tmap_k,
                              const CUtensorMap& tmap_v, const PrefillItem* items, int n_items,
                              int max_blocks, int splits, const int32_t* tables,
                              __nv_bfloat16* out, float* part_o, float* part_ml, const AttnShape& s,
                              cudaStream_t stream);

// Split-KV paged decode attention.  tmap_kv: the pool as (col, row, half, K|V, page) with a
// box of one whole block (64 rows x hd, K and V) -- make_tmap_kv_sub(.., box_rows = 64).
// part_* workspaces are sized by the caller for n_items * hq * max_splits entries.
// counters: [n_items][hkv] zero-initialised ints; the last split CTA of each (row, kv head)
// merges the partials itself and resets its counter (no combine launch).
cudaError_t decode_attention(const CUtensorMap& tmap_kv, const __nv_bfloat16* q, const DecodeItem* items,
                             int n_items, int max_ctx, const int32_t* tables, __nv_bfloat16* out,
                             float* part_o, float* part_ml, int* counters, int max_splits, int num_sms,
                             const AttnShape& s, cudaStream_t stream);

int decode_splits(int n_items, int hkv, int max_ctx, int num_sms, int max_splits);
int decode_splits_persist(int base, int pages, int num_sms, int max_splits);

}  // namespace asb
