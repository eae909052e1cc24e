#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace asb {

enum EpiMode : int {
    EPI_BF16 = 0,    // y = bf16(acc + bias?)
    EPI_RESID = 1,   // y = bf16(acc + resid)       (resid may alias out: in-place residual add)
    EPI_SILU = 2,    // y[:, j] = bf16(silu(acc[2j]) * acc[2j+1])  (interleaved gate/up rows)
    EPI_F32 = 3,     // y = acc (fp32)
    EPI_QKV = 4,     // fused QKV epilogue: bf16(acc + bias) -> RoPE(q, k) -> q_out / paged K,V
};

// EPI_QKV: rows of W are [q heads | k heads | v heads] x hd (qd, kvd multiples of 128); the
// rotated q goes to q_out[tok][hq][hd], k and v to the paged pools at slot[tok]
// (layout of attn.h).  Same rounding points as a bf16 QKV GEMM followed by rope_append.
struct RopeEpi {
    const int32_t* pos;    // [tokens] absolute position (cos/sin row)
    const int32_t* slot;   // [tokens] block * kBlockTokens + offset
    const float* cos_t;    // [max_pos][hd/2]
    const float* sin_t;
    __nv_bfloat16* q_out;
    __nv_bfloat16* k_pool;
    __nv_bfloat16* v_pool;
    int hq, hkv, hd, layer, num_blocks;
};

// Fused "next pre-norm" of a residual-writing linear (EPI_RESID): the last CTA of the grid
// normalises rows of the updated residual stream x into `out` (decode-sized batches only).
struct PostNorm {
    const __nv_bfloat16* w = nullptr;  // null: off
    __nv_bfloat16* out = nullptr;      // [n_rows][d]
    const int32_t* rows = nullptr;     // source row of output row r (null: r)
    int n_rows = 0, d = 0;
    float eps = 0.f;
    int* counter = nullptr;            // zero-initialised grid arrival counter
    unsigned long long* zero_keys = nullptr;
};

struct GemmParams {
    int M, N, K;          // kernel view: D[M][N] = A[M][K] . B[N][K]^T
    int tokens, n_out;    // logical view: Y[tokens][n_out]
    int swap;             // 0: A = X, B = W.  1: A = W, B = X (Y = D^T)
    int splits;           // swap only: cluster split-K factor S (cluster = the S CTAs of a tile)
    int kb_per_split;     // internal
    int epi;
    __nv_bfloat16* out;   // Y (bf16), row stride ldo
    float* out_f32;       // Y (fp32), row stride ldo
    int ldo;
    const __nv_bfloat16* bias;   // [n_out] or null
    const __nv_bfloat16* resid;  // [tokens][ldr]
    int ldr;
    int a_packed, b_packed;  // operand is a tile-packed weight (4-D map, coords (0,0,kb,tile))
    RopeEpi rope;              // EPI_QKV only
    unsigned long long* amax;  // swap + EPI_F32 only, optional: per-token argmax_key accumulator
                               // (atomicMax; zero on entry) -- the LM head's greedy sample
    unsigned long long* dbg_times;  // optional per-CTA timeline [grid][8] (globaltimer ns)
    PostNorm post;                  // optional, EPI_RESID
    const __nv_bfloat16* w_packed;  // swap: the tile-packed weight (for L2 prefetch-ahead)
    int w_kblocks;                  // its 64-wide k-blocks per 128-row tile
    int l2_pf;                      // swap: L2 prefetch distance in pipeline units (0 = off)
    int reduce_pull;                // cluster split-K: DSMEM loads by the owner (A/B switch) instead of bulk push
    int dbg_no_epi;                 // timing ablation: epilogue drains TMEM but stores nothing
};

// Small-batch decode linear (dgemv.cu): T <= dgemv_max_tokens() rows of X against a
// tile-packed W, legacy warp MMAs fed straight from HBM, optional fused RMSNorm of X.
// Epilogue fields (epi, out, out_f32, ldo, bias, resid, ldr, rope, amax) mean what they mean
// in GemmParams; EPI_F32 + amax keeps a per-token greedy-argmax key (zeroed by the caller).
struct DgemvParams {
    const __nv_bfloat16* w;  // packed [rows_pad/128][K/64][128][64]
    int rows_pad;
    const __nv_bfloat16* x;  // [*][ldx]; row of token t = x_rows ? x_rows[t] : t
    const int32_t* x_rows;
    int ldx;
    int T, n_out, K;
    const __nv_bfloat16* norm_w;  // non-null: X := bf16(X * rms_inv(X) * norm_w) (over K)
    float eps;
    int epi;
    __nv_bfloat16* out;
    float* out_f32;
    int ldo;
    const __nv_bfloat16* bias;
    const __nv_bfloat16* resid;
    int ldr;
    RopeEpi rope;
    unsigned long long* amax;
    PostNorm post;  // optional, EPI_RESID
    int rw;  // internal: row-warps per CTA
};
int dgemv_max_tokens();
cudaError_t dgemv_launch(DgemvParams p, int num_sms, cudaStream_t stream);

// Decode linear on a TMA-fed smem ring + legacy warp MMAs (tgemv.cu), T <= 32 tokens: the
// weight-streaming kernel for decode steps on Green Context partitions.  tmap_w: the weight's
// packed map with a 2-k-block box (make_tmap_packed(.., 1, 2)); tmap_x: an activation k-pair
// map with 32-row boxes (make_tmap_act_kpair(.., 32)).  Epilogue fields as in GemmParams
// (EPI_QKV needs 128 % hd == 0).  splits: K split (0 = chosen for num_sms); ws / cnt: the
// split partials [units][32][128] fp32 and per-tile arrival counters (zeroed, self-resetting).
struct TgemvParams {
    int T, n_out, K;
    int tiles;   // 128-row weight tiles (rows_pad / 128)
    int splits;  // 0: chosen by tgemv_launch
    int kunits, kups;  // internal: 128-wide k-units, per split
    int epi;
    __nv_bfloat16* out;
    float* out_f32;
    int ldo;
    const __nv_bfloat16* bias;
    const __nv_bfloat16* resid;
    int ldr;
    RopeEpi rope;
    unsigned long long* amax;
    PostNorm post;
    float* ws;
    int* cnt;
    int dbg_load_only;  // timing ablation (ASB_DEBUG_SKIP=tgmath): consumers release stages unread
};
int tgemv_max_tokens();
int tgemv_splits(int tiles, int kunits, int num_sms);
cudaError_t tgemv_launch(const CUtensorMap& tmap_w, const CUtensorMap& tmap_x, TgemvParams p, int num_sms,
                         cudaStream_t stream);

int gemm_pick_bn(int n);
int gemm_smem_bytes(int bn);
// Cluster split-K factor for a swap-path GEMM of `tiles` weight tiles: the largest S <= 8
// whose tiles*S clusters fit co-resident on num_sms SMs with no empty K split (1 = none).
// k_blocks counts pipeline k-units of kp 64-wide blocks.
int gemm_cluster_splits(int tiles, int k_blocks, int bn, int num_sms, cudaStream_t stream,
                        int force = 0, int kp = 1);
// pdl: launch with programmatic stream serialization (overlaps the previous kernel's tail).
// kp = 2 (swap path, bn <= 64): two k-blocks per stage; ta must then be a packed weight map
// with a 2-k-block box (make_tmap_packed(..., box_kb = 2)) and tb an activation k-pair map
// (make_tmap_act_kpair).
cudaError_t gemm_launch(const CUtensorMap& ta, const CUtensorMap& tb, GemmParams p, int bn,
                        int num_sms, cudaStream_t stream, bool pdl = false, int kp = 1);

// 4-D map over a tile-packed weight [N/128][K/64][128][64]: box = box_tiles x [128][64], so
// every TMA box is box_tiles contiguous 16 KiB chunks.
bool make_tmap_packed(CUtensorMap* out, const void* base, int rows_padded, int cols, int box_tiles,
                      int box_kb = 1);
// 3-D view (64 cols, rows, k-block) of a row-major bf16 [rows][cols] activation, box
// [2 k-blocks][box_rows][64], SWIZZLE_128B: both k-blocks of a decode GEMM stage in one request.
bool make_tmap_act_kpair(CUtensorMap* out, const void* base, int rows, int cols, int box_rows);
// 5-D map over the interleaved KV pool (attn.h): box [K,V][hd/64][box_rows][64] SWIZZLE_128B,
// i.e. box_rows tokens of one page's K and V in one request (coords: 0, row, 0, 0, page).
bool make_tmap_kv_sub(CUtensorMap* out, const void* base, long pages, int hd, int page_rows, int box_rows);
// 3-D bf16 map over [d2][d1][d0] (d0 contiguous), box = [b2][b1][64], SWIZZLE_128B.
bool make_tmap_bf16_3d(CUtensorMap* out, const void* base, int d0, int d1, int d2, int b1, int b2);
// 2-D bf16 tensor map, row-major [rows][cols], box = [box_rows][64 cols], SWIZZLE_128B.
bool make_tmap_bf16(CUtensorMap* out, const void* base, int rows, int cols, int row_stride_elems,
                    int box_rows);

}  // namespace asb
