#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include <cstdint>
#include <string>

namespace asb {

struct ModelSpec {
    std::string name = "custom";
    int layers = 0, d = 0, hq = 0, hkv = 0, hd = 0, ffn = 0, vocab = 0;
    bool tied = true, qkv_bias = false;
    double theta = 10000.0;
    float eps = 1e-6f;
    bool rope_llama3 = false;
    double rope_factor = 1.0, rope_lo = 1.0, rope_hi = 4.0, rope_orig = 8192.0;
};

struct Weight {
    __nv_bfloat16* ptr = nullptr;  // tile-packed [rows_pad/128][cols/64][128][64]
    int rows = 0, rows_pad = 0, cols = 0;
    CUtensorMap map_b256;  // B operand of the normal path (box 256 rows)
    CUtensorMap map_a128;  // A operand of the swap path / B with BN=128 (box 128 rows)
    CUtensorMap map_a128k2;  // swap path, two k-blocks per stage (box [2][128][64], 32 KiB)
};

uint64_t substream_state(uint64_t seed, const std::string& name);

}  // namespace asb
