// Legacy warp-level tensor-core helpers (mma.sync m16n8k16, ldmatrix) and the SW128 tile
// addressing shared by the memory-bound decode kernels (decode_attn.cu, dgemv.cu), where
// a register-resident warp MMA beats a TMEM round trip for M <= 16-row problems.
#pragma once
#include <cstdint>

#include "sm100.cuh"

namespace asb {

__device__ __forceinline__ void named_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                        uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr));
}
// D = A (16x16 bf16, row) * B (16x8 bf16, col) + D, fp32 accumulate.  Not volatile: a pure
// register function, so the compiler may interleave independent MMAs with the ldmatrix loads
// of the next k-step (volatile pinned every MMA behind the load just before it, serialising
// load latency and MMA latency).  Accumulation order is fixed by the data dependence.
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
    asm(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// byte offset of 16-byte chunk `c` (0..HD/8-1) of row `r` in a [32 rows][HD] K/V sub-block
// stored as HD/64 SWIZZLE_128B TMA boxes of [32 rows][64 cols]
constexpr int kSwRows = 32;
template <int HD>
__device__ __forceinline__ uint32_t sw_off(int r, int c) {
    const int box = c >> 3, cc = c & 7;
    return box * (kSwRows * 128) + r * 128 + ((cc ^ (r & 7)) << 4);
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

}  // namespace asb
