// Probe: tcgen05.mma kind::f16 with the A operand in TMEM (the ".ts" form used to feed P from
// TMEM into P.V).  D[128x64] = A[128x64] (TMEM, bf16 pairs per 32-bit column) . B[64x64]^T
// (smem, K-major SWIZZLE_128B).  Prints the max abs error vs a host fp32 reference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I paper_2603_10342_b200/csrc scripts/probes/tsmma.cu -o /tmp/tsmma
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "sm100.cuh"
using namespace asb;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n"
                 :: "r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
                 "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]),
                    "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
                    "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
                    "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
                    "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int b_mn) {
    __shared__ __align__(1024) uint8_t sb[64 * 128];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int t = threadIdx.x, warp = t / 32, lane = t % 32;
    if (warp == 0) tmem_alloc<256>(&slot);
    if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    // B into smem. b_mn == 0: K-major rows n (64 k each).  b_mn == 1: MN-major (rows k, 64 n each).
    for (int i = t; i < 64 * 64; i += blockDim.x) {
        const int r = i / 64, c = i % 64;  // r = n, c = k   (B[n][k])
        const int row = b_mn ? c : r, col = b_mn ? r : c;
        const int off = row * 128 + (((col / 8) ^ (row % 8)) * 16) + (col % 8) * 2;
        *reinterpret_cast<__nv_bfloat16*>(sb + off) = B[r * 64 + c];
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = slot;
    // A row (lane quarter = warp) into TMEM columns [128, 160): column c holds k = 2c (lo), 2c+1 (hi)
    {
        const int r = warp * 32 + lane;
        uint32_t v[32];
        for (int c = 0; c < 32; ++c) {
            __nv_bfloat162 p = __halves2bfloat162(A[r * 64 + 2 * c], A[r * 64 + 2 * c + 1]);
            v[c] = *reinterpret_cast<uint32_t*>(&p);
        }
        tmem_st32(tm + ((warp * 32u) << 16) + 128, v);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (t == 0) {
        const uint32_t idesc = make_idesc_bf16(128, 64, false, b_mn != 0);
        for (int k = 0; k < 4; ++k) {
            // K-major B: +32 bytes per 16-k step; MN-major B: +16 k rows = 2048 bytes
            const uint64_t bd = b_mn ? make_sw128_desc(smem_u32(sb) + k * 2048, 64 * 128, 1024)
                                     : make_sw128_desc(smem_u32(sb) + k * 32, 16, 1024);
            umma_ts(tm, tm + 128 + 8 * k, bd, idesc, k > 0);
        }
        umma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int r = warp * 32 + lane;
    for (int c = 0; c < 64; c += 32) {
        uint32_t v[32];
        tmem_ld32(tm + ((warp * 32u) << 16) + c, v);
        tmem_ld_wait();
        for (int j = 0; j < 32; ++j) D[r * 64 + c + j] = __uint_as_float(v[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tm); }
}

int main() {
    std::vector<__nv_bfloat16> A(128 * 64), B(64 * 64);
    std::vector<float> Af(A.size()), Bf(B.size());
    srand(1);
    for (size_t i = 0; i < A.size(); ++i) { float x = (rand() % 2001 - 1000) / 1000.f; A[i] = __float2bfloat16(x); Af[i] = __bfloat162float(A[i]); }
    for (size_t i = 0; i < B.size(); ++i) { float x = (rand() % 2001 - 1000) / 1000.f; B[i] = __float2bfloat16(x); Bf[i] = __bfloat162float(B[i]); }
    __nv_bfloat16 *dA, *dB; float* dD;
    cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, 128 * 64 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    for (int b_mn = 0; b_mn < 2; ++b_mn) {
        cudaMemset(dD, 0, 128 * 64 * 4);
        probe<<<1, 128>>>(dA, dB, dD, b_mn);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> D(128 * 64);
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 64; ++n) {
                double ref = 0;
                for (int k = 0; k < 64; ++k) ref += double(Af[m * 64 + k]) * Bf[n * 64 + k];
                err = std::max(err, std::fabs(ref - D[m * 64 + n]));
            }
        printf("b_mn=%d status=%s max_abs_err=%.3e  D[0][0..3]=%f %f %f %f\n", b_mn, cudaGetErrorString(e), err, D[0], D[1], D[2], D[3]);
    }
    return 0;
}
