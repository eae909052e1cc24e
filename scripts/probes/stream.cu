// Probe: per-SM HBM streaming rate with G CTAs (one per SM), the limit of every decode-step
// kernel on a small Green Context partition.  Each CTA streams a contiguous share of a 2 GiB
// buffer into shared memory (no compute):
//   bulk : one thread issues cp.async.bulk of `chunk` bytes into a `stages`-deep mbarrier ring
//   ldg  : 256 threads, `unroll` 16-byte ld.global.nc.L1::no_allocate per thread in flight
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc scripts/probes/stream.cu -o /tmp/stream
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
#include "gemm.h"
using namespace asb;

// 4-D tensor TMA over a tile-packed weight view [nt][kb][128][64] bf16 (box [kbox][128][64]),
// the decode GEMM's weight stream, vs the same bytes by 1-D bulk copies
__global__ void __launch_bounds__(64, 1) stream_tma4d(const __grid_constant__ CUtensorMap map, int nt, int kbs,
                                                       int kbox, int stages, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int chunk = kbox * 16384;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
    uint64_t* empty = full + stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
        tma_prefetch_desc(&map);
    }
    __syncthreads();
    const int t0 = (nt * blockIdx.x) / gridDim.x, t1 = (nt * (blockIdx.x + 1)) / gridDim.x;
    const long long n = (long long)(t1 - t0) * (kbs / kbox);
    if (threadIdx.x == 0) {
        for (long long i = 0; i < n; ++i) {
            const int st = i % stages;
            mbar_wait(&empty[st], ((i / stages) & 1) ^ 1);
            mbar_expect_tx(&full[st], chunk);
            const int tile = t0 + (int)(i / (kbs / kbox)), kb = (int)(i % (kbs / kbox)) * kbox;
            tma_load_4d_hint(sm + (size_t)st * chunk, &map, &full[st], 0, 0, kb, tile, policy_evict_first());
        }
    } else if (threadIdx.x == 32) {
        unsigned long long acc = 0;
        for (long long i = 0; i < n; ++i) {
            const int st = i % stages;
            mbar_wait(&full[st], (i / stages) & 1);
            acc += sm[(size_t)st * chunk];
            mbar_arrive(&empty[st]);
        }
        if (acc == 0xdeadbeef) *sink = acc;
    }
}

__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// mbarrier wait without the suspend-time hint (pure try_wait spin)
__device__ __forceinline__ void mbar_wait_spin(uint64_t* bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n\t"
        "DONE_%=:\n\t}\n" ::"r"(addr), "r"(parity) : "memory");
}
__device__ int g_spin = 0;

__global__ void __launch_bounds__(64, 1) stream_bulk(const uint8_t* buf, size_t per_cta, int chunk, int stages,
                                                      unsigned long long* sink, int issuers) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * chunk);
    uint64_t* empty = full + stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const uint8_t* src = buf + per_cta * blockIdx.x;
    const long long n = per_cta / chunk;
    if (threadIdx.x < issuers) {  // issuer q takes chunks i = q, q + issuers, ...
        for (long long i = threadIdx.x; i < n; i += issuers) {
            const int st = i % stages;
            if (g_spin) mbar_wait_spin(&empty[st], ((i / stages) & 1) ^ 1);
            else mbar_wait(&empty[st], ((i / stages) & 1) ^ 1);
            mbar_expect_tx(&full[st], chunk);
            bulk(sm + (size_t)st * chunk, src + i * chunk, chunk, &full[st]);
        }
    } else if (threadIdx.x == 32) {
        unsigned long long acc = 0;
        for (long long i = 0; i < n; ++i) {
            const int st = i % stages;
            if (g_spin) mbar_wait_spin(&full[st], (i / stages) & 1);
            else mbar_wait(&full[st], (i / stages) & 1);
            acc += sm[(size_t)st * chunk];
            mbar_arrive(&empty[st]);
        }
        if (acc == 0xdeadbeef) *sink = acc;
    }
}

template <int U, int NTH>
__global__ void __launch_bounds__(NTH, 1) stream_ldg(const uint4* buf, size_t per_cta16, unsigned long long* sink) {
    const uint4* src = buf + per_cta16 * blockIdx.x;
    uint32_t acc = 0;
    for (size_t i = threadIdx.x; i < per_cta16; i += NTH * U) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t k = i + (size_t)u * NTH;
            if (k < per_cta16)
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(src + k));
            else v[u] = make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0xdeadbeef) *sink = acc;
}

int main() {
    const size_t total = size_t(2) << 30;
    uint8_t* buf;
    unsigned long long* sink;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 1, total);
    cudaMalloc(&sink, 8);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(stream_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaFuncSetAttribute(stream_tma4d, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    const int K = 896, nt = int(total / (size_t(128) * K * 2));
    CUtensorMap maps[3];
    for (int kb : {1, 2, 4}) make_tmap_packed(&maps[kb == 1 ? 0 : kb == 2 ? 1 : 2], buf, nt * 128, K, 1, kb);
    for (int G : {16, 148}) {
        for (int kb : {1, 2, 4})
            for (int stages : {3, 4, 6, 8}) {
                const int chunk = kb * 16384;
                if ((size_t)stages * chunk > 200 * 1024 || (K / 64) % kb) continue;
                const int smem = stages * chunk + 2 * stages * 8 + 64;
                CUtensorMap m = maps[kb == 1 ? 0 : kb == 2 ? 1 : 2];
                stream_tma4d<<<G, 64, smem>>>(m, nt, K / 64, kb, stages, sink);
                cudaEventRecord(a);
                stream_tma4d<<<G, 64, smem>>>(m, nt, K / 64, kb, stages, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double gbs = double(nt) * 128 * K * 2 / (ms * 1e-3) / 1e9;
                printf("tma4d G=%3d box=%d kb (%5d B) stages=%d  %7.1f GB/s  %6.1f GB/s/SM\n", G, kb, chunk, stages, gbs,
                       gbs / G);
            }
        const size_t per = (total / G) & ~size_t(65535);
        for (int chunk : {16384, 32768, 65536})
            for (int stages : {3, 4, 6}) {
                if ((size_t)stages * chunk > 200 * 1024) continue;
                const int smem = stages * chunk + 2 * stages * 8;
                stream_bulk<<<G, 64, smem>>>(buf, per, chunk, stages, sink, 1);
                cudaEventRecord(a);
                stream_bulk<<<G, 64, smem>>>(buf, per, chunk, stages, sink, 1);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double gbs = per * (double)G / (ms * 1e-3) / 1e9;
                printf("bulk  G=%3d chunk=%6d stages=%d  %7.1f GB/s  %6.1f GB/s/SM\n", G, chunk, stages, gbs, gbs / G);
            }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
