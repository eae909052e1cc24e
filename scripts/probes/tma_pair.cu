// Probe: per-CTA TMA streaming rate of the decode-GEMM operand pattern.  Each stage of the
// swap-AB decode GEMM moves one big weight box (streamed from HBM) AND one small activation
// box (the same few KiB re-read from L2 by every CTA).  Does the second request per stage cost
// streaming rate (per-SM TMA request issue), and what do 64 KiB weight boxes buy?
//   w_kb  : weight box KiB per stage (32 or 64), x_kb : activation box KiB (0 = none)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc \
//        scripts/probes/tma_pair.cu paper_2603_10342_b200/csrc/tmap.cpp -lcuda -o /tmp/tma_pair
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
#include "gemm.h"
using namespace asb;

__global__ void __launch_bounds__(64, 1) stream_pair(const __grid_constant__ CUtensorMap wmap,
                                                     const __grid_constant__ CUtensorMap xmap, int n_boxes_total,
                                                     int w_bytes, int x_bytes, int x_rows, int stages,
                                                     unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int stage_bytes = w_bytes + x_bytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * stage_bytes);
    uint64_t* empty = full + stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
        tma_prefetch_desc(&wmap);
        tma_prefetch_desc(&xmap);
    }
    __syncthreads();
    const int b0 = (int)((long long)n_boxes_total * blockIdx.x / gridDim.x);
    const int b1 = (int)((long long)n_boxes_total * (blockIdx.x + 1) / gridDim.x);
    const int n = b1 - b0;
    const int w_rows = w_bytes / 128;
    if (threadIdx.x == 0) {
        const uint64_t pw = policy_evict_first(), px = policy_evict_last();
        for (int i = 0; i < n; ++i) {
            const int st = i % stages;
            mbar_wait(&empty[st], ((i / stages) & 1) ^ 1);
            mbar_expect_tx(&full[st], stage_bytes);
            uint8_t* d = sm + (size_t)st * stage_bytes;
            tma_load_3d_hint(d, &wmap, &full[st], 0, 0, (b0 + i) * (w_rows > 256 ? w_rows / 256 : 1), pw);
            if (x_bytes) tma_load_3d_hint(d + w_bytes, &xmap, &full[st], 0, 0, i % 16, px);
        }
        (void)w_rows;
        (void)x_rows;
    } else if (threadIdx.x == 32) {
        unsigned long long acc = 0;
        for (int i = 0; i < n; ++i) {
            const int st = i % stages;
            mbar_wait(&full[st], (i / stages) & 1);
            acc += sm[(size_t)st * stage_bytes + (i & 63)];
            mbar_arrive(&empty[st]);
        }
        sink[blockIdx.x] = acc;
    }
}

// the same ring over the tile-packed weight layout: CTA c streams tiles c, c + grid, ... (all
// k-units of a tile in order), as tgemv does with one split
__global__ void __launch_bounds__(64, 1) stream_packed(const __grid_constant__ CUtensorMap pmap,
                                                       const __grid_constant__ CUtensorMap xmap, int tiles, int kunits,
                                                       int stages, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const int stage_bytes = 32768 + 4096;
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * stage_bytes);
    uint64_t* empty = full + stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint64_t pw = policy_evict_first(), px = policy_evict_last();
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x)
            for (int ku = 0; ku < kunits; ++ku, ++i) {
                const int st = i % stages;
                mbar_wait(&empty[st], ((i / stages) & 1) ^ 1);
                mbar_expect_tx(&full[st], stage_bytes);
                uint8_t* d = sm + (size_t)st * stage_bytes;
                tma_load_4d_hint(d, &pmap, &full[st], 0, 0, 2 * ku, tile, pw);
                tma_load_3d_hint(d + 32768, &xmap, &full[st], 0, 0, ku % 16, px);
            }
    } else if (threadIdx.x == 32) {
        unsigned long long acc = 0;
        int i = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x)
            for (int ku = 0; ku < kunits; ++ku, ++i) {
                const int st = i % stages;
                mbar_wait(&full[st], (i / stages) & 1);
                acc += sm[(size_t)st * stage_bytes + (i & 63)];
                mbar_arrive(&empty[st]);
            }
        sink[blockIdx.x] = acc;
    }
}

int main() {
    const size_t bytes = 1ull << 30;
    void *buf, *xbuf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    cudaMalloc(&xbuf, 16 << 20);
    cudaMemset(xbuf, 1, 16 << 20);
    unsigned long long* sink;
    cudaMalloc(&sink, 1024 * 8);
    {  // packed weight layout [tiles][kb][128][64] through the 4-D map the GEMMs use, box (64,128,2,1)
        const int K = 3072, kbs = K / 64, tiles = (int)(bytes / (size_t(K) * 128 * 2));
        CUtensorMap pmap, xmap;
        make_tmap_packed(&pmap, buf, tiles * 128, K, 1, 2);
        make_tmap_bf16_3d(&xmap, xbuf, 64, 32, 16, 32, 1);  // box 32 rows x 128 B = 4 KiB
        for (int ctas : {16, 32, 64, 148})
            for (int stages : {4, 5, 6}) {
                const int wb = 32768, xb = 4096, smem = stages * (wb + xb) + 2 * stages * 8 + 1024;
                cudaFuncSetAttribute(stream_packed, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                stream_packed<<<ctas, 64, smem>>>(pmap, xmap, tiles, kbs / 2, stages, sink);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                stream_packed<<<ctas, 64, smem>>>(pmap, xmap, tiles, kbs / 2, stages, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                const double gbs = (double)tiles * K * 128 * 2 / (ms * 1e-3) / 1e9;
                printf("packed 4-D w 32 KiB + x 4 KiB, CTAs %3d, stages %d: %7.1f GB/s  %6.1f GB/s/CTA  %s\n", ctas, stages,
                       gbs, gbs / ctas, cudaGetErrorString(cudaGetLastError()));
            }
    }
    for (int w_kb : {32, 64}) {
        const int w_bytes = w_kb * 1024, w_rows = w_bytes / 128;
        CUtensorMap wmap;
        const int n_boxes = (int)(bytes / w_bytes);
        // [n * planes][rows <= 256][64] bf16; box (64, rows, planes)
        const int prow = w_rows > 256 ? 256 : w_rows, planes = w_rows / prow;
        if (!make_tmap_bf16_3d(&wmap, buf, 64, prow, n_boxes * planes, prow, planes)) { printf("wmap failed\n"); continue; }
        for (int x_kb : {0, 4, 8}) {
            CUtensorMap xmap;
            const int x_bytes = x_kb * 1024, x_rows = x_kb ? x_bytes / 128 : 8;
            if (!make_tmap_bf16_3d(&xmap, xbuf, 64, x_rows, 16, x_rows, 1)) { printf("xmap failed\n"); continue; }
            for (int ctas : {16, 32, 64, 148}) {
                for (int stages : {3, 4, 5, 6}) {
                    const int smem = stages * (w_bytes + x_bytes) + 2 * stages * 8 + 1024;
                    if (smem > 227 * 1024) continue;
                    cudaFuncSetAttribute(stream_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                    stream_pair<<<ctas, 64, smem>>>(wmap, xmap, n_boxes, w_bytes, x_bytes, x_rows, stages, sink);
                    cudaEvent_t e0, e1;
                    cudaEventCreate(&e0);
                    cudaEventCreate(&e1);
                    cudaEventRecord(e0);
                    stream_pair<<<ctas, 64, smem>>>(wmap, xmap, n_boxes, w_bytes, x_bytes, x_rows, stages, sink);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    float ms = 0.f;
                    cudaEventElapsedTime(&ms, e0, e1);
                    const double gbs = (double)n_boxes * w_bytes / (ms * 1e-3) / 1e9;
                    printf("w %2d KiB + x %d KiB, CTAs %3d, stages %d (%3d KiB in flight): %7.1f GB/s  %6.1f GB/s/CTA  %s\n",
                           w_kb, x_kb, ctas, stages, stages * (w_kb + x_kb), gbs, gbs / ctas,
                           cudaGetErrorString(cudaGetLastError()));
                }
            }
        }
    }
    return 0;
}
