// Probe: per-CTA TMA streaming rate vs the global layout of the box, the decode-attention
// K/V stream.  Each CTA streams its own contiguous share of a 1 GiB bf16 buffer into a
// `stages`-deep ring (one elected producer thread, consumers release immediately).
//   mode 0 "rowmajor": view [rows][128] (256 B rows), box = [2 halves][32 rows][64 cols]
//          (3-D, strides 256 B / 128 B): 8 KiB of 128 B pieces at 256 B stride
//   mode 1 "halfmajor": view [rows][64] (128 B rows), box = [32 rows][64 cols] x 2 requests or
//          one 3-D box [2][32][64] whose halves are 4 KiB contiguous runs
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc \
//        scripts/probes/tma_stride.cu paper_2603_10342_b200/csrc/tmap.cpp -lcuda -o /tmp/tma_stride
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
#include "gemm.h"
using namespace asb;

__global__ void __launch_bounds__(64, 1) stream3d(const __grid_constant__ CUtensorMap map, int n_boxes_total,
                                                  int box_bytes, int stages, int mode, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * box_bytes);
    uint64_t* empty = full + stages;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        fence_barrier_init();
        tma_prefetch_desc(&map);
    }
    __syncthreads();
    const int b0 = (int)((long long)n_boxes_total * blockIdx.x / gridDim.x);
    const int b1 = (int)((long long)n_boxes_total * (blockIdx.x + 1) / gridDim.x);
    const int n = b1 - b0;
    if (threadIdx.x == 0) {
        const uint64_t pol = policy_evict_first();
        for (int i = 0; i < n; ++i) {
            const int st = i % stages;
            mbar_wait(&empty[st], ((i / stages) & 1) ^ 1);
            mbar_expect_tx(&full[st], box_bytes);
            const int b = b0 + i;
            if (mode == 0) tma_load_3d_hint(sm + (size_t)st * box_bytes, &map, &full[st], 0, b * 32, 0, pol);
            else tma_load_3d_hint(sm + (size_t)st * box_bytes, &map, &full[st], 0, 0, b, pol);
        }
    } else if (threadIdx.x == 32) {
        unsigned long long acc = 0;
        for (int i = 0; i < n; ++i) {
            const int st = i % stages;
            mbar_wait(&full[st], (i / stages) & 1);
            acc += sm[(size_t)st * box_bytes + (i & 63)];
            mbar_arrive(&empty[st]);
        }
        sink[blockIdx.x] = acc;
    }
}

int main() {
    const size_t bytes = 1ull << 30;
    void* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    unsigned long long* sink;
    cudaMalloc(&sink, 1024 * 8);
    for (int box_kb : {8, 16, 32}) {
        const int box_bytes = box_kb * 1024;
        const int box_rows = box_bytes / 128;
        CUtensorMap map;  // contiguous [n][box_rows][64] bf16, box (64, box_rows, 1)
        const int n_boxes = (int)(bytes / box_bytes);
        if (!make_tmap_bf16_3d(&map, buf, 64, box_rows, n_boxes, box_rows > 256 ? 256 : box_rows, 1)) {
            printf("tmap failed %d KiB\n", box_kb);
            continue;
        }
        for (int ctas : {32, 148}) {
            for (int stages : {2, 4, 6, 8, 12}) {
                const int smem = stages * box_bytes + 2 * stages * 8 + 1024;
                if (smem > 227 * 1024) continue;
                cudaFuncSetAttribute(stream3d, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                stream3d<<<ctas, 64, smem>>>(map, n_boxes, box_bytes, stages, 1, sink);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                stream3d<<<ctas, 64, smem>>>(map, n_boxes, box_bytes, stages, 1, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, e0, e1);
                const double gbs = (double)n_boxes * box_bytes / (ms * 1e-3) / 1e9;
                printf("box %2d KiB CTAs %4d stages %2d (%3d KiB in flight): %7.1f GB/s  %6.1f GB/s/CTA  %s\n", box_kb,
                       ctas, stages, stages * box_kb, gbs, gbs / ctas, cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
