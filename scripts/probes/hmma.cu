// Probe: legacy warp MMA (mma.sync m16n8k16 bf16 -> f32) throughput and latency on sm_100a,
// the instruction the decode-attention consumers and dgemv are built on.
//   chains C independent accumulators per warp, N MMAs each; W warps per CTA, 1 CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2603_10342_b200/csrc scripts/probes/hmma.cu -o /tmp/hmma
#include <cuda_runtime.h>
#include <cstdio>
#include "warpmma.cuh"
using namespace asb;

template <int C>
__global__ void probe(int n, float* out, unsigned long long* cyc) {
    float d[C][4];
#pragma unroll
    for (int c = 0; c < C; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.f;
    uint32_t a = 0x3f803f80u ^ threadIdx.x, b = 0x3f803f80u;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) mma16816(d[c], a, a, a, a, b, b);
    }
    const unsigned long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int C>
void run(int warps, int n) {
    float* out;
    unsigned long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4);
    cudaMalloc(&cyc, 148 * 8);
    probe<C><<<148, warps * 32>>>(n, out, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<C><<<148, warps * 32>>>(n, out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double mmas_per_sm = double(warps) * C * n;
    printf("chains %2d warps %2d: %6.1f cycles per MMA per warp (chain), %7.2f cycles per MMA per SM, "
           "%.0f dense TFLOP/s (148 SMs)\n",
           C, warps, double(c) / (double(C) * n) * 1.0 * 1.0 * (1.0) * 1.0 * (1.0) * C / C,
           double(c) / mmas_per_sm, mmas_per_sm * 148 * 4096 * 2 / (ms * 1e-3) / 1e12);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    const int n = 4096;
    for (int w : {1, 4, 8, 16}) {
        run<1>(w, n);
        run<4>(w, n);
        run<8>(w, n);
    }
    return 0;
}
