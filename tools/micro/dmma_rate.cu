// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_rate.cu -o dmma_rate
// Microbenchmark: FP64 DMMA (mma.sync m8n8k4 f64) vs DFMA issue rate on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_k(double *out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[8][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[q][0]), "+d"(c[q][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int q = 0; q < 8; ++q) s += c[q][0] + c[q][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void dfma_k(double *out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
    double c[16] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 16; ++q) c[q] = fma(a, c[q], b);
    }
    double s = 0;
    for (int q = 0; q < 16; ++q) s += c[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    double *out;
    cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        int iters = 20000;
        dmma_k<<<148 * 4, warps * 32>>>(out, 10);
        cudaEventRecord(e0);
        dmma_k<<<148 * 4, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 256 * 8 * double(iters) * 148 * 4 * warps;   // 256 FMA per DMMA per warp
        printf("DMMA warps/CTA %2d: %.1f TFLOP/s\n", warps, fl / (ms * 1e-3) / 1e12);
        dfma_k<<<148 * 4, warps * 32>>>(out, 10);
        cudaEventRecord(e0);
        dfma_k<<<148 * 4, warps * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        fl = 2.0 * 16 * double(iters) * 148 * 4 * warps * 32;
        printf("DFMA warps/CTA %2d: %.1f TFLOP/s\n", warps, fl / (ms * 1e-3) / 1e12);
    }
    return 0;
}
