// Microbenchmarks for the resident-CG design (DESIGN.md §6 "resident CG"):
//  (1) TMEM as per-thread storage: tcgen05.st / tcgen05.ld 32x32b throughput
//      with 8 warps per SM (two warps per lane quarter, column halves);
//  (2) a grid-wide barrier (one CTA per SM, atomic arrive + acquire spin).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/tmem_gridbar tools/micro/tmem_gridbar.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tst32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
}
__device__ __forceinline__ void tld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}

__global__ void __launch_bounds__(256, 1) tmem_kernel(int reps, unsigned long long *cyc, double *sink) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * (warp >> 2));
    uint32_t v[32];
    for (int q = 0; q < 32; ++q) v[q] = threadIdx.x * 32 + q;
    // write then read 8 chunks of 32 columns = this thread's 256 columns (128 doubles)
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int c = 0; c < 8; ++c) tst32(base + 32 * c, v);
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    unsigned long long t1 = clock64();
    double acc = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
            tld32(base + 32 * c, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            acc += v[(r + c) & 31];
        }
    }
    unsigned long long t2 = clock64();
    // read-modify-write (the CG pointwise pattern): ld, wait, fma, st
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int c = 0; c < 8; ++c) {
            tld32(base + 32 * c, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] += 1u;
            tst32(base + 32 * c, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    unsigned long long t3 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) {
        cyc[blockIdx.x * 3 + 0] = t1 - t0;
        cyc[blockIdx.x * 3 + 1] = t2 - t1;
        cyc[blockIdx.x * 3 + 2] = t3 - t2;
    }
    sink[blockIdx.x * 256 + threadIdx.x] = acc + v[0];
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

__device__ unsigned int g_count;
__device__ volatile unsigned int g_gen;

__global__ void __launch_bounds__(256, 1) gridbar_kernel(int reps, double *part, double *out) {
    __shared__ double s;
    unsigned int gen = 0;
    double acc = 0;
    for (int r = 0; r < reps; ++r) {
        if (threadIdx.x == 0) part[blockIdx.x] = acc + blockIdx.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            gen += 1;
            unsigned int prev;
            asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(prev) : "l"(&g_count) : "memory");
            const unsigned int target = gen * gridDim.x;
            unsigned int cur = prev + 1;
            while (cur < target) asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(&g_count) : "memory");
        }
        __syncthreads();
        // every CTA re-reduces all partials (the deterministic reduction)
        double v = 0;
        for (int b = threadIdx.x; b < gridDim.x; b += 256) v += __ldcg(part + b);
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if ((threadIdx.x & 31) == 0 && threadIdx.x < 32) s = v;
        __syncthreads();
        acc += s * 1e-9;
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *cyc;
    double *sink, *part, *out;
    cudaMalloc(&cyc, nsm * 3 * 8);
    cudaMalloc(&sink, nsm * 256 * 8);
    cudaMalloc(&part, nsm * 8);
    cudaMalloc(&out, nsm * 8);
    const int reps = 200;
    tmem_kernel<<<nsm, 256>>>(reps, cyc, sink);
    cudaError_t e = cudaDeviceSynchronize();
    printf("tmem: %s\n", cudaGetErrorString(e));
    unsigned long long h[3 * 200];
    cudaMemcpy(h, cyc, nsm * 3 * 8, cudaMemcpyDeviceToHost);
    const double bytes = double(reps) * 8 * 32 * 4 * 256;  // per SM
    printf("per SM: st %.1f B/cyc, ld(wait each) %.1f B/cyc, rmw %.1f B/cyc moved each way\n", bytes / h[0],
           bytes / h[1], bytes / h[2]);
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    void *args[] = {(void *)&reps, (void *)&part, (void *)&out};
    int greps = 2000;
    void *gargs[] = {(void *)&greps, (void *)&part, (void *)&out};
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int it = 0; it < 3; ++it) {
        cudaEventRecord(a);
        e = cudaLaunchCooperativeKernel((void *)gridbar_kernel, nsm, 256, gargs, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("gridbar (%s): %.3f us per barrier+reduce over %d CTAs\n", cudaGetErrorString(e),
               ms * 1e3 / greps, nsm);
    }
    (void)args;
    return 0;
}
