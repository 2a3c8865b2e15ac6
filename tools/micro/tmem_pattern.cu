// TMEM access patterns of the resident CG's R phase: per
// element slot i a thread loads 16 columns (r, w) + 1 column (meta), waits,
// computes, stores 8 columns (r).  Cycles per element slot for variants:
//   0: ld16 + ld1, wait, st8           (the kernel's R loop)
//   1: ld16 + ld1, wait                 (no store)
//   2: ld16, wait, st8                  (no meta column)
//   3: two slots: ld16 x2 + ld1 x2, wait, st8 x2
//   4: ld16 + ld1, wait, st8, wait::st  (store completion each slot)
//   5: bulk-copy issue cost: one thread issues 2 x 24 KB cp.async.bulk from
//      global (cold) and waits; cycles at the issuing thread for the issue only
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/tmem_pattern tools/micro/tmem_pattern.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define LD16(ta, v)                                                                                      \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), \
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),       \
                   "=r"(v[15])                                                                           \
                 : "r"(ta))
#define LD1(ta, x) asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(x) : "r"(ta))
#define ST8(ta, v)                                                                                       \
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(v[0]), \
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])                   \
                 : "memory")
#define WLD() asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory")
#define WST() asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory")

__global__ void __launch_bounds__(256, 1) k(int mode, int reps, unsigned long long *cyc, uint32_t *sink,
                                            const double *gsrc) {
    __shared__ uint32_t tbase;
    __shared__ __align__(128) double buf[2][2048];
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, g = warp >> 2;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(256 * g);
    uint32_t v[16], w[16], acc = 0, m0 = 0, m1 = 0;
    for (int q = 0; q < 16; ++q) v[q] = w[q] = threadIdx.x + q;
    __syncthreads();
    unsigned long long t0 = clock64();
    if (mode == 5) {
        if (threadIdx.x == 0) {
            uint32_t ph = 0;
            unsigned long long ti = 0;
            for (int r = 0; r < reps; ++r) {
                const uint32_t bb = (uint32_t)__cvta_generic_to_shared(&bar);
                unsigned long long a0 = clock64();
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(2 * 16384) : "memory");
                for (int h = 0; h < 2; ++h)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     (uint32_t)__cvta_generic_to_shared(&buf[h][0])),
                                 "l"(gsrc + (size_t)(blockIdx.x * reps + r) * 6144 + h * 2048), "r"(16384), "r"(bb)
                                 : "memory");
                ti += clock64() - a0;
                asm volatile(
                    "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(bb),
                    "r"(ph)
                    : "memory");
                ph ^= 1;
            }
            cyc[blockIdx.x] = ti;
        }
        __syncthreads();
    } else {
        for (int r = 0; r < reps; ++r) {
#pragma unroll 1
            for (int i = 0; i < 14; i += (mode == 3 ? 2 : 1)) {
                const uint32_t a = tb + 16 * i;
                if (mode == 0 || mode == 1 || mode == 4) {
                    LD16(a, v);
                    LD1(tb + 224 + i, m0);
                    WLD();
                } else if (mode == 2) {
                    LD16(a, v);
                    WLD();
                } else {
                    LD16(a, v);
                    LD16(a + 16, w);
                    LD1(tb + 224 + i, m0);
                    LD1(tb + 225 + i, m1);
                    WLD();
                }
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    v[q] += m0;
                    w[q] += m1;
                }
                if (mode != 1) ST8(a, v);
                if (mode == 3) ST8(a + 16, w);
                if (mode == 4) WST();
                acc += v[3] + w[5];
            }
        }
        WST();
        __syncthreads();
        if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
    }
    sink[blockIdx.x * 256 + threadIdx.x] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long *cyc;
    uint32_t *sink;
    double *gsrc;
    const int reps = 100;
    cudaMalloc(&cyc, nsm * 8);
    cudaMalloc(&sink, nsm * 256 * 4);
    cudaMalloc(&gsrc, (size_t)nsm * reps * 6144 * 8);
    cudaMemset(gsrc, 0, (size_t)nsm * reps * 6144 * 8);
    const char *names[] = {"ld16+ld1,wait,st8", "ld16+ld1,wait", "ld16,wait,st8", "2 slots batched",
                           "ld16+ld1,wait,st8,wait::st", "bulk issue 2x16KB (cycles per issue pair)"};
    for (int mode = 0; mode < 6; ++mode) {
        k<<<nsm, 256>>>(mode, reps, cyc, sink, gsrc);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[256];
        cudaMemcpy(h, cyc, nsm * 8, cudaMemcpyDeviceToHost);
        double mx = 0, av = 0;
        for (int b = 0; b < nsm; ++b) {
            av += h[b];
            mx = h[b] > mx ? h[b] : mx;
        }
        av /= nsm;
        const double per = mode == 5 ? av / reps : av / (reps * 14.0);
        printf("mode %d %-45s %s: %.1f cycles per %s (avg over SMs; max SM %.1f)\n", mode, names[mode],
               cudaGetErrorString(e), per, mode == 5 ? "issue" : "slot", mode == 5 ? mx / reps : mx / (reps * 14.0));
    }
    return 0;
}
