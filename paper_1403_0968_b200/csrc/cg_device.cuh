// cg_device.cuh -- device-side CG bookkeeping shared by the two K1 kernels
// (ax_kernel<N,true> and ax_tma_kernel<N,true>).  Included by .cu files only.
#pragma once
#include <cstdlib>

#include "sem_internal.h"

namespace sem {

struct CgStep {
    bool done;            // stopping rule fired (or fired earlier): kernel is a no-op
    int k;                // current iteration
    double beta;          // rho_k / rho_{k-1}  (0 at k = 0)
    double alpha_prev;    // alpha_{k-1}        (0 at k = 0)
};

// Programmatic dependent launch: the CG kernels are launched with
// programmaticStreamSerialization; each waits for its predecessor's memory
// before touching data the predecessor produced, and lets its successor
// launch early (its launch latency and static-data prologue then overlap).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem,
                              cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    // off by default: measured slower on c3 (dependents parked at
    // griddepcontrol.wait hold SM slots the primary's tail could use)
    static const bool enabled = [] {
        const char *e = getenv("SEM_PDL");
        return e && e[0] == '1';
    }();
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = enabled ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Deterministic block reduction: fixed shuffle tree per warp, then thread 0
// sums the warp results in warp order.  Valid in thread 0 only.
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    constexpr int NW = (NT + 31) / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
        for (int q = 0; q < NW; ++q) s += red[q];
    }
    return s;
}

// Fixed-order sum of cnt partials by one whole block (deterministic for a
// fixed blockDim).  The first 16*NT partials are loaded in one unrolled batch
// (one L2 round trip instead of a dependent chain).  Valid in thread 0.
template <int NT>
__device__ double block_sum_array(const double *a, int cnt, double *red) {
    constexpr int PER = 16;
    double v[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const int t = threadIdx.x + q * NT;
        v[q] = (t < cnt) ? __ldcg(a + t) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < PER; ++q) s += v[q];
    for (int t = threadIdx.x + PER * NT; t < cnt; t += NT) s += __ldcg(a + t);
    return block_sum<NT>(s, red);
}

// Last-block-done protocol: every block has written its partial (thread 0);
// returns true in the block that arrived last, which then sees all partials.
// Only thread 0 fences: the other threads' stores need not be ordered.
__device__ __forceinline__ bool last_block(uint32_t *ticket, int *sflag) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t t = atomicAdd(ticket, 1u);
        *sflag = (t == gridDim.x - 1);
    }
    __syncthreads();
    const bool last = *sflag;
    if (last) __threadfence();
    return last;
}

// gpu-scope relaxed load of a state word written by an earlier kernel (or the
// last block of this one): no system-scope strong access, no L1 reuse.
__device__ __forceinline__ int32_t ld_state(const int32_t *p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ double sum_rank_slot(const double *rr_all, int slot, int nranks) {
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s += __ldcg(rr_all + slot * nranks + q);
    return s;
}

// ---------------------------------------------------------------------------
// CG scalar bookkeeping.  The kernel that completes a global reduction (its
// last block, or a one-thread finaliser after the multi-rank all-gather)
// derives the next scalars, so a consumer kernel needs ONE round trip of
// independent loads, not a chain.
// ---------------------------------------------------------------------------

// End of iteration k (k_next = k + 1), or CG start (k_next = 0, rho = rho_0):
// records rho_{k+1}, beta_{k+1} = rho_{k+1} / rho_k, alpha_k for K1's deferred
// x update, advances k, and evaluates the stopping rule of SURVEY.md §8(c) O7
// for iteration k_next: stop when k_next >= maxit or sqrt(rho) <= tol sqrt(rho_0)
// (rho_0 == 0: stop with rel_res 0).  The done flag is sticky: every later
// kernel of this solve is a no-op.  One thread.
__device__ __forceinline__ void cg_finalize_rho(CgState *st, int k_next, double rho) {
    double rho0;
    if (k_next == 0) {
        rho0 = rho;
        st->rho0 = rho;
        st->beta = 0.0;
        st->alpha_km1 = 0.0;
    } else {
        rho0 = st->rho0;
        st->beta = rho / st->rho_cur;
        st->alpha_km1 = st->alpha_k;
    }
    st->rho_cur = rho;
    bool done;
    if (k_next == 0 && rho0 == 0.0) done = true;
    else done = !(k_next < st->maxit && sqrt(rho) > st->tol * sqrt(rho0));
    if (done) {
        st->iters = k_next;
        st->rel_res = (rho0 == 0.0) ? 0.0 : sqrt(rho) / sqrt(rho0);
        st->converged = (rho0 == 0.0) || !(sqrt(rho) > st->tol * sqrt(rho0));
    }
    __threadfence();
    st->kcur = k_next;
    if (done) st->done = 1;
}

// After K1 of iteration k: alpha_k = rho_k / (p, A p).  One thread.
__device__ __forceinline__ void cg_finalize_pap(CgState *st, double pap) {
    st->alpha_k = st->rho_cur / pap;
}

// K1 prologue: one round trip of independent state loads.
__device__ __forceinline__ CgStep cg_k1_prologue(CgState *st) {
    CgStep c{};
    const int done = ld_state(&st->done);
    const int k = ld_state(&st->kcur);
    const double beta = __ldcg(&st->beta);
    const double am1 = __ldcg(&st->alpha_km1);
    c.done = done != 0;
    c.k = k;
    c.beta = beta;
    c.alpha_prev = am1;
    return c;
}

}  // namespace sem
