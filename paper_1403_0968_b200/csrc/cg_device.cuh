// cg_device.cuh -- device-side CG bookkeeping shared by the two K1 kernels
// (ax_kernel<N,true> and ax_tma_kernel<N,true>).  Included by .cu files only.
#pragma once
#include "sem_internal.h"

namespace sem {

struct CgStep {
    bool done;            // stopping rule fired (or fired earlier): kernel is a no-op
    int k;                // current iteration
    double beta;          // rho_k / rho_{k-1}  (0 at k = 0)
    double alpha_prev;    // alpha_{k-1}        (0 at k = 0)
    double *x;            // the caller's x of this solve
};

__device__ __forceinline__ double sum_rank_slot(const double *rr_all, int slot, int nranks) {
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s += __ldcg(rr_all + slot * nranks + q);
    return s;
}

// Stopping rule of SURVEY.md §8(c) O7, evaluated identically by every block:
// stop before iteration k when k >= maxit or sqrt(rho_k) <= tol sqrt(rho_0)
// (rho_0 == 0: stop with rel_res 0).  Block 0 records the outcome; the flag
// is sticky so every later kernel of this solve is a no-op.
__device__ __forceinline__ CgStep cg_k1_prologue(CgState *st, const double *rr_all, int nranks) {
    CgStep c{};
    if (*(volatile int32_t *)&st->done) {
        c.done = true;
        return c;
    }
    const int k = *(volatile int32_t *)&st->kcur;
    c.k = k;
    const double rho = sum_rank_slot(rr_all, k & 3, nranks);
    const double rho0 = (k == 0) ? rho : __ldcg(&st->rho0);
    bool done;
    if (k == 0 && rho0 == 0.0) done = true;
    else done = !(k < st->maxit && sqrt(rho) > st->tol * sqrt(rho0));
    if (done) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->rho0 = rho0;
            st->iters = k;
            st->rel_res = (rho0 == 0.0) ? 0.0 : sqrt(rho) / sqrt(rho0);
            st->converged = (rho0 == 0.0) || !(sqrt(rho) > st->tol * sqrt(rho0));
            __threadfence();
            st->done = 1;
        }
        c.done = true;
        return c;
    }
    if (k == 0) {
        if (blockIdx.x == 0 && threadIdx.x == 0) st->rho0 = rho0;
    } else {
        c.beta = rho / sum_rank_slot(rr_all, (k - 1) & 3, nranks);
        c.alpha_prev = __ldcg(&st->alpha[(k - 1) & 3]);
    }
    c.x = reinterpret_cast<double *>(__ldcg(reinterpret_cast<const unsigned long long *>(&st->xptr)));
    return c;
}

}  // namespace sem
