// cg_device.cuh -- device-side CG bookkeeping shared by K1 (ax_kernel<N,true>,
// ax_tma_kernel<N,true>) and K2 (k2_kernel).  Included by .cu files only.
//
// Reductions are DEFERRED to the consumer: a producing kernel only writes one
// partial per block (no atomics, no last-block tail); every block of the
// consuming kernel re-reduces the few hundred partials in the same fixed order
// (so all blocks, and all runs, see bit-identical scalars) while its own bulk
// loads are already in flight.  Scalars of iteration k:
//     rho_k  = (r_k, r_k)_c   partials of K2(k-1)  (K2(-1) = the CG start)
//     pap_k  = (p_k, A p_k)   partials of K1(k)
//     alpha_k = rho_k / pap_k,  beta_k = rho_k / rho_{k-1}
// Jacobi PCG (CgRed::pc, NEXT-2): rho_k = (r_k, z_k)_c from K2's second set of
// partials drives alpha and beta; rr_k = (r_k, r_k)_c still drives the stopping
// rule (reading R4).  Without pc rr_k = rho_k.
// With nranks > 1 a one-block kernel folds the partials into this rank's
// value, NCCL all-gathers it, and consumers sum the ranks in ascending order.
#pragma once
#include <cstdlib>

#include "sem_internal.h"

namespace sem {

// Programmatic dependent launch: the CG kernels are launched with
// programmaticStreamSerialization (opt-in, SEM_PDL=1); each waits for its
// predecessor's memory before touching data the predecessor produced.
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
    // off by default: with the trigger at kernel start measured slower on c3
    // (dependents parked at griddepcontrol.wait hold SM slots the primary's
    // tail could use: 46.1 vs 44.4 us/it, r02); with the trigger at the end
    // of K1's / K2's work (SEM_PDL_LATE, now the placement) within noise
    // (bench 47.6-47.8 vs 47.4-47.5 GDOF/s; the full GPU suite passes with it)
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

// gpu-scope relaxed load of a state word written by an earlier kernel.
__device__ __forceinline__ int32_t ld_state(const int32_t *p) {
    int32_t v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Deterministic block reduction of NV values per thread: fixed shuffle tree
// per warp, then the warp results summed in warp order.  Result in every
// thread (broadcast through shared memory).  red: >= NV * (NT/32) doubles.
template <int NT, int NV>
__device__ __forceinline__ void block_sum_vec(double (&v)[NV], double *red) {
    constexpr int NW = (NT + 31) / 32;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) red[q * NW + wid] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double s = 0.0;
        for (int w = 0; w < NW; ++w) s += red[q * NW + w];
        v[q] = s;
    }
    __syncthreads();
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double *red) {
    double a[1] = {v};
    block_sum_vec<NT, 1>(a, red);
    return a[0];
}

// Where the per-block partials of the two reductions live (see top).
struct CgRed {
    const double *part1;   // [2][s1] K1 partials of (p, A p), parity of k
    const double *part2;   // [2][s2] K2 partials of (r, r), parity of the producing k
    int nb1, s1, nb2, s2;
    const double *pap_all; // nranks > 1: [4][nranks] all-gathered rank values
    const double *rr_all;
    int nranks;
    // 1: Jacobi PCG, rho from the (r, z) partials, which sit right after the
    // (r, r) ones: part3 = part2 + 2 s2 and rz_all = rr_all + kRing nranks
    // (derived, not stored: the kernels' parameter blocks keep their size --
    // K1's register allocation is sensitive to it)
    int pc;
};

inline CgRed make_red(const DevMesh &m, const CgVecs &v) {
    CgRed R;
    R.part1 = v.part1;
    R.part2 = v.part2;
    R.nb1 = v.nb1;
    R.s1 = v.s1;
    R.nb2 = v.nb2;
    R.s2 = v.s2;
    R.pap_all = v.pap_all;
    R.rr_all = v.rr_all;
    R.nranks = m.nranks;
    R.pc = v.dinv != nullptr;
    return R;
}

// Location of the values whose ordered sum is rr_k = (r_k, r_k)_c (the
// stopping norm), rho_k (= rr_k, or (r_k, z_k)_c with pc) and pap_k.
__device__ __forceinline__ void rr_src(const CgRed &R, int k, const double *&p, int &n) {
    if (R.nranks == 1) {
        p = R.part2 + ((k - 1) & 1) * R.s2;
        n = R.nb2;
    } else {
        p = R.rr_all + (k & 3) * R.nranks;
        n = R.nranks;
    }
}
__device__ __forceinline__ void pap_src(const CgRed &R, int k, const double *&p, int &n) {
    if (R.nranks == 1) {
        p = R.part1 + (k & 1) * R.s1;
        n = R.nb1;
    } else {
        p = R.pap_all + (k & 3) * R.nranks;
        n = R.nranks;
    }
}

// Block-cooperative ordered sums of NV sources (each <= ~1000 values): every
// thread loads its share of all sources in one batch (one round trip), then
// one block reduction.  Identical result in every block.
template <int NT, int NV>
__device__ __forceinline__ void block_sums(const double *const (&src)[NV], const int (&cnt)[NV],
                                           double (&out)[NV], double *red) {
    constexpr int PER = 8;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double v[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int t = threadIdx.x + u * NT;
            v[u] = (t < cnt[q]) ? __ldcg(src[q] + t) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < PER; ++u) s += v[u];
        for (int t = threadIdx.x + PER * NT; t < cnt[q]; t += NT) s += __ldcg(src[q] + t);
        out[q] = s;
    }
    block_sum_vec<NT, NV>(out, red);
}

// Stopping rule of SURVEY.md §8(c) O7 before iteration k: stop when
// k >= maxit or sqrt(rho_k) <= tol sqrt(rho_0); rho_0 == 0 stops at once.
__device__ __forceinline__ bool cg_stop(int k, double rho, double rho0, int maxit, double tol) {
    if (k == 0 && rho0 == 0.0) return true;
    return !(k < maxit && sqrt(rho) > tol * sqrt(rho0));
}

struct CgStep {
    bool done;            // stop before this iteration (or stopped earlier): no-op
    int k;                // current iteration
    double beta;          // beta_k  (0 at k = 0)
    double alpha_prev;    // alpha_{k-1} (0 at k = 0)
};

// Location of the rho_k sources for a compile-time preconditioner flag.
template <bool PC>
__device__ __forceinline__ void rho_src_t(const CgRed &R, int k, const double *&p, int &n) {
    if constexpr (PC) {
        if (R.nranks == 1) {
            p = R.part2 + 2 * R.s2 + ((k - 1) & 1) * R.s2;
            n = R.nb2;
        } else {
            p = R.rr_all + kRing * R.nranks + (k & 3) * R.nranks;
            n = R.nranks;
        }
    } else {
        rr_src(R, k, p, n);
    }
}

// One thread's share of an ordered partial sum (the per-thread part of
// block_sums: PER strided values, then the tail).
template <int NT>
__device__ __forceinline__ double thread_sum(const double *src, int cnt) {
    constexpr int PER = 8;
    double v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int t = threadIdx.x + u * NT;
        v[u] = (t < cnt) ? __ldcg(src + t) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < PER; ++u) s += v[u];
    for (int t = threadIdx.x + PER * NT; t < cnt; t += NT) s += __ldcg(src + t);
    return s;
}

// The scalars' sources of iteration k.  One rank: the partial slots are
// selected by the parity of k, which is itself read from the state, so both
// parities are summed speculatively in the SAME round trip as the state
// loads (the slot of the wrong parity may be written concurrently by this
// very kernel's blocks; its sum is discarded) -- one memory round trip
// instead of two.  Several ranks: the all-gathered rank values, after k.
// K1 prologue (all threads of the block): k, the stopping decision, beta_k
// and alpha_{k-1}.  Block 0 records a stop for the host (iters, rel_res,
// alpha_{it-1} for the final x update, the sticky flag) and, at k = 0, rr_0.
// PC: rho = (r,z) drives alpha / beta, rr = (r,r) the stop.  Only K1 takes the
// stopping decision (K2 follows the sticky flag).  Split in two so a kernel can
// issue the scalar loads BEFORE its bulk copies (they would otherwise queue
// behind them: ncu r01g put 25% of K1's stall samples in the prologue):
//   cg_k1_load    state + partial loads, per-thread partial sums (no barrier)
//   cg_k1_finish  block reduction (__syncthreads), decisions, state writes
template <bool PC>
struct K1Pre {
    static constexpr int NS = PC ? 4 : 3;     // sums: rho_k, rho_{k-1}, pap_{k-1} [, rr_k]
    static constexpr int NL = PC ? 6 : 4;     // loaded partial sets (both parities)
    static constexpr int PER = 4;             // loads in flight per thread and set
    int done, k, maxit, multi;
    double tol, rho0;
    double raw[NL][PER];
    double v[NS];
};

// first PER strided values of one partial set (issued, not consumed)
template <int NT, int PER>
__device__ __forceinline__ void thread_load(const double *src, int cnt, double (&v)[PER]) {
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int t = threadIdx.x + u * NT;
        v[u] = (t < cnt) ? __ldcg(src + t) : 0.0;
    }
}
template <int NT, int PER>
__device__ __forceinline__ double thread_finish(const double *src, int cnt, const double (&v)[PER]) {
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < PER; ++u) s += v[u];
    for (int t = threadIdx.x + PER * NT; t < cnt; t += NT) s += __ldcg(src + t);
    return s;
}

// Issue every load of the prologue (state words, partials of both parities)
// without consuming any, so a kernel can put its bulk copies behind them and
// only then wait (cg_k1_finish).
template <int NT, bool PC>
__device__ __forceinline__ void cg_k1_load(CgState *st, const CgRed &R, K1Pre<PC> &P) {
    constexpr int NS = K1Pre<PC>::NS, PER = K1Pre<PC>::PER;
    P.done = ld_state(&st->done);
    P.k = ld_state(&st->k1);
    P.maxit = st->maxit;
    P.tol = st->tol;
    P.rho0 = __ldcg(&st->rho0);
    P.multi = R.nranks > 1;
    if (!P.multi) {
        // rho sources: part2 ((r,r)) or part3 ((r,z)); pap: part1
        const double *prho = PC ? R.part2 + 2 * R.s2 : R.part2;
        thread_load<NT, PER>(prho, R.nb2, P.raw[0]);
        thread_load<NT, PER>(prho + R.s2, R.nb2, P.raw[1]);
        thread_load<NT, PER>(R.part1, R.nb1, P.raw[2]);
        thread_load<NT, PER>(R.part1 + R.s1, R.nb1, P.raw[3]);
        if constexpr (PC) {
            thread_load<NT, PER>(R.part2, R.nb2, P.raw[4]);
            thread_load<NT, PER>(R.part2 + R.s2, R.nb2, P.raw[5]);
        }
    } else {
        const int k = P.k;
        const double *src[NS];
        int cnt[NS];
        rho_src_t<PC>(R, k, src[0], cnt[0]);     // rho_k
        rho_src_t<PC>(R, k - 1, src[1], cnt[1]); // rho_{k-1}
        pap_src(R, k - 1, src[2], cnt[2]);       // pap_{k-1}
        if (k == 0) cnt[1] = cnt[2] = 0;
        if constexpr (PC) rr_src(R, k, src[NS - 1], cnt[NS - 1]);   // rr_k (stopping norm)
#pragma unroll
        for (int q = 0; q < NS; ++q) P.v[q] = thread_sum<NT>(src[q], cnt[q]);
    }
}

template <int NT, bool PC>
__device__ __forceinline__ CgStep cg_k1_finish(CgState *st, const CgRed &R, double *red,
                                               K1Pre<PC> &P) {
    constexpr int NS = K1Pre<PC>::NS, PER = K1Pre<PC>::PER;
    CgStep c{};
    const int k = P.k;
    c.k = k;
    if (P.done) {
        c.done = true;
        return c;
    }
    if (!P.multi) {
        const double *prho = PC ? R.part2 + 2 * R.s2 : R.part2;
        const double r0 = thread_finish<NT, PER>(prho, R.nb2, P.raw[0]);
        const double r1 = thread_finish<NT, PER>(prho + R.s2, R.nb2, P.raw[1]);
        const double q0 = thread_finish<NT, PER>(R.part1, R.nb1, P.raw[2]);
        const double q1 = thread_finish<NT, PER>(R.part1 + R.s1, R.nb1, P.raw[3]);
        const bool odd = (k - 1) & 1;           // parity of the slots of rho_k, pap_{k-1}
        P.v[0] = odd ? r1 : r0;                   // rho_k
        P.v[1] = (k == 0) ? 0.0 : (odd ? r0 : r1);   // rho_{k-1}
        P.v[2] = (k == 0) ? 0.0 : (odd ? q1 : q0);   // pap_{k-1}
        if constexpr (PC) {
            const double rr0 = thread_finish<NT, PER>(R.part2, R.nb2, P.raw[4]);
            const double rr1 = thread_finish<NT, PER>(R.part2 + R.s2, R.nb2, P.raw[5]);
            P.v[NS - 1] = odd ? rr1 : rr0;        // rr_k (stopping norm)
        }
    }
    block_sum_vec<NT, NS>(P.v, red);
    const double rho = P.v[0], rho_m1 = P.v[1], pap_m1 = P.v[2];
    const double rr = P.v[NS - 1 - (PC ? 0 : 2)];
    const double rho0 = (k == 0) ? rr : P.rho0;
    const double alpha_prev = (k == 0) ? 0.0 : rho_m1 / pap_m1;
    c.beta = (k == 0) ? 0.0 : rho / rho_m1;
    c.alpha_prev = alpha_prev;
    c.done = cg_stop(k, rr, rho0, P.maxit, P.tol);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (k == 0) st->rho0 = rho0;
        st->k2 = k;                      // for K2 of this iteration
        if (c.done) {
            st->iters = k;
            st->rel_res = (rho0 == 0.0) ? 0.0 : sqrt(rr) / sqrt(rho0);
            st->converged = (rho0 == 0.0) || !(sqrt(rr) > P.tol * sqrt(rho0));
            st->alpha_km1 = alpha_prev;
            __threadfence();
            st->done = 1;
        }
    }
    return c;
}

template <int NT, bool PC>
__device__ __forceinline__ CgStep cg_k1_prologue_t(CgState *st, const CgRed &R, double *red) {
    K1Pre<PC> P;
    cg_k1_load<NT, PC>(st, R, P);
    return cg_k1_finish<NT, PC>(st, R, red, P);
}

// The PCG prologue is kept out of line so the CG kernels' main loops compile
// exactly as without a preconditioner (K1's register allocation is sensitive).
template <int NT>
__device__ __noinline__ CgStep cg_k1_prologue_pc(CgState *st, const CgRed &R, double *red) {
    return cg_k1_prologue_t<NT, true>(st, R, red);
}

template <int NT>
__device__ __forceinline__ CgStep cg_k1_prologue(CgState *st, const CgRed &R, double *red) {
    if (R.pc) return cg_k1_prologue_pc<NT>(st, R, red);
    return cg_k1_prologue_t<NT, false>(st, R, red);
}

// K2 prologue (all threads): k and alpha_k = rho_k / pap_k.  The stopping
// decision of iteration k was taken by K1(k) (sticky flag): K2 only follows
// it, so the two kernels can never disagree.  K2 is instantiated per
// preconditioner (k2_kernel<N, INIT, PC>).  Split like K1's: cg_k2_load
// issues every load (both parities), cg_k2_finish consumes them.
struct K2Pre {
    // loads in flight per thread and partial set: 2 x 256 threads cover the
    // K2 grid's 444 (r,r) partials and K1's <= 148 (p,Ap) partials in one
    // round trip (a tail loop takes any rest)
    static constexpr int PER = 2;
    int done, k, multi;
    double raw[4][PER];
    double v[2];
};

template <int NT, bool PC>
__device__ __forceinline__ void cg_k2_load(CgState *st, const CgRed &R, K2Pre &P) {
    constexpr int PER = K2Pre::PER;
    P.done = ld_state(&st->done);
    P.k = ld_state(&st->k2);
    P.multi = R.nranks > 1;
    if (!P.multi) {
        const double *prho = PC ? R.part2 + 2 * R.s2 : R.part2;
        thread_load<NT, PER>(prho, R.nb2, P.raw[0]);
        thread_load<NT, PER>(prho + R.s2, R.nb2, P.raw[1]);
        thread_load<NT, PER>(R.part1, R.nb1, P.raw[2]);
        thread_load<NT, PER>(R.part1 + R.s1, R.nb1, P.raw[3]);
    } else {
        const int k = P.k;
        const double *src[2];
        int cnt[2];
        rho_src_t<PC>(R, k, src[0], cnt[0]);     // rho_k
        pap_src(R, k, src[1], cnt[1]);           // pap_k
        P.v[0] = thread_sum<NT>(src[0], cnt[0]);
        P.v[1] = thread_sum<NT>(src[1], cnt[1]);
    }
}

template <int NT, bool PC>
__device__ __forceinline__ CgStep cg_k2_finish(CgState *st, const CgRed &R, double *red, K2Pre &P,
                                               double &alpha) {
    constexpr int PER = K2Pre::PER;
    CgStep c{};
    const int k = P.k;
    c.k = k;
    if (P.done) {
        c.done = true;
        return c;
    }
    if (!P.multi) {
        const double *prho = PC ? R.part2 + 2 * R.s2 : R.part2;
        const double r0 = thread_finish<NT, PER>(prho, R.nb2, P.raw[0]);
        const double r1 = thread_finish<NT, PER>(prho + R.s2, R.nb2, P.raw[1]);
        const double q0 = thread_finish<NT, PER>(R.part1, R.nb1, P.raw[2]);
        const double q1 = thread_finish<NT, PER>(R.part1 + R.s1, R.nb1, P.raw[3]);
        P.v[0] = ((k - 1) & 1) ? r1 : r0;        // rho_k
        P.v[1] = (k & 1) ? q1 : q0;              // pap_k
    }
    block_sum_vec<NT, 2>(P.v, red);
    alpha = P.v[0] / P.v[1];
    if (blockIdx.x == 0 && threadIdx.x == 0) st->k1 = k + 1;   // for K1 of k+1
    return c;
}

}  // namespace sem
