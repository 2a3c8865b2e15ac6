// ax_tma.cuh -- TMA-pipelined, persistent sm_100a kernels for the local stiffness
// apply w = A_L u (eq:semOperator) and its fused CG variant
// K1 (x += alpha_{k-1} p_{k-1}; p = r + beta_k p_{k-1}; w = A_L p; (w,p) over
// element-interior nodes).  Used for N <= kTmaMaxN; larger N use ax_kernel.
//
// Design:
//  * one CTA per SM (persistent); the CTA holds NG independent "groups" of GT
//    threads; a group works on a UNIT of EPG consecutive elements at a time,
//    thread (i,j) of element el owning the k-column of nodes (i,j,0..N).
//  * every group double-buffers its units in shared memory: the group leader
//    issues 1-D bulk copies (cp.async.bulk, TMA engine) of the unit's input
//    vectors and its six geometric-factor blocks, completing on an mbarrier
//    with expect_tx; while the group computes unit t, unit t+1 is in flight.
//    G^ is streamed exactly once (L2 evict_first policy); nothing is re-read.
//  * sum factorisation: u_r and u_s from the k-slice in shared memory (D rows
//    of the thread in registers), u_t from the register column with D in
//    constant memory (uniform index -> constant-bank operand); f_r, f_s are
//    written over the thread's own (already consumed) G^ slots, f_t stays in
//    registers; the transposed contraction reads f_r, f_s after one group
//    barrier.  FP64 FMA throughout.
//  * MASS = true adds the lumped screened-Coulomb mass term w += h u with
//    h = alpha w_i w_j w_k J (NEXT-1), h read per column into
//    registers while the unit's copies fly.  The h pointer travels in the
//    field the variant does not use (u for CG, r for the plain apply) so the
//    parameter block -- and the Poisson kernels' code generation -- is unchanged.
//
// Included by ax_tma.cu (Poisson instantiations) and ax_tma_mass.cu (MASS),
// compiled as separate translation units; each has its own copy of c_D.
#pragma once
#include <cstdio>

#include "cg_device.cuh"
#include "sem_internal.h"

namespace sem {

// ---------------------------------------------------------------------------
// D in constant memory, one block per order N (values depend on N only).
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int d_off(int N) {
    int o = 0;
    for (int q = 1; q < N; ++q) o += (q + 1) * (q + 1);
    return o;
}
constexpr int kDConstTotal = d_off(16);
static __constant__ double c_D[kDConstTotal];   // one copy per translation unit

static cudaError_t upload_D_this_tu(int N, const double *D_host) {
    return cudaMemcpyToSymbol(c_D, D_host, sizeof(double) * (N + 1) * (N + 1),
                              sizeof(double) * d_off(N), cudaMemcpyHostToDevice);
}

// ---------------------------------------------------------------------------
// per-N configuration
// ---------------------------------------------------------------------------
template <int N>
struct TmaCfg {
    static constexpr int n = N + 1, n2 = n * n, n3 = n2 * n;
    // elements per unit (packs small elements into ~64-128 threads)
    static constexpr int EPG = (N == 1) ? 16 : (N == 2) ? 7 : (N == 3) ? 4 : (N == 4) ? 5
                             : (N == 5) ? 3 : (N == 6) ? 2 : 1;
    static constexpr int GT = ((EPG * n2 + 31) / 32) * 32;   // threads per group
    static constexpr int VL = ((EPG * n3 + 2 + 1) / 2) * 2;  // vector slot (doubles)
};

template <int N, bool CG>
struct TmaLayout {
    using C = TmaCfg<N>;
    static constexpr int NV = CG ? 3 : 1;                           // r,p,x | u
    static constexpr int STAGE = NV * C::VL + 6 * C::EPG * C::n3;   // doubles
    static constexpr int SMEM_MAX = 227 * 1024 - 1024;
    static constexpr int NG_FIT = SMEM_MAX / (2 * STAGE * 8);
    static constexpr int NG = NG_FIT > 4 ? 4 : NG_FIT;              // groups per CTA
    static constexpr int NT = NG * C::GT;
    static constexpr size_t SMEM = size_t(NG) * 2 * STAGE * 8 + 128;
};

// ---------------------------------------------------------------------------
// PTX helpers (mbarrier + bulk copy)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void group_bar(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 16-byte aligned superset [a0, a1) (in doubles) of the E-vector range
// [first, first + nd) for a bulk copy; element data then starts at smem slot
// + (first - a0).  When the superset would run past the end L of the caller's
// buffer, a1 is pulled back and the last double(s) are copied by plain loads
// (no over-read).
struct VecRange {
    int64_t a0, a1;
};
__device__ __forceinline__ VecRange vec_range(int64_t first, int64_t nd, int64_t L) {
    VecRange r;
    r.a0 = first & ~int64_t(1);
    r.a1 = (first + nd + 1) & ~int64_t(1);
    if (r.a1 > L) r.a1 -= 2;
    return r;
}

// expect_tx without an arrival (the arrival comes later, after the plain-load
// tails are in shared memory) and a plain arrival (release semantics).
__device__ __forceinline__ void mbar_expect_tx_only(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct TmaArgs {
    int64_t E;
    const double *G;
    // plain: u -> w.  CG: r, p (in/out), x (in/out, the solve's x work vector) -> w
    const double *u;
    const double *r;
    double *p, *x, *w;
    CgRed red;            // where the scalar reductions live
    double *part1;        // this kernel's (p, A p) partials, [2][s1]
    CgState *st;
};

// PC: Jacobi PCG scalars (cg_k1_prologue_t); a separate instantiation so the
// CG kernel's code is unchanged (ax_tma_pc.cu).
// DOT (with CG = false): KA of the single-reduction CG (NEXT-3, ax_tma_sr.cu):
// the plain apply w = A_L u plus per-CTA partials of (u, A_L u) = (u, w)_c for
// continuous masked u; no scalars needed (only the iteration parity k1, and
// the sticky stop flag to skip iterations after the stop).
template <int N, bool CG, bool MASS, bool PC = false, bool DOT = false>
__global__ void __launch_bounds__(TmaLayout<N, CG>::NT, 1) ax_tma_kernel(TmaArgs a) {
    using C = TmaCfg<N>;
    using Lo = TmaLayout<N, CG>;
    constexpr int n = C::n, n2 = C::n2, n3 = C::n3, EPG = C::EPG, GT = C::GT, VL = C::VL;
    constexpr int NG = Lo::NG, NV = Lo::NV, STAGE = Lo::STAGE;
    constexpr int DO = d_off(N);
    extern __shared__ __align__(128) double smem[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + size_t(NG) * 2 * STAGE);  // [NG][2]
    __shared__ double sred[3 * ((Lo::NT + 31) / 32)];   // K1 prologue: up to 4 sums

    const int tid = threadIdx.x;
    const int g = tid / GT;                 // group
    const int gt = tid - g * GT;            // thread in group
    const int el = gt / n2;                 // element within unit
    const int elc = (el < EPG) ? el : 0;    // spare lanes address element 0 (results unused)
    const int ij = gt - el * n2;
    const int i = ij % n, j = ij / n;
    const bool lane_on = el < EPG;
    const bool leader = (gt == 0);
    double *stage0 = smem + size_t(g) * 2 * STAGE;
    uint64_t *gbar = bars + 2 * g;

    const int64_t nunits = (a.E + EPG - 1) / EPG;
    const int64_t TG = int64_t(gridDim.x) * NG;
    const int64_t u0 = int64_t(blockIdx.x) * NG + g;
    const int64_t L = a.E * n3;

    if (leader) {
        mbar_init(gbar + 0, 1);
        mbar_init(gbar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if constexpr (CG) pdl_trigger();   // let the gather-scatter grid launch early

    const uint64_t pol_g = policy_evict_first();
    const uint64_t pol_v = CG ? policy_evict_last() : policy_evict_first();

    // Leader, two steps per unit.  issue_G: expect the unit's bytes, start the
    // geometric-factor copy (static data: may run before the previous kernel
    // has finished).  issue_V: plain-load tails of the vectors into shared
    // memory, the arrival (release), then the vector bulk copies.
    auto unit_bytes = [&](int64_t unit, VecRange &vr, int64_t &first, int64_t &nd, uint32_t &vb,
                          uint32_t &gb) {
        const int64_t e0 = unit * EPG;
        const int64_t ne = (a.E - e0 < EPG) ? (a.E - e0) : EPG;
        first = e0 * n3;
        nd = ne * n3;
        vr = vec_range(first, nd, L);
        vb = (uint32_t)((vr.a1 - vr.a0) * 8);
        gb = (uint32_t)(ne * 6 * n3 * 8);
    };
    auto issue_G = [&](int64_t unit, int s) {
        VecRange vr;
        int64_t first, nd;
        uint32_t vb, gb;
        unit_bytes(unit, vr, first, nd, vb, gb);
        double *sb = stage0 + size_t(s) * STAGE;
        mbar_expect_tx_only(gbar + s, NV * vb + gb);
        bulk_g2s(sb + NV * VL, a.G + unit * EPG * 6 * n3, gb, gbar + s, pol_g);
    };
    auto issue_V = [&](int64_t unit, int s) {
        VecRange vr;
        int64_t first, nd;
        uint32_t vb, gb;
        unit_bytes(unit, vr, first, nd, vb, gb);
        double *sb = stage0 + size_t(s) * STAGE;
        const double *vsrc[3];
        if constexpr (CG) {
            vsrc[0] = a.r;
            vsrc[1] = a.p;
            vsrc[2] = a.x;
        } else {
            vsrc[0] = a.u;
        }
        for (int v = 0; v < NV; ++v)
            for (int64_t q = vr.a1; q < first + nd; ++q) sb[v * VL + (q - vr.a0)] = __ldg(vsrc[v] + q);
        mbar_arrive(gbar + s);
        for (int v = 0; v < NV; ++v) bulk_g2s(sb + v * VL, vsrc[v] + vr.a0, vb, gbar + s, pol_v);
    };

    // ---- the scalar loads of this iteration go out first (small, L2-resident:
    // ahead of the bulk copies in the memory queues), then the geometric
    // factors and the vectors produced by the previous kernels; the scalars
    // are reduced while all those copies are in flight ----
    K1Pre<PC> pre;
    if constexpr (CG) {
        pdl_wait();
        cg_k1_load<Lo::NT, PC>(a.st, a.red, pre);
    }
    int dot_done = 0, kit = 0;
    if constexpr (DOT) {
        dot_done = ld_state(&a.st->done);
        kit = ld_state(&a.st->k1);
    }
    if (leader) {
        if (u0 < nunits) issue_G(u0, 0);
        if (u0 + TG < nunits) issue_G(u0 + TG, 1);
        if (u0 < nunits) issue_V(u0, 0);
        if (u0 + TG < nunits) issue_V(u0 + TG, 1);
    }
    if constexpr (DOT) {
        if (dot_done) {
            if (leader) {
                if (u0 < nunits) mbar_wait(gbar + 0, 0);
                if (u0 + TG < nunits) mbar_wait(gbar + 1, 0);
            }
            return;
        }
        if (blockIdx.x == 0 && tid == 0) a.st->k2 = kit;   // for KB of this iteration
    }
    double beta = 0.0, alpha_prev = 0.0;
    if constexpr (CG) {
        const CgStep c = cg_k1_finish<Lo::NT, PC>(a.st, a.red, sred, pre);
        if (c.done) {
            // drain the copies already in flight, then leave
            if (leader) {
                if (u0 < nunits) mbar_wait(gbar + 0, 0);
                if (u0 + TG < nunits) mbar_wait(gbar + 1, 0);
            }
            return;
        }
        beta = c.beta;
        alpha_prev = c.alpha_prev;
        kit = c.k;
    }

    // thread-varying D entries in registers
    double Dri[n], Drj[n], Dci[n], Dcj[n];
#pragma unroll
    for (int m = 0; m < n; ++m) {
        Dri[m] = c_D[DO + i * n + m];
        Drj[m] = c_D[DO + j * n + m];
        Dci[m] = c_D[DO + m * n + i];
        Dcj[m] = c_D[DO + m * n + j];
    }

    double pap = 0.0;
    int t = 0;
    for (int64_t unit = u0; unit < nunits; unit += TG, ++t) {
        const int s = t & 1;
        double *sb = stage0 + size_t(s) * STAGE;
        const int64_t e0 = unit * EPG;
        const int64_t e = e0 + el;
        const bool on = lane_on && (e < a.E);
        const int sh = (int)((e0 * n3) & 1);  // element data offset in each vector slot
        double hc[MASS ? n : 1];              // mass diagonal of the column (MASS)
        if constexpr (MASS) {
            const double *hv = (CG ? a.u : a.r) + e * n3 + ij;
#pragma unroll
            for (int k = 0; k < n; ++k) hc[k] = on ? __ldg(hv + k * n2) : 0.0;
        }
        mbar_wait(gbar + s, (t >> 1) & 1);

        double *su;     // Ax input in smem (u, or p after the CG update)
        double col[n];  // input column (i,j,0..N)
        const int64_t gbase = e * n3 + ij;
        if constexpr (CG) {
            double *sr = sb + 0 * VL + sh + elc * n3;
            double *sp = sb + 1 * VL + sh + elc * n3;
            double *sx = sb + 2 * VL + sh + elc * n3;
            su = sp;
            if (on) {
#pragma unroll
                for (int k = 0; k < n; ++k) {
                    const int q = k * n2 + ij;
                    const double rl = sr[q];
                    double pl;
                    if (kit == 0) {
                        pl = rl;
                    } else {
                        const double po = sp[q];
                        a.x[gbase + k * n2] = sx[q] + alpha_prev * po;
                        pl = rl + beta * po;
                    }
                    sp[q] = pl;
                    a.p[gbase + k * n2] = pl;
                    col[k] = pl;
                }
            } else {
#pragma unroll
                for (int k = 0; k < n; ++k) col[k] = 0.0;
            }
            group_bar(1 + g, GT);  // p visible to the group
        } else {
            su = sb + sh + elc * n3;
#pragma unroll
            for (int k = 0; k < n; ++k) col[k] = on ? su[k * n2 + ij] : 0.0;
        }
        double *sG = sb + NV * VL + elc * 6 * n3;

        // ---- phase A: gradient, geometric factors ----
        double ft[n];
#pragma unroll
        for (int k = 0; k < n; ++k) {
            const double *uk = su + k * n2;
            double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                ur = fma(Dri[m], uk[j * n + m], ur);
                us = fma(Drj[m], uk[m * n + i], us);
                ut = fma(c_D[DO + k * n + m], col[m], ut);
            }
            const int q = k * n2 + ij;
            double fr = 0.0, fs = 0.0, f3 = 0.0;
            if (on) {
                const double g0 = sG[0 * n3 + q], g1 = sG[1 * n3 + q], g2 = sG[2 * n3 + q];
                const double g3 = sG[3 * n3 + q], g4 = sG[4 * n3 + q], g5 = sG[5 * n3 + q];
                fr = g0 * ur + g1 * us + g2 * ut;
                fs = g1 * ur + g3 * us + g4 * ut;
                f3 = g2 * ur + g4 * us + g5 * ut;
                sG[0 * n3 + q] = fr;   // own node's slots, already consumed
                sG[1 * n3 + q] = fs;
            }
            ft[k] = f3;
        }
        group_bar(1 + g, GT);

        // ---- phase B: transposed contraction, epilogue ----
#pragma unroll
        for (int k = 0; k < n; ++k) {
            const double *frk = sG + 0 * n3 + k * n2;
            const double *fsk = sG + 1 * n3 + k * n2;
            double wr = 0.0, ws = 0.0, wt = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                wr = fma(Dci[m], frk[j * n + m], wr);
                ws = fma(Dcj[m], fsk[m * n + i], ws);
                wt = fma(c_D[DO + m * n + k], ft[m], wt);
            }
            double wv = wr + ws + wt;
            if constexpr (MASS) wv = fma(hc[k], col[k], wv);
            if (on) {
                a.w[gbase + k * n2] = wv;
                if constexpr (CG || DOT) pap = fma(wv, col[k], pap);
            }
        }
        fence_proxy_async();     // generic smem writes before the next async refill
        group_bar(1 + g, GT);    // stage s fully consumed
        if (leader && unit + 2 * TG < nunits) {
            issue_G(unit + 2 * TG, s);
            issue_V(unit + 2 * TG, s);
        }
    }

    if constexpr (CG || DOT) {
        // (p, mask Q Q^T A_L p)_c = sum_e p_e^T A_e p_e because p is continuous
        // and zero on the Dirichlet boundary: every local node counts, no
        // weights, no assembly.  One deterministic partial per CTA; the
        // consumers reduce them (see cg_device.cuh).
        const double bs = block_sum<Lo::NT>(pap, sred);
        if (tid == 0) a.part1[(kit & 1) * a.red.s1 + blockIdx.x] = bs;
    }
}

// ---------------------------------------------------------------------------
// High orders: a whole element's G^ (6 n^3 doubles, up to 196 KB) does not fit
// a double-buffered stage, so the hi kernel streams G^ by k-SLICES: G^ is laid
// out slice-major ([E][n][6][n^2], chosen at setup for this kernel) so one
// 48 n^2-byte bulk copy fetches slice k, into a ring of R slots per group with
// one mbarrier each; the leader keeps R slices in flight across element
// boundaries.  The Ax input vector (r and p for K1) is staged per element,
// double-buffered, as in the low-order kernel.  f_r, f_s live in a
// double-buffered k-slice (one barrier per slice); D comes from shared memory
// (lane-dependent rows/columns) and constant memory (uniform k, m).
// ---------------------------------------------------------------------------
template <int N, bool CG>
struct HiCfg {
    static constexpr int n = N + 1, n2 = n * n, n3 = n2 * n;
    static constexpr int GT = ((n2 + 31) / 32) * 32;
    static constexpr int VL = ((n3 + 2 + 1) / 2) * 2;
    static constexpr int NV = CG ? 2 : 1;                  // r, p | u
    static constexpr int STAGE = NV * VL;                  // doubles per element buffer
    static constexpr int SL = 6 * n2;                      // doubles per G^ slice
    static constexpr int R = 4;                            // G^ slices in flight per group
    static constexpr int PERG = 2 * STAGE + R * SL + 4 * n2;
    static constexpr int SMEM_MAX = 227 * 1024 - 2048;
    static constexpr int NG_FIT = SMEM_MAX / (PERG * 8);
    static constexpr int NG = NG_FIT > 3 ? 3 : NG_FIT;
    static constexpr int NT = NG * GT;
    static constexpr size_t SMEM = size_t(NG) * PERG * 8 + size_t(NG) * (2 + R) * 8 + 64;
};

template <int N, bool CG, bool MASS, bool PC = false, bool DOT = false>
__global__ void __launch_bounds__(HiCfg<N, CG>::NT, 1) ax_hi_kernel(TmaArgs a) {
    using C = HiCfg<N, CG>;
    constexpr int n = C::n, n2 = C::n2, n3 = C::n3, GT = C::GT, VL = C::VL, NV = C::NV;
    constexpr int STAGE = C::STAGE, PERG = C::PERG, NG = C::NG, SL = C::SL, R = C::R;
    constexpr int DO = d_off(N);
    extern __shared__ __align__(128) double smem[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + size_t(NG) * PERG);   // [NG][2 + R]
    constexpr int DS = n | 1;                  // odd row stride: conflict-free lane-indexed rows
    __shared__ double sD[n * DS];
    __shared__ double sred[4 * ((C::NT + 31) / 32)];

    const int tid = threadIdx.x;
    const int g = tid / GT;
    const int ij = tid - g * GT;
    const bool lane_on = ij < n2;
    const int ijc = lane_on ? ij : 0;
    const int i = ijc % n, j = ijc / n;
    const bool leader = (ij == 0);
    double *base_g = smem + size_t(g) * PERG;
    double *ring = base_g + 2 * STAGE;                      // [R][6][n2]
    double *sf = ring + R * SL;                             // [2 slices][f_r, f_s][n2]
    uint64_t *vbar = bars + (2 + R) * g;                    // element stages
    uint64_t *gbar = vbar + 2;                              // G^ ring slots
    const int64_t TG = int64_t(gridDim.x) * NG;
    const int64_t e0 = int64_t(blockIdx.x) * NG + g;
    const int64_t L = a.E * n3;
    const int64_t nel = (e0 < a.E) ? (a.E - e0 + TG - 1) / TG : 0;   // elements of this group
    const int64_t nsl = nel * n;                                     // G^ slices of this group
    for (int t = tid; t < n2; t += C::NT) sD[(t / n) * DS + t % n] = c_D[DO + t];
    if (leader) {
        for (int q = 0; q < 2 + R; ++q) mbar_init(vbar + q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if constexpr (CG) pdl_trigger();
    const uint64_t pol_v = CG ? policy_evict_last() : policy_evict_first();
    const uint64_t pol_g = policy_evict_first();
    // G^ slice gs of this group's stream (element e0 + (gs / n) TG, slice gs % n)
    auto issue_slice = [&](int64_t gs) {
        const int slot = (int)(gs % R);
        const int64_t e = e0 + (gs / n) * TG;
        const int k = (int)(gs % n);
        mbar_expect_tx_only(gbar + slot, SL * 8);
        mbar_arrive(gbar + slot);
        bulk_g2s(ring + slot * SL, a.G + e * 6 * n3 + (int64_t)k * SL, SL * 8, gbar + slot, pol_g);
    };
    auto issue_vec = [&](int64_t e, int s) {
        double *sb = base_g + size_t(s) * STAGE;
        const int64_t first = e * n3;
        const VecRange vr = vec_range(first, n3, L);
        const double *vsrc[2];
        if constexpr (CG) {
            vsrc[0] = a.r;
            vsrc[1] = a.p;
        } else {
            vsrc[0] = a.u;
        }
        const uint32_t vb = (uint32_t)((vr.a1 - vr.a0) * 8);
        mbar_expect_tx_only(vbar + s, NV * vb);
        for (int v = 0; v < NV; ++v)
            for (int64_t q = vr.a1; q < first + n3; ++q) sb[v * VL + (q - vr.a0)] = __ldg(vsrc[v] + q);
        mbar_arrive(vbar + s);
        for (int v = 0; v < NV; ++v) bulk_g2s(sb + v * VL, vsrc[v] + vr.a0, vb, vbar + s, pol_v);
    };
    // scalar loads first (see ax_tma_kernel), then G^ slices and vectors
    K1Pre<PC> pre;
    if constexpr (CG) {
        pdl_wait();
        cg_k1_load<C::NT, PC>(a.st, a.red, pre);
    }
    int dot_done = 0, kit = 0;
    if constexpr (DOT) {
        dot_done = ld_state(&a.st->done);
        kit = ld_state(&a.st->k1);
    }
    if (leader) {
        for (int64_t gs = 0; gs < R && gs < nsl; ++gs) issue_slice(gs);
        if (nel > 0) issue_vec(e0, 0);
        if (nel > 1) issue_vec(e0 + TG, 1);
    }
    if constexpr (DOT) {
        if (dot_done) {
            if (leader) {
                for (int64_t gs = 0; gs < R && gs < nsl; ++gs) mbar_wait(gbar + gs, 0);
                if (nel > 0) mbar_wait(vbar + 0, 0);
                if (nel > 1) mbar_wait(vbar + 1, 0);
            }
            return;
        }
        if (blockIdx.x == 0 && tid == 0) a.st->k2 = kit;
    }
    double beta = 0.0, alpha_prev = 0.0;
    if constexpr (CG) {
        const CgStep c = cg_k1_finish<C::NT, PC>(a.st, a.red, sred, pre);
        if (c.done) {
            if (leader) {       // drain everything in flight
                for (int64_t gs = 0; gs < R && gs < nsl; ++gs) mbar_wait(gbar + gs, 0);
                if (nel > 0) mbar_wait(vbar + 0, 0);
                if (nel > 1) mbar_wait(vbar + 1, 0);
            }
            return;
        }
        beta = c.beta;
        alpha_prev = c.alpha_prev;
        kit = c.k;
    }

    double pap = 0.0;
    int64_t gs = 0;                                          // slice stream position
    for (int64_t t = 0; t < nel; ++t) {
        const int64_t e = e0 + t * TG;
        const int s = (int)(t & 1);
        double *sb = base_g + size_t(s) * STAGE;
        const int sh = (int)((e * n3) & 1);
        const int64_t gb = e * n3 + ijc;
        double xc[CG ? n : 1];
        if constexpr (CG) {
            if (kit > 0) {
#pragma unroll
                for (int k = 0; k < n; ++k) xc[k] = a.x[gb + k * n2];
            }
        }
        double hc[MASS ? n : 1];
        if constexpr (MASS) {
            const double *hv = (CG ? a.u : a.r) + gb;
#pragma unroll
            for (int k = 0; k < n; ++k) hc[k] = lane_on ? __ldg(hv + k * n2) : 0.0;
        }
        mbar_wait(vbar + s, (int)((t >> 1) & 1));
        double col[n];
        double *su;
        if constexpr (CG) {
            double *sr = sb + sh;
            double *sp = sb + VL + sh;
            su = sp;
#pragma unroll
            for (int k = 0; k < n; ++k) {
                const int q = k * n2 + ijc;
                // (padding lanes share a real lane's column: they must not
                // read it while its owner rewrites it -- racecheck r02m)
                const double rl = lane_on ? sr[q] : 0.0;
                double pl = rl;
                if (kit > 0) {
                    const double po = lane_on ? sp[q] : 0.0;
                    if (lane_on) a.x[gb + k * n2] = xc[k] + alpha_prev * po;
                    pl = rl + beta * po;
                }
                if (lane_on) {
                    sp[q] = pl;
                    a.p[gb + k * n2] = pl;
                }
                col[k] = pl;
            }
            group_bar(1 + g, GT);
        } else {
            su = sb + sh;
#pragma unroll
            for (int k = 0; k < n; ++k) col[k] = su[k * n2 + ijc];
        }
        double rw[n];
#pragma unroll
        for (int k = 0; k < n; ++k) rw[k] = 0.0;
#pragma unroll
        for (int k = 0; k < n; ++k, ++gs) {
            const int slot = (int)(gs % R);
            mbar_wait(gbar + slot, (int)((gs / R) & 1));
            const double *gk = ring + slot * SL + ijc;
            const double g0 = gk[0 * n2], g1 = gk[1 * n2], g2 = gk[2 * n2];
            const double g3 = gk[3 * n2], g4 = gk[4 * n2], g5 = gk[5 * n2];
            const double *uk = su + k * n2;
            double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                ur = fma(sD[i * DS + m], uk[j * n + m], ur);
                us = fma(sD[j * DS + m], uk[m * n + i], us);
                ut = fma(c_D[DO + k * n + m], col[m], ut);
            }
            const double fr = g0 * ur + g1 * us + g2 * ut;
            const double fs = g1 * ur + g3 * us + g4 * ut;
            const double ft = g2 * ur + g4 * us + g5 * ut;
            double *sfk = sf + (k & 1) * 2 * n2;
            if (lane_on) {
                sfk[ij] = fr;
                sfk[n2 + ij] = fs;
            }
#pragma unroll
            for (int m = 0; m < n; ++m) rw[m] = fma(c_D[DO + k * n + m], ft, rw[m]);
            group_bar(1 + g, GT);   // f slice visible; every thread is done with G^ slot
            if (leader && gs + R < nsl) issue_slice(gs + R);
            double acc = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                acc = fma(sD[m * DS + i], sfk[j * n + m], acc);
                acc = fma(sD[m * DS + j], sfk[n2 + m * n + i], acc);
            }
            rw[k] += acc;
        }
        if (lane_on) {
#pragma unroll
            for (int k = 0; k < n; ++k) {
                if constexpr (MASS) rw[k] = fma(hc[k], col[k], rw[k]);
                a.w[gb + k * n2] = rw[k];
                if constexpr (CG || DOT) pap = fma(rw[k], col[k], pap);
            }
        }
        fence_proxy_async();
        group_bar(1 + g, GT);    // stage s and both f slices consumed
        if (leader && t + 2 < nel) issue_vec(e + 2 * TG, s);
    }
    if constexpr (CG || DOT) {
        const double bs = block_sum<C::NT>(pap, sred);
        if (tid == 0) a.part1[(kit & 1) * a.red.s1 + blockIdx.x] = bs;
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
#define SEM_TMA_DISPATCH(N_, ...)                                            \
    switch (N_) {                                                            \
    case 1: { constexpr int NN = 1; __VA_ARGS__; } break;                    \
    case 2: { constexpr int NN = 2; __VA_ARGS__; } break;                    \
    case 3: { constexpr int NN = 3; __VA_ARGS__; } break;                    \
    case 4: { constexpr int NN = 4; __VA_ARGS__; } break;                    \
    case 5: { constexpr int NN = 5; __VA_ARGS__; } break;                    \
    case 6: { constexpr int NN = 6; __VA_ARGS__; } break;                    \
    case 7: { constexpr int NN = 7; __VA_ARGS__; } break;                    \
    case 8: { constexpr int NN = 8; __VA_ARGS__; } break;                    \
    case 9: { constexpr int NN = 9; __VA_ARGS__; } break;                    \
    case 10: { constexpr int NN = 10; __VA_ARGS__; } break;                  \
    default: break;                                                          \
    }

template <int N, bool CG>
static int tma_grid(int64_t E, int nsm) {
    using Lo = TmaLayout<N, CG>;
    const int64_t nunits = (E + TmaCfg<N>::EPG - 1) / TmaCfg<N>::EPG;
    int64_t need = (nunits + Lo::NG - 1) / Lo::NG;
    return (int)(need < nsm ? (need < 1 ? 1 : need) : nsm);
}

template <int N, bool CG, bool MASS, bool PC = false>
static cudaError_t tma_attr() {
    using Lo = TmaLayout<N, CG>;
    static_assert(Lo::NG >= 1, "stage does not fit in shared memory");
    return cudaFuncSetAttribute(ax_tma_kernel<N, CG, MASS, PC>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lo::SMEM);
}

// PC = false: the plain and CG kernels; PC = true: the PCG K1 only
template <bool MASS, bool PC = false>
static cudaError_t tma_prepare_t(int N) {
    cudaError_t e = cudaSuccess;
    if constexpr (PC) {
        SEM_TMA_DISPATCH(N, (e = tma_attr<NN, true, MASS, true>()));
    } else {
        SEM_TMA_DISPATCH(N, (e = tma_attr<NN, false, MASS>(),
                             e = (e == cudaSuccess ? tma_attr<NN, true, MASS>() : e)));
    }
    return e;
}

template <bool MASS>
static cudaError_t launch_ax_tma_t(const DevMesh &m, const double *u, double *w, cudaStream_t s) {
    TmaArgs a{};
    a.E = m.E;
    a.G = m.G;
    a.u = u;
    a.w = w;
    if (MASS) a.r = m.H;      // the plain apply does not use r
    SEM_TMA_DISPATCH(m.N, (ax_tma_kernel<NN, false, MASS><<<tma_grid<NN, false>(m.E, m.nsm),
                                                            TmaLayout<NN, false>::NT,
                                                            TmaLayout<NN, false>::SMEM, s>>>(a)));
    return cudaGetLastError();
}

// ---- high-order kernel ----
#define SEM_HI_DISPATCH(N_, ...)                                             \
    switch (N_) {                                                            \
    case 6: { constexpr int NN = 6; __VA_ARGS__; } break;                    \
    case 7: { constexpr int NN = 7; __VA_ARGS__; } break;                    \
    case 8: { constexpr int NN = 8; __VA_ARGS__; } break;                    \
    case 9: { constexpr int NN = 9; __VA_ARGS__; } break;                    \
    case 10: { constexpr int NN = 10; __VA_ARGS__; } break;                  \
    case 11: { constexpr int NN = 11; __VA_ARGS__; } break;                  \
    case 12: { constexpr int NN = 12; __VA_ARGS__; } break;                  \
    case 13: { constexpr int NN = 13; __VA_ARGS__; } break;                  \
    case 14: { constexpr int NN = 14; __VA_ARGS__; } break;                  \
    case 15: { constexpr int NN = 15; __VA_ARGS__; } break;                  \
    default: break;                                                          \
    }

template <int N, bool CG>
static int hi_grid(int64_t E, int nsm) {
    int64_t need = (E + HiCfg<N, CG>::NG - 1) / HiCfg<N, CG>::NG;
    return (int)(need < nsm ? (need < 1 ? 1 : need) : nsm);
}

template <int N, bool CG, bool MASS, bool PC = false>
static cudaError_t hi_attr() {
    static_assert(HiCfg<N, CG>::NG >= 1, "element stage does not fit in shared memory");
    return cudaFuncSetAttribute(ax_hi_kernel<N, CG, MASS, PC>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)HiCfg<N, CG>::SMEM);
}

template <bool MASS, bool PC = false>
static cudaError_t hi_prepare_t(int N) {
    cudaError_t e = cudaSuccess;
    if constexpr (PC) {
        SEM_HI_DISPATCH(N, (e = hi_attr<NN, true, MASS, true>()));
    } else {
        SEM_HI_DISPATCH(N, (e = hi_attr<NN, false, MASS>(),
                            e = (e == cudaSuccess ? hi_attr<NN, true, MASS>() : e)));
    }
    return e;
}

template <bool MASS>
static cudaError_t launch_ax_hi_t(const DevMesh &m, const double *u, double *w, cudaStream_t s) {
    TmaArgs a{};
    a.E = m.E;
    a.G = m.G;
    a.u = u;
    a.w = w;
    if (MASS) a.r = m.H;
    SEM_HI_DISPATCH(m.N, (ax_hi_kernel<NN, false, MASS><<<hi_grid<NN, false>(m.E, m.nsm),
                                                          HiCfg<NN, false>::NT,
                                                          HiCfg<NN, false>::SMEM, s>>>(a)));
    return cudaGetLastError();
}

// KA of the single-reduction CG: w = A_L r plus (r, w) partials (DOT)
static TmaArgs sr_args(const DevMesh &m, const CgVecs &v) {
    TmaArgs a{};
    a.E = m.E;
    a.G = m.G;
    a.u = v.r;
    a.w = v.w;
    a.red = make_red(m, v);
    a.part1 = v.part1;
    a.st = v.st;
    return a;
}

static cudaError_t tma_prepare_dot(int N) {
    cudaError_t e = cudaSuccess;
    SEM_TMA_DISPATCH(N, (e = cudaFuncSetAttribute(ax_tma_kernel<NN, false, false, false, true>,
                                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)TmaLayout<NN, false>::SMEM)));
    return e;
}

static cudaError_t launch_ax_dot_tma_t(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    const TmaArgs a = sr_args(m, v);
    SEM_TMA_DISPATCH(m.N, (ax_tma_kernel<NN, false, false, false, true>
                           <<<tma_grid<NN, false>(m.E, m.nsm), TmaLayout<NN, false>::NT,
                              TmaLayout<NN, false>::SMEM, s>>>(a)));
    return cudaGetLastError();
}

static cudaError_t hi_prepare_dot(int N) {
    cudaError_t e = cudaSuccess;
    SEM_HI_DISPATCH(N, (e = cudaFuncSetAttribute(ax_hi_kernel<NN, false, false, false, true>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)HiCfg<NN, false>::SMEM)));
    return e;
}

static cudaError_t launch_ax_dot_hi_t(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    const TmaArgs a = sr_args(m, v);
    SEM_HI_DISPATCH(m.N, (ax_hi_kernel<NN, false, false, false, true>
                          <<<hi_grid<NN, false>(m.E, m.nsm), HiCfg<NN, false>::NT,
                             HiCfg<NN, false>::SMEM, s>>>(a)));
    return cudaGetLastError();
}

// K1 over the element range [eb, eb + ne): the kernels see a mesh of ne
// elements through pointers offset by eb (eb * n^3 must be even: the bulk
// copies of the vectors need 16-byte aligned sources), and write their
// per-CTA (p, A p) partials to slots [pidx0, pidx0 + grid) of part1.
template <bool MASS>
static TmaArgs cg_args(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, int pidx0) {
    const int64_t o = eb * m.n3;
    TmaArgs a{};
    a.E = ne;
    a.G = m.G + 6 * o;
    a.r = k1_src(v) + o;
    a.p = v.p + o;
    a.x = v.xw + o;
    a.w = v.w + o;
    a.red = make_red(m, v);
    a.part1 = v.part1 + pidx0;
    a.st = v.st;
    if (MASS) a.u = m.H + o;  // K1 does not use u
    return a;
}

template <bool MASS, bool PC = false>
static cudaError_t launch_ax_cg_hi_t(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                                     int pidx0, cudaStream_t s) {
    const TmaArgs a = cg_args<MASS>(m, v, eb, ne, pidx0);
    cudaError_t e = cudaSuccess;
    SEM_HI_DISPATCH(m.N, e = launch_pdl(ax_hi_kernel<NN, true, MASS, PC>, hi_grid<NN, true>(ne, m.nsm),
                                        HiCfg<NN, true>::NT, HiCfg<NN, true>::SMEM, s, a));
    return e;
}

template <bool MASS, bool PC = false>
static cudaError_t launch_ax_cg_tma_t(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                                      int pidx0, cudaStream_t s) {
    const TmaArgs a = cg_args<MASS>(m, v, eb, ne, pidx0);
    cudaError_t e = cudaSuccess;
    SEM_TMA_DISPATCH(m.N, e = launch_pdl(ax_tma_kernel<NN, true, MASS, PC>,
                                         tma_grid<NN, true>(ne, m.nsm), TmaLayout<NN, true>::NT,
                                         TmaLayout<NN, true>::SMEM, s, a));
    return e;
}

}  // namespace sem
