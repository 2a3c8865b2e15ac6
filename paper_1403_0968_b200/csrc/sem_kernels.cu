// sem_kernels.cu -- sm_100a kernels of the SEM Poisson hot path (arXiv 1403.0968,
// PAPER.md:578-784).  FP64 on the CUDA cores: the operator is HBM-bound at
// 64 B per local node (u, six G^ factors, w) and tcgen05 has no FP64 kind.
//
//   geom_kernel      a1: isoparametric geometric factors G^ = w J (dr/dx)(dr/dx)^T
//   ax_kernel<N,..>  a3-a5: w = D^T G^ D u per element (sum factorisation)
//   gs_kernel        a6/a8: Q Q^T over element-surface groups (+ mask, + (w,p)_c)
//
// Layout: local node (i,j,k) of element e at e*n^3 + i + n*j + n^2*k.
#include <cstdio>

#include "cg_device.cuh"
#include "p2p_dev.cuh"
#include "sem_internal.h"

namespace sem {

// --------------------------------------------------------------------------
// helpers
// --------------------------------------------------------------------------
// (block_sum, block_sum_array, last_block: cg_device.cuh)

__device__ __forceinline__ double sum_ranks(const double *a, int nranks) {
    double s = 0.0;
    for (int q = 0; q < nranks; ++q) s += __ldcg(a + q);
    return s;
}

// --------------------------------------------------------------------------
// a1: geometric factors (setup).  One thread per local node, reading the
// element's coordinates from global memory (setup-only; not a hot path).
// --------------------------------------------------------------------------
__global__ void geom_kernel(int n, int64_t E, const double *__restrict__ D,
                            const double *__restrict__ wq, const double *__restrict__ xyz,
                            const double *__restrict__ kappa, double *__restrict__ G,
                            double *__restrict__ BM, double *__restrict__ H, int *bad,
                            bool slice_major) {
    const int n3 = n * n * n;
    const int64_t L = E * n3;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / n3;
        const int q = (int)(l - e * n3);
        const int i = q % n, j = (q / n) % n, k = q / (n * n);
        const double *X = xyz + e * 3 * n3;
        double a[3][3];  // a[c][d] = d x_c / d r_d
        for (int c = 0; c < 3; ++c) {
            const double *Xc = X + c * n3;
            double dr = 0.0, ds = 0.0, dt = 0.0;
            for (int m = 0; m < n; ++m) {
                dr += D[i * n + m] * Xc[m + n * j + n * n * k];
                ds += D[j * n + m] * Xc[i + n * m + n * n * k];
                dt += D[k * n + m] * Xc[i + n * j + n * n * m];
            }
            a[c][0] = dr;
            a[c][1] = ds;
            a[c][2] = dt;
        }
        // cofactors C[c][d]; J = sum_d a[0][d] C[0][d]; (dr_d/dx_c) = C[c][d] / J
        double C[3][3];
        C[0][0] = a[1][1] * a[2][2] - a[1][2] * a[2][1];
        C[0][1] = a[1][2] * a[2][0] - a[1][0] * a[2][2];
        C[0][2] = a[1][0] * a[2][1] - a[1][1] * a[2][0];
        C[1][0] = a[0][2] * a[2][1] - a[0][1] * a[2][2];
        C[1][1] = a[0][0] * a[2][2] - a[0][2] * a[2][0];
        C[1][2] = a[0][1] * a[2][0] - a[0][0] * a[2][1];
        C[2][0] = a[0][1] * a[1][2] - a[0][2] * a[1][1];
        C[2][1] = a[0][2] * a[1][0] - a[0][0] * a[1][2];
        C[2][2] = a[0][0] * a[1][1] - a[0][1] * a[1][0];
        const double J = a[0][0] * C[0][0] + a[0][1] * C[0][1] + a[0][2] * C[0][2];
        if (!(J > 0.0)) atomicExch(bad, 1);
        const double wJ = wq[i] * wq[j] * wq[k] * J;
        // G_de = w J sum_c (dr_d/dx_c)(dr_e/dx_c) = (w / J) sum_c C[c][d] C[c][e]
        const double s = wq[i] * wq[j] * wq[k] / J;
        double g[6];
        const int pd[6] = {0, 0, 0, 1, 1, 2}, pe[6] = {0, 1, 2, 1, 2, 2};
        for (int f = 0; f < 6; ++f)
            g[f] = s * (C[0][pd[f]] * C[0][pe[f]] + C[1][pd[f]] * C[1][pe[f]] +
                        C[2][pd[f]] * C[2][pe[f]]);
        // screened Coulomb (NEXT-1): kappa weights the flux at the node
        // (reading G2), the mass term is alpha w J (lumped)
        if (kappa) {
            const double kq = kappa[l];
            for (int f = 0; f < 6; ++f) g[f] *= kq;
        }
        if (H) H[l] = H[l] * wJ;
        if (slice_major) {      // [E][n][6][n^2]: one contiguous block per k-slice
            double *Ge = G + e * 6 * n3 + (int64_t)k * 6 * n * n + (i + n * j);
            for (int f = 0; f < 6; ++f) Ge[f * n * n] = g[f];
        } else {                // [E][6][n^3]
            double *Ge = G + e * 6 * n3 + q;
            for (int f = 0; f < 6; ++f) Ge[f * n3] = g[f];
        }
        BM[l] = wJ;
    }
}

// --------------------------------------------------------------------------
// NEXT-2 (Jacobi PCG): the diagonal of the local operator.
// A^e = D_r^T G_rr D_r + ... (6 factor products, G^ symmetric), so for node
// q = (i,j,k) the unit vector's reference gradient is nonzero only on the
// three GLL lines through q, which gives
//   d_q = sum_m D_mi^2 G_rr(m,j,k) + sum_m D_mj^2 G_ss(i,m,k) + sum_m D_mk^2 G_tt(i,j,m)
//       + 2 D_ii D_jj G_rs(q) + 2 D_ii D_kk G_rt(q) + 2 D_jj D_kk G_st(q) + H(q)
// (kappa is folded into G^, H = alpha w J).  Setup-only; one thread per node.
// --------------------------------------------------------------------------
__global__ void diag_kernel(int n, int64_t E, const double *__restrict__ D,
                            const double *__restrict__ G, const double *__restrict__ H,
                            double *__restrict__ d, bool slice_major) {
    const int n2 = n * n, n3 = n2 * n;
    const int64_t L = E * n3;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = l / n3;
        const int q = (int)(l - e * n3);
        const int i = q % n, j = (q / n) % n, k = q / n2;
        const double *Ge = G + e * 6 * n3;
        // factor f at node (a,b,c) of this element, in either G^ layout
        auto g = [&](int f, int a, int b, int c) {
            return slice_major ? Ge[(int64_t)c * 6 * n2 + f * n2 + a + n * b]
                               : Ge[f * n3 + a + n * b + n2 * c];
        };
        double s = 0.0;
        for (int m = 0; m < n; ++m) {
            const double dr = D[m * n + i], ds = D[m * n + j], dt = D[m * n + k];
            s += dr * dr * g(0, m, j, k) + ds * ds * g(3, i, m, k) + dt * dt * g(5, i, j, m);
        }
        const double di = D[i * n + i], dj = D[j * n + j], dk = D[k * n + k];
        s += 2.0 * (di * dj * g(1, i, j, k) + di * dk * g(2, i, j, k) + dj * dk * g(4, i, j, k));
        if (H) s += H[l];
        d[l] = s;
    }
}

__global__ void recip_kernel(int64_t L, const double *__restrict__ d, double *__restrict__ dinv) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x)
        dinv[l] = 1.0 / d[l];
}

// --------------------------------------------------------------------------
// a3-a5: local stiffness apply.  Block = EPB elements x (n x n) threads; thread
// (i,j) owns the k-column of its element in registers:
//   u_r, u_s from the k-slice in shared memory, u_t from the register column,
//   f = G^ (u_r,u_s,u_t) with G^ streamed once from HBM,
//   w[:,:,m] += D_km f_t (register column), then the r/s transposed
//   contractions from f_r, f_s staged per slice in shared memory.
// CG = true fuses the CG prologue/epilogue (K1 of DESIGN.md):
//   x += alpha_{k-1} p_{k-1};  p = r + beta_k p_{k-1};  w = A_L p;
//   (w,p) over all local nodes (= p^T mask QQ^T A_L p), reduced into
//   pap_all[k & 3][rank] by the last block.
// --------------------------------------------------------------------------
template <int N>
struct AxCfg {
    static constexpr int n = N + 1;
    static constexpr int n2 = n * n;
    static constexpr int n3 = n2 * n;
    static constexpr int EPB = (n2 >= 256) ? 1 : (256 / n2);
    static constexpr int NT = EPB * n2;
};

struct AxCgArgs {
    const double *r;
    double *p, *x;
    CgRed red;
    double *part1;
    CgState *st;
};

// Grid-stride over blocks of EPB elements (grid <= 4 CTAs per SM, so the
// (p, A p) partials stay few).
template <int N, bool CG>
__global__ void __launch_bounds__(AxCfg<N>::NT)
ax_kernel(int64_t E, const double *__restrict__ Dg, const double *__restrict__ G,
          const double *__restrict__ u, double *__restrict__ wout, AxCgArgs cg) {
    using C = AxCfg<N>;
    constexpr int n = C::n, n2 = C::n2, n3 = C::n3, EPB = C::EPB, NT = C::NT;
    __shared__ double sD[n2];
    __shared__ double su[EPB][n3];
    __shared__ double sfr[EPB][n2];
    __shared__ double sfs[EPB][n2];
    __shared__ double sred[4 * ((NT + 31) / 32)];

    double beta = 0.0, alpha_prev = 0.0;
    int kit = 0;
    double *xg = cg.x;
    if constexpr (CG) {
        pdl_trigger();
        pdl_wait();
        const CgStep c = cg_k1_prologue<NT>(cg.st, cg.red, sred);
        if (c.done) return;
        beta = c.beta;
        alpha_prev = c.alpha_prev;
        kit = c.k;
    }

    const int tid = threadIdx.x;
    for (int t = tid; t < n2; t += NT) sD[t] = Dg[t];
    const int el = tid / n2;
    const int ij = tid - el * n2;
    const int i = ij % n, j = ij / n;
    const int64_t nblk = (E + EPB - 1) / EPB;
    double part = 0.0;
    for (int64_t eb = blockIdx.x; eb < nblk; eb += gridDim.x) {
        const int64_t e = eb * EPB + el;
        const bool active = e < E;
        const int64_t base = e * n3 + ij;

        double ru[n], rw[n];
        if (active) {
            if constexpr (CG) {
#pragma unroll
                for (int k = 0; k < n; ++k) {
                    const int64_t l = base + k * n2;
                    const double rl = cg.r[l];
                    double pl;
                    if (kit == 0) {
                        pl = rl;
                    } else {
                        const double po = cg.p[l];
                        xg[l] += alpha_prev * po;
                        pl = rl + beta * po;
                    }
                    cg.p[l] = pl;
                    ru[k] = pl;
                }
            } else {
#pragma unroll
                for (int k = 0; k < n; ++k) ru[k] = u[base + k * n2];
            }
        } else {
#pragma unroll
            for (int k = 0; k < n; ++k) ru[k] = 0.0;
        }
        __syncthreads();   // previous element block done with su / sfr / sfs
#pragma unroll
        for (int k = 0; k < n; ++k) {
            su[el][k * n2 + ij] = ru[k];
            rw[k] = 0.0;
        }
        __syncthreads();

        const double *Ge = G + e * 6 * n3 + ij;
#pragma unroll
        for (int k = 0; k < n; ++k) {
            double ur = 0.0, us = 0.0, ut = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                ur += sD[i * n + m] * su[el][k * n2 + j * n + m];
                us += sD[j * n + m] * su[el][k * n2 + m * n + i];
                ut += sD[k * n + m] * ru[m];
            }
            double g0 = 0, g1 = 0, g2 = 0, g3 = 0, g4 = 0, g5 = 0;
            if (active) {
                const double *Gk = Ge + k * n2;
                g0 = __ldg(Gk + 0 * n3);
                g1 = __ldg(Gk + 1 * n3);
                g2 = __ldg(Gk + 2 * n3);
                g3 = __ldg(Gk + 3 * n3);
                g4 = __ldg(Gk + 4 * n3);
                g5 = __ldg(Gk + 5 * n3);
            }
            const double fr = g0 * ur + g1 * us + g2 * ut;
            const double fs = g1 * ur + g3 * us + g4 * ut;
            const double ft = g2 * ur + g4 * us + g5 * ut;
            sfr[el][ij] = fr;
            sfs[el][ij] = fs;
#pragma unroll
            for (int m = 0; m < n; ++m) rw[m] += sD[k * n + m] * ft;
            __syncthreads();
            double acc = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                acc += sD[m * n + i] * sfr[el][j * n + m];
                acc += sD[m * n + j] * sfs[el][m * n + i];
            }
            rw[k] += acc;
            __syncthreads();
        }

        if (active) {
#pragma unroll
            for (int k = 0; k < n; ++k) wout[base + k * n2] = rw[k];
            if constexpr (CG) {
                // (p, mask Q Q^T A_L p)_c = sum_e p_e^T A_e p_e (p continuous,
                // zero on the Dirichlet boundary)
#pragma unroll
                for (int k = 0; k < n; ++k) part += rw[k] * ru[k];
            }
        }
    }
    if constexpr (CG) {
        const double s = block_sum<NT>(part, sred);
        if (tid == 0) cg.part1[(kit & 1) * cg.red.s1 + blockIdx.x] = s;
    }
}

// --------------------------------------------------------------------------
// a6/a8: gather-scatter over element-surface groups, one thread per group.
// Groups are stored by CLASS (Dirichlet flag, multiplicity m); inside a class
// the copy indices are transposed ([m][count]) so lane-consecutive groups read
// their t-th copy index coalesced, and all m value loads are in flight at
// once (m is a compile-time constant on the common classes).
// mode 0: Q Q^T; 1: + mask; 2: CG iteration (+ mask; waits for K1 when
// launched as a programmatic dependent and is a no-op after the stop).
// The (w,p) dot product is NOT needed here: K1 already has it (see K1).
// --------------------------------------------------------------------------
struct GsArgs {
    GsClasses cls;
    const int32_t *idx;
    int32_t ngroups;
    double *w;
    const CgState *st;
};

__device__ __forceinline__ int gs_find_class(const GsClasses &c, int g) {
    int q = 0;
    while (q + 1 < c.n && g >= c.start[q + 1]) ++q;
    return q;
}

// CG mode: the plan indices are static, so they are loaded before waiting
// for the producer of w; then the stop flag decides.
template <int MODE>
__device__ __forceinline__ bool gs_ready(const CgState *st) {
    if constexpr (MODE == 2) {
        pdl_wait();
        return !ld_state(&st->done);
    }
    return true;
}

template <int MODE, int M>
__device__ __forceinline__ void gs_group(const int32_t *__restrict__ idx, int cnt, int gl, bool dir,
                                         double *__restrict__ w, const CgState *st) {
    int li[M];
    double v[M];
#pragma unroll
    for (int t = 0; t < M; ++t) li[t] = __ldg(idx + t * cnt + gl);
    if (!gs_ready<MODE>(st)) return;
#pragma unroll
    for (int t = 0; t < M; ++t) v[t] = w[li[t]];
    double s = v[0];
#pragma unroll
    for (int t = 1; t < M; ++t) s += v[t];          // ascending local order
    if (MODE >= 1 && dir) s = 0.0;
#pragma unroll
    for (int t = 0; t < M; ++t) w[li[t]] = s;
}

template <int MODE>
__device__ __forceinline__ void gs_group_generic(const int32_t *__restrict__ idx, int m, int cnt,
                                                 int gl, bool dir, double *__restrict__ w,
                                                 const CgState *st) {
    if (!gs_ready<MODE>(st)) return;
    double s = w[__ldg(idx + gl)];
    for (int t = 1; t < m; ++t) s += w[__ldg(idx + t * cnt + gl)];
    if (MODE >= 1 && dir) s = 0.0;
    for (int t = 0; t < m; ++t) w[__ldg(idx + t * cnt + gl)] = s;
}

template <int MODE>
__global__ void __launch_bounds__(kGsThreads) gs_kernel(const __grid_constant__ GsArgs a) {
    if constexpr (MODE == 2) pdl_trigger();
    const int g = blockIdx.x * kGsThreads + threadIdx.x;
    if (g >= a.ngroups) return;
    const int c = gs_find_class(a.cls, g);
    const int m = a.cls.m[c], cnt = a.cls.start[c + 1] - a.cls.start[c];
    const int gl = g - a.cls.start[c];
    const bool dir = a.cls.dir[c] != 0;
    const int32_t *ix = a.idx + a.cls.idxoff[c];
    switch (m) {
    case 1: gs_group<MODE, 1>(ix, cnt, gl, dir, a.w, a.st); break;
    case 2: gs_group<MODE, 2>(ix, cnt, gl, dir, a.w, a.st); break;
    case 3: gs_group<MODE, 3>(ix, cnt, gl, dir, a.w, a.st); break;
    case 4: gs_group<MODE, 4>(ix, cnt, gl, dir, a.w, a.st); break;
    case 6: gs_group<MODE, 6>(ix, cnt, gl, dir, a.w, a.st); break;
    case 8: gs_group<MODE, 8>(ix, cnt, gl, dir, a.w, a.st); break;
    default: gs_group_generic<MODE>(ix, m, cnt, gl, dir, a.w, a.st); break;
    }
}

// zero every copy of the Dirichlet groups (the leading classes)
__global__ void mask_kernel(const __grid_constant__ GsClasses cls, const int32_t *__restrict__ idx,
                            int32_t ndir, double *__restrict__ w) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= ndir) return;
    const int c = gs_find_class(cls, g);
    const int m = cls.m[c], cnt = cls.start[c + 1] - cls.start[c], gl = g - cls.start[c];
    const int32_t *ix = idx + cls.idxoff[c];
    for (int t = 0; t < m; ++t) w[__ldg(ix + t * cnt + gl)] = 0.0;
}

__global__ void mass_kernel(int64_t L, const double *__restrict__ BM, const double *f,
                            double *b) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x)
        b[l] = BM[l] * f[l];
}

// CG start: xw = x0 (K1 updates the workspace copy), reset the device state.
__global__ void cg_init_kernel(int64_t L, CgState *st, const double *__restrict__ x,
                               double *__restrict__ xw) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x)
        xw[l] = x[l];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->done = 0;
        st->iters = 0;
        st->converged = 0;
        st->rel_res = 0.0;
        st->alpha_km1 = 0.0;
        st->k1 = 0;
        st->k2 = 0;
    }
}

// Multi-rank: this rank's value = ordered sum of its block partials, into its
// slot of the all-gather buffer (slot k & 3 for (p,Ap)_k, k_next & 3 for rho).
// With the peer-memory transport (p2p != nullptr) the same kernel then does
// the all-gather itself (warp 0, p2p_dev.cuh): the fold and the collective in
// one launch.  After the stop the fold is skipped but the all-gather still
// runs (every rank's epochs stay in step).
constexpr int kRedThreads = 256;
__global__ void __launch_bounds__(kRedThreads) cg_red_kernel(const double *part, int s, int nb,
                                                             double *all, const CgState *st,
                                                             int which, int rank, int nranks,
                                                             const P2PDev *p2p, int site) {
    __shared__ double sred[kRedThreads / 32];
    const bool done = ld_state(&st->done);
    // (p,Ap): K1 of iteration k = st->k2.  rho: K2 of iteration k1 - 1 (k1 = k_next).
    const int kk = (which == 0) ? ld_state(&st->k2) : ld_state(&st->k1);
    if (!done) {
        const double *src = part + ((which == 0 ? kk : kk - 1) & 1) * s;
        double v = 0.0;
        for (int t = threadIdx.x; t < nb; t += kRedThreads) v += __ldcg(src + t);
        v = block_sum<kRedThreads>(v, sred);
        if (threadIdx.x == 0) all[(kk & 3) * nranks + rank] = v;
    } else if (!p2p) {
        return;
    }
    if (p2p) {
        __syncthreads();
        if (threadIdx.x < 32) p2p_allgather_warp(*p2p, site, all + (kk & 3) * nranks, 1);
    }
}

// K1, first half, of the split schedule (use_k1ax, N >= 10 on the tensor
// cores): the scalar prologue of the iteration (stop, beta_k, alpha_{k-1};
// cg_device.cuh) and the vector update x += alpha_{k-1} p_{k-1},
// p = r + beta_k p_{k-1} (z instead of r for Jacobi PCG) over [0, L).  40 B
// per node (r, p, x read; p, x written; 16 at k = 0).  The second half,
// ax_dmmag_kernel<DOT>, applies the operator to the new p.
constexpr int kKuThreads = 256;
__global__ void __launch_bounds__(kKuThreads) k1u_kernel(const double *__restrict__ src, double *p,
                                                         double *x, int64_t L, CgRed R, CgState *st) {
    __shared__ double sred[4 * (kKuThreads / 32)];
    pdl_wait();
    const CgStep c = cg_k1_prologue<kKuThreads>(st, R, sred);
    if (c.done) return;
    const double beta = c.beta, ap = c.alpha_prev;
    const int64_t npair = L >> 1;
    const int64_t stride = int64_t(gridDim.x) * kKuThreads;
    for (int64_t q = blockIdx.x * int64_t(kKuThreads) + threadIdx.x; q < npair; q += stride) {
        const double2 rv = __ldcs(reinterpret_cast<const double2 *>(src) + q);
        double2 *pp = reinterpret_cast<double2 *>(p) + q;
        if (c.k == 0) {
            *pp = rv;
        } else {
            const double2 pv = *pp;
            double2 *xp = reinterpret_cast<double2 *>(x) + q;
            const double2 xv = *xp;
            *xp = make_double2(xv.x + ap * pv.x, xv.y + ap * pv.y);
            *pp = make_double2(rv.x + beta * pv.x, rv.y + beta * pv.y);
        }
    }
    if ((L & 1) && blockIdx.x == 0 && threadIdx.x == 0) {     // odd length: the last node
        const int64_t l = L - 1;
        if (c.k == 0) {
            p[l] = src[l];
        } else {
            const double pv = p[l];
            x[l] = x[l] + ap * pv;
            p[l] = src[l] + beta * pv;
        }
    }
}

cudaError_t launch_k1u(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, cudaStream_t s) {
    const int64_t o = eb * m.n3;
    return launch_pdl(k1u_kernel, m.nsm * 4, kKuThreads, 0, s, k1_src(v) + o, v.p + o, v.xw + o,
                      ne * m.n3, make_red(m, v), v.st);
}

// x = xw + alpha_{it-1} p_{it-1}: the update K1 would have applied next.
__global__ void cg_finish_kernel(int64_t L, double *__restrict__ x, const double *__restrict__ xw,
                                 const double *__restrict__ p, const CgState *st) {
    const int it = st->iters;
    const double a = (it >= 1) ? st->alpha_km1 : 0.0;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x)
        x[l] = (it >= 1) ? xw[l] + a * p[l] : xw[l];
}

// --------------------------------------------------------------------------
// launchers
// --------------------------------------------------------------------------
template <int N>
static int ax_blocks_t(int64_t E) {
    return (int)((E + AxCfg<N>::EPB - 1) / AxCfg<N>::EPB);
}

#define SEM_DISPATCH_N(N_, CALL)                                             \
    switch (N_) {                                                            \
    case 1: { constexpr int NN = 1; CALL; } break;                           \
    case 2: { constexpr int NN = 2; CALL; } break;                           \
    case 3: { constexpr int NN = 3; CALL; } break;                           \
    case 4: { constexpr int NN = 4; CALL; } break;                           \
    case 5: { constexpr int NN = 5; CALL; } break;                           \
    case 6: { constexpr int NN = 6; CALL; } break;                           \
    case 7: { constexpr int NN = 7; CALL; } break;                           \
    case 8: { constexpr int NN = 8; CALL; } break;                           \
    case 9: { constexpr int NN = 9; CALL; } break;                           \
    case 10: { constexpr int NN = 10; CALL; } break;                         \
    case 11: { constexpr int NN = 11; CALL; } break;                         \
    case 12: { constexpr int NN = 12; CALL; } break;                         \
    case 13: { constexpr int NN = 13; CALL; } break;                         \
    case 14: { constexpr int NN = 14; CALL; } break;                         \
    case 15: { constexpr int NN = 15; CALL; } break;                         \
    default: break;                                                          \
    }

int ax_blocks(int N, int64_t E) {
    int nb = 0;
    SEM_DISPATCH_N(N, nb = ax_blocks_t<NN>(E));
    return nb;
}

// grid of the simple Ax kernels: grid-stride, at most 4 CTAs per SM
static int ax_grid(int N, int64_t E, int nsm) {
    const int nb = ax_blocks(N, E);
    return nb < 4 * nsm ? (nb < 1 ? 1 : nb) : 4 * nsm;
}

// grid of K1 over ne elements (range launches: TMA / high-order kernels only)
int ax_cg_range_blocks(const DevMesh &m, int64_t ne) {
    if (m.use_k1ax) return m.use_dmmag ? dmmag_blocks(m.N, ne, m.nsm) : k1dot_blocks(m, ne);
    if (m.use_dmma) return dmma_blocks(ne, m.nsm, true);
    if (m.use_hi) return hi_blocks(m.N, ne, m.nsm, true);
    return m.use_tma ? tma_blocks(m.N, ne, m.nsm, true) : ax_grid(m.N, ne, m.nsm);
}

bool k1_split(const DevMesh &m) {
    return m.nranks > 1 && (m.use_tma || m.use_hi) && m.nbnd > 0 && m.nbnd < m.E;
}

int ax_cg_blocks(const DevMesh &m) {
    if (k1_split(m)) return ax_cg_range_blocks(m, m.nbnd) + ax_cg_range_blocks(m, m.E - m.nbnd);
    return ax_cg_range_blocks(m, m.E);
}

static int grid_for(int64_t L, int threads) {
    int64_t b = (L + threads - 1) / threads;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

cudaError_t launch_geom(const DevMesh &m, const double *xyz, const double *kappa, double *G,
                        double *BM, double *H, int *bad, cudaStream_t s) {
    // D and the 1-D weights live at the start of the D buffer: [n*n] D, [n] w
    // the high-order kernel streams G^ by k-slices: slice-major layout
    geom_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.n, m.E, m.D, m.D + m.n * m.n, xyz, kappa, G,
                                                   BM, H, bad, m.use_hi);
    return cudaGetLastError();
}

cudaError_t launch_ax(const DevMesh &m, const double *u, double *w, cudaStream_t s) {
    if (m.E == 0) return cudaSuccess;
    if (m.use_dmmag && !m.H) return launch_ax_dmmag(m, u, w, s);
    if (m.use_hi) return launch_ax_hi(m, u, w, s);
    if (m.use_tma) return launch_ax_tma(m, u, w, s);
    if (m.H) return cudaErrorInvalidValue;      // the simple kernel has no mass term
    AxCgArgs none{};
    SEM_DISPATCH_N(m.N, (ax_kernel<NN, false><<<ax_grid(m.N, m.E, m.nsm), AxCfg<NN>::NT, 0, s>>>(
                             m.E, m.D, m.G, u, w, none)));
    return cudaGetLastError();
}

cudaError_t launch_ax_cg(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    if (m.use_k1ax) return launch_ax_cg_dmmag(m, v, 0, m.E, 0, s);
    if (m.use_hi) return launch_ax_cg_hi(m, v, 0, m.E, 0, s);
    if (m.use_tma) return launch_ax_cg_tma(m, v, 0, m.E, 0, s);
    if (m.H) return cudaErrorInvalidValue;
    AxCgArgs a{k1_src(v), v.p, v.xw, make_red(m, v), v.part1, v.st};
    cudaError_t e = cudaSuccess;
    SEM_DISPATCH_N(m.N, (e = launch_pdl(ax_kernel<NN, true>, ax_grid(m.N, m.E, m.nsm), AxCfg<NN>::NT,
                                        0, s, m.E, m.D, m.G, (const double *)nullptr, v.w, a)));
    return e;
}

cudaError_t launch_ax_cg_range(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, int pidx0,
                               cudaStream_t s) {
    if (m.use_k1ax) return launch_ax_cg_dmmag(m, v, eb, ne, pidx0, s);
    if (m.use_hi) return launch_ax_cg_hi(m, v, eb, ne, pidx0, s);
    if (m.use_tma) return launch_ax_cg_tma(m, v, eb, ne, pidx0, s);
    return cudaErrorInvalidValue;   // the simple kernel covers all elements only
}

cudaError_t launch_gs(const DevMesh &m, double *w, int mode, const CgVecs *v, cudaStream_t s) {
    GsArgs a{};
    a.cls = m.cls;
    a.idx = m.gs_idx;
    a.ngroups = m.ngroups;
    a.w = w;
    int nb = (m.ngroups + kGsThreads - 1) / kGsThreads;
    if (nb < 1) nb = 1;
    if (mode == 2) {
        a.st = v->st;
        return launch_pdl(gs_kernel<2>, nb, kGsThreads, 0, s, a);
    } else if (mode == 1) {
        gs_kernel<1><<<nb, kGsThreads, 0, s>>>(a);
    } else {
        gs_kernel<0><<<nb, kGsThreads, 0, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_mask(const DevMesh &m, double *w, cudaStream_t s) {
    if (m.ndir == 0) return cudaSuccess;
    mask_kernel<<<(m.ndir + 255) / 256, 256, 0, s>>>(m.cls, m.gs_idx, m.ndir, w);
    return cudaGetLastError();
}

cudaError_t launch_mass(const DevMesh &m, const double *f, double *b, cudaStream_t s) {
    mass_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.L, m.BM, f, b);
    return cudaGetLastError();
}

cudaError_t launch_cg_init(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    cg_init_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.L, v.st, v.x, v.xw);
    return cudaGetLastError();
}

cudaError_t launch_cg_red_pap(const DevMesh &m, const CgVecs &v, const P2PDev *p2p, cudaStream_t s) {
    cg_red_kernel<<<1, kRedThreads, 0, s>>>(v.part1, v.s1, v.nb1, v.pap_all, v.st, 0, m.rank,
                                             m.nranks, p2p, kSitePap);
    return cudaGetLastError();
}

cudaError_t launch_cg_red_rr(const DevMesh &m, const CgVecs &v, const P2PDev *p2p, cudaStream_t s) {
    cg_red_kernel<<<1, kRedThreads, 0, s>>>(v.part2, v.s2, v.nb2, v.rr_all, v.st, 1, m.rank,
                                             m.nranks, p2p, kSiteRr);
    return cudaGetLastError();
}

cudaError_t launch_cg_red_rz(const DevMesh &m, const CgVecs &v, const P2PDev *p2p, cudaStream_t s) {
    cg_red_kernel<<<1, kRedThreads, 0, s>>>(v.part3, v.s2, v.nb2, v.rz_all, v.st, 1, m.rank,
                                             m.nranks, p2p, kSiteRz);
    return cudaGetLastError();
}

cudaError_t launch_diag(const DevMesh &m, double *d, cudaStream_t s) {
    diag_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.n, m.E, m.D, m.G, m.H, d, m.use_hi);
    return cudaGetLastError();
}

cudaError_t launch_recip(const DevMesh &m, const double *d, double *dinv, cudaStream_t s) {
    recip_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.L, d, dinv);
    return cudaGetLastError();
}

cudaError_t launch_cg_finish(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    cg_finish_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.L, v.x, v.xw, v.p, v.st);
    return cudaGetLastError();
}

}  // namespace sem
