// sem_kernels.cu -- sm_100a kernels of the SEM Poisson hot path (arXiv 1403.0968,
// PAPER.md:578-784).  FP64 on the CUDA cores: the operator is HBM-bound at
// 64 B per local node (u, six G^ factors, w) and tcgen05 has no FP64 kind.
//
//   geom_kernel      a1: isoparametric geometric factors G^ = w J (dr/dx)(dr/dx)^T
//   ax_kernel<N,..>  a3-a5: w = D^T G^ D u per element (sum factorisation)
//   gs_kernel        a6/a8: Q Q^T over element-surface groups (+ mask, + (w,p)_c)
//   rr_kernel        a9: r -= alpha w and (r,r)_c, deterministic last-block reduce
//
// Layout: local node (i,j,k) of element e at e*n^3 + i + n*j + n^2*k.
#include <cstdio>

#include "sem_internal.h"

namespace sem {

// --------------------------------------------------------------------------
// helpers
// --------------------------------------------------------------------------
template <int NT>
__device__ __forceinline__ double block_sum(double v, double *red) {
    // deterministic: fixed shuffle tree per warp, then warp 0 sums the warp
    // results in warp order.
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
    return s;  // valid in thread 0 only
}

// Fixed-order sum of cnt partials by one whole block (deterministic for a
// fixed blockDim).  Result valid in thread 0.
template <int NT>
__device__ double block_sum_array(const double *a, int cnt, double *red) {
    double s = 0.0;
    for (int t = threadIdx.x; t < cnt; t += NT) s += __ldcg(a + t);
    return block_sum<NT>(s, red);
}

// Last-block-done protocol: every block has written its partial; returns true
// in the block that arrived last (all partials are then visible to it).
__device__ __forceinline__ bool last_block(uint32_t *ticket, int *sflag) {
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = atomicAdd(ticket, 1u);
        *sflag = (t == gridDim.x - 1);
    }
    __syncthreads();
    bool last = *sflag;
    if (last) __threadfence();
    return last;
}

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
                            double *__restrict__ G, double *__restrict__ BM, int *bad) {
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
        double *Ge = G + e * 6 * n3 + q;
        for (int f = 0; f < 6; ++f) Ge[f * n3] = g[f];
        BM[l] = wJ;
    }
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
//   per-block partial of (w,p) over element-interior nodes.
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
    double *x, *p, *w;
    double *partials;
    const double *rr_all;
    CgState *st;
    int k, nranks;
};

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
    __shared__ double sred[(NT + 31) / 32];

    double beta = 0.0, alpha_prev = 0.0;
    if constexpr (CG) {
        CgState *st = cg.st;
        if (*(volatile int32_t *)&st->done) return;
        const int k = cg.k;
        const double rho = sum_ranks(cg.rr_all + (k & 3) * cg.nranks, cg.nranks);
        double rho0 = (k == 0) ? rho : st->rho0;
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
            return;
        }
        if (k == 0) {
            if (blockIdx.x == 0 && threadIdx.x == 0) st->rho0 = rho0;
        } else {
            const double rho_old = sum_ranks(cg.rr_all + ((k - 1) & 3) * cg.nranks, cg.nranks);
            beta = rho / rho_old;
            alpha_prev = st->alpha[(k - 1) & 3];
        }
    }

    const int tid = threadIdx.x;
    for (int t = tid; t < n2; t += NT) sD[t] = Dg[t];
    const int el = tid / n2;
    const int ij = tid - el * n2;
    const int i = ij % n, j = ij / n;
    const int64_t e = (int64_t)blockIdx.x * EPB + el;
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
                if (cg.k == 0) {
                    pl = rl;
                } else {
                    const double po = cg.p[l];
                    cg.x[l] += alpha_prev * po;
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
    }
    if constexpr (CG) {
        double part = 0.0;
        if (active && i > 0 && i < N && j > 0 && j < N) {
#pragma unroll
            for (int k = 1; k < N; ++k) part += rw[k] * ru[k];
        }
        const double s = block_sum<NT>(part, sred);
        if (tid == 0) cg.partials[blockIdx.x] = s;
    }
}

// --------------------------------------------------------------------------
// a6/a8: gather-scatter over element-surface groups, one thread per group.
// mode 0: Q Q^T; 1: + mask; 2: + mask + (w,p)_c partial with last-block
// reduction of [Ax partials | gs partials] into pap_all[k&3][rank].
// --------------------------------------------------------------------------
struct GsArgs {
    const int32_t *off, *idx;
    int32_t ngroups, ndir;
    double *w;
    const double *p;
    double *partials;     // Ax partials [0, nb_ax), gs partials after
    int nb_ax;
    double *pap_out;
    CgState *st;
};

template <int MODE>
__global__ void __launch_bounds__(kGsThreads) gs_kernel(GsArgs a) {
    __shared__ double sred[kGsThreads / 32];
    __shared__ int sflag;
    if constexpr (MODE == 2) {
        if (*(volatile int32_t *)&a.st->done) return;
    }
    const int g = blockIdx.x * kGsThreads + threadIdx.x;
    double part = 0.0;
    if (g < a.ngroups) {
        const int o0 = a.off[g], o1 = a.off[g + 1];
        double s = 0.0;
        for (int t = o0; t < o1; ++t) s += a.w[a.idx[t]];
        if (MODE >= 1 && g < a.ndir) s = 0.0;
        for (int t = o0; t < o1; ++t) a.w[a.idx[t]] = s;
        if (MODE == 2 && g >= a.ndir) part = s * a.p[a.idx[o0]];
    }
    if constexpr (MODE == 2) {
        const double bs = block_sum<kGsThreads>(part, sred);
        if (threadIdx.x == 0) a.partials[a.nb_ax + blockIdx.x] = bs;
        if (last_block(&a.st->ticket[0], &sflag)) {
            const double tot = block_sum_array<kGsThreads>(a.partials, a.nb_ax + gridDim.x, sred);
            if (threadIdx.x == 0) {
                *a.pap_out = tot;
                a.st->ticket[0] = 0;
            }
        }
    }
}

__global__ void mask_kernel(const int32_t *__restrict__ off, const int32_t *__restrict__ idx,
                            int32_t ndir, double *__restrict__ w) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g < ndir)
        for (int t = off[g]; t < off[g + 1]; ++t) w[idx[t]] = 0.0;
}

__global__ void mass_kernel(int64_t L, const double *__restrict__ BM, const double *f,
                            double *b) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x)
        b[l] = BM[l] * f[l];
}

__global__ void cg_init_kernel(int64_t L, const double *__restrict__ b,
                               const double *__restrict__ w, double *__restrict__ r,
                               CgState *st) {
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x)
        r[l] = b[l] - w[l];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->done = 0;
        st->iters = 0;
        st->converged = 0;
        st->rel_res = 0.0;
        for (int q = 0; q < kRing; ++q) st->alpha[q] = 0.0;
        st->ticket[0] = st->ticket[1] = 0;
    }
}

// a9: r -= alpha_k w (update) and (r,r)_c over owner copies.
template <bool UPDATE>
__global__ void __launch_bounds__(kRrThreads)
rr_kernel(int64_t L, double *__restrict__ r, const double *__restrict__ w,
          const uint32_t *__restrict__ owner, double *partials, const double *rr_in,
          const double *pap_all, double *rr_out, CgState *st, int k, int nranks) {
    __shared__ double sred[kRrThreads / 32];
    __shared__ int sflag;
    double alpha = 0.0;
    if constexpr (UPDATE) {
        if (*(volatile int32_t *)&st->done) return;
        const double rho = sum_ranks(rr_in, nranks);
        const double pap = sum_ranks(pap_all, nranks);
        alpha = rho / pap;
        if (blockIdx.x == 0 && threadIdx.x == 0) st->alpha[k & 3] = alpha;
    }
    double part = 0.0;
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x) {
        double rl = r[l];
        if constexpr (UPDATE) {
            rl -= alpha * w[l];
            r[l] = rl;
        }
        if ((__ldg(owner + (l >> 5)) >> (l & 31)) & 1u) part += rl * rl;
    }
    const double bs = block_sum<kRrThreads>(part, sred);
    if (threadIdx.x == 0) partials[blockIdx.x] = bs;
    if (last_block(&st->ticket[1], &sflag)) {
        const double tot = block_sum_array<kRrThreads>(partials, gridDim.x, sred);
        if (threadIdx.x == 0) {
            *rr_out = tot;
            st->ticket[1] = 0;
        }
    }
}

__global__ void cg_finish_kernel(int64_t L, double *__restrict__ x,
                                 const double *__restrict__ p, const CgState *st) {
    const int it = st->iters;
    if (it < 1) return;
    const double a = st->alpha[(it - 1) & 3];
    for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < L;
         l += (int64_t)gridDim.x * blockDim.x)
        x[l] += a * p[l];
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

static int grid_for(int64_t L, int threads) {
    int64_t b = (L + threads - 1) / threads;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

cudaError_t launch_geom(const DevMesh &m, const double *xyz, double *G, double *BM,
                        int *bad, cudaStream_t s) {
    // D and the 1-D weights live at the start of the D buffer: [n*n] D, [n] w
    geom_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.n, m.E, m.D, m.D + m.n * m.n, xyz, G, BM,
                                                   bad);
    return cudaGetLastError();
}

cudaError_t launch_ax(const DevMesh &m, const double *u, double *w, cudaStream_t s) {
    if (m.E == 0) return cudaSuccess;
    if (m.use_tma) return launch_ax_tma(m, u, w, s);
    AxCgArgs none{};
    SEM_DISPATCH_N(m.N, (ax_kernel<NN, false><<<ax_blocks_t<NN>(m.E), AxCfg<NN>::NT, 0, s>>>(
                             m.E, m.D, m.G, u, w, none)));
    return cudaGetLastError();
}

cudaError_t launch_ax_cg(const DevMesh &m, const CgVecs &v, int k, cudaStream_t s) {
    if (m.use_tma) return launch_ax_cg_tma(m, v, k, s);
    AxCgArgs a{v.r, v.x, v.p, v.w, v.partials, v.rr_all, v.st, k, m.nranks};
    SEM_DISPATCH_N(m.N, (ax_kernel<NN, true><<<ax_blocks_t<NN>(m.E), AxCfg<NN>::NT, 0, s>>>(
                             m.E, m.D, m.G, nullptr, v.w, a)));
    return cudaGetLastError();
}

cudaError_t launch_gs(const DevMesh &m, double *w, int mode, const CgVecs *v, int k, int nb_ax,
                      cudaStream_t s) {
    GsArgs a{};
    a.off = m.gs_off;
    a.idx = m.gs_idx;
    a.ngroups = m.ngroups;
    a.ndir = m.ndir;
    a.w = w;
    int nb = (m.ngroups + kGsThreads - 1) / kGsThreads;
    if (nb < 1) nb = 1;
    if (mode == 2) {
        a.p = v->p;
        a.partials = v->partials;
        a.nb_ax = nb_ax;
        a.pap_out = v->pap_all + (k & 3) * m.nranks + m.rank;
        a.st = v->st;
        gs_kernel<2><<<nb, kGsThreads, 0, s>>>(a);
    } else if (mode == 1) {
        gs_kernel<1><<<nb, kGsThreads, 0, s>>>(a);
    } else {
        gs_kernel<0><<<nb, kGsThreads, 0, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_mask(const DevMesh &m, double *w, cudaStream_t s) {
    if (m.ndir == 0) return cudaSuccess;
    mask_kernel<<<(m.ndir + 255) / 256, 256, 0, s>>>(m.gs_off, m.gs_idx, m.ndir, w);
    return cudaGetLastError();
}

cudaError_t launch_mass(const DevMesh &m, const double *f, double *b, cudaStream_t s) {
    mass_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.L, m.BM, f, b);
    return cudaGetLastError();
}

cudaError_t launch_cg_init(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    cg_init_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.L, v.b, v.w, v.r, v.st);
    return cudaGetLastError();
}

cudaError_t launch_rr(const DevMesh &m, const CgVecs &v, int k, bool update, cudaStream_t s) {
    const int P = m.nranks;
    if (update) {
        rr_kernel<true><<<kRrBlocks, kRrThreads, 0, s>>>(
            m.L, v.r, v.w, m.owner, v.partials, v.rr_all + (k & 3) * P, v.pap_all + (k & 3) * P,
            v.rr_all + ((k + 1) & 3) * P + m.rank, v.st, k, P);
    } else {
        rr_kernel<false><<<kRrBlocks, kRrThreads, 0, s>>>(m.L, v.r, v.w, m.owner, v.partials,
                                                          nullptr, nullptr, v.rr_all + m.rank,
                                                          v.st, 0, P);
    }
    return cudaGetLastError();
}

cudaError_t launch_cg_finish(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    cg_finish_kernel<<<grid_for(m.L, 256), 256, 0, s>>>(m.L, v.x, v.p, v.st);
    return cudaGetLastError();
}

}  // namespace sem
