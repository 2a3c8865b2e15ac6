// cg_update.cu -- K2 of the CG iteration: the
// direct-stiffness summation of w = A_L p fused with the residual update and
// the new residual norm (PAPER.md:667 global-local numbering; :672-673 PCG):
//
//   for every element-surface global node g (one thread):
//       s_g = sum of its local copies of w, ascending local order  (= Q Q^T w)
//       Dirichlet: nothing (r stays 0, contributes 0)              (mask)
//       else      r_g <- r_g - alpha s_g, written to every copy; rho += r_g^2
//   for every element-interior node (m = 1, never Dirichlet):
//       r <- r - alpha w; rho += r^2
//
// so the assembled w is never written back, (r,r)_c needs no weights (each
// global node is visited once) and one launch + one reduction replaces the
// gather-scatter pass and the separate r-update pass.  alpha = rho_k / pAp_k
// with pAp from K1.  INIT = true forms r0 = mask (b - Q Q^T A_L x0) and rho_0.
// PC = true (Jacobi PCG, NEXT-2): also z = dinv r at every copy (dinv is
// continuous: read once per group) and the second partial (r, z).
#include "cg_device.cuh"
#include "sem_internal.h"

namespace sem {

struct K2Args {
    GsClasses cls;
    const int32_t *idx;       // class-transposed copies of every surface group
    const uint32_t *own;      // nranks > 1: groups counted in (r,r) on this rank
    int32_t ngroups;
    int64_t E;
    const double *w;
    const double *b;          // INIT only
    double *r;
    CgRed red;                // where the scalar reductions live
    double *part2;            // this kernel's (r, r) partials, [2][s2]
    const double *dinv;       // PC: Jacobi inverse diagonal (continuous, 0 on Dirichlet)
    double *z;                // PC: z = dinv r
    double *part3;            // PC: (r, z) partials, [2][s2]
    CgState *st;
    int32_t nich;                      // element-interior chunks (first)
    int32_t cchunk[kMaxClasses + 1];   // then: first group chunk of each class
    int32_t nchunks;
};

#ifndef SEM_PDL_LATE
#define SEM_PDL_LATE 1
#endif
constexpr bool PDL_LATE_K2 = SEM_PDL_LATE != 0;

constexpr int kK2Threads = 256;
constexpr int kK2BlocksPerSM = 3;
constexpr int kK2IntU = 4;           // element-interior nodes per thread per chunk

// groups per thread in one chunk, by multiplicity
// (the PC kernel carries dinv and z as well: half the groups per thread, or
// its registers spill)
// (pc && !zs: dinv but no z stores -- three face groups per thread fit)
__host__ __device__ constexpr int k2_upb(int m, bool pc = false, bool zs = true) {
    return pc ? ((m == 1 || m == 2) ? (zs ? 2 : 3) : 1) : ((m == 1 || m == 2) ? 4 : (m == 4 ? 2 : 1));
}

// One batch of U groups of a class with compile-time multiplicity M (M = 0:
// runtime m, up to 8).  All index loads, then all value loads, are issued
// before any use, so a thread keeps U*M requests in flight.
__device__ __forceinline__ bool k2_owned(const K2Args &a, int g) {
    return !a.own || ((__ldg(a.own + (g >> 5)) >> (g & 31)) & 1u);
}

template <int M, int U, bool INIT, bool PC, bool ZS = PC>
__device__ __forceinline__ void k2_groups(const K2Args &a, const int32_t *__restrict__ ix, int m,
                                          int cnt, int q0, int qstride, double alpha, int gstart,
                                          double &part, double &partz) {
    constexpr int MM = M ? M : 8;
    const int mm = M ? M : m;
    int li[U][MM];
    bool on[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int q = q0 + u * qstride;
        on[u] = q < cnt;
#pragma unroll
        for (int t = 0; t < MM; ++t) li[u][t] = (on[u] && t < mm) ? __ldg(ix + t * cnt + q) : 0;
    }
    double v[U][MM], r0[U], dv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int t = 0; t < MM; ++t) v[u][t] = (on[u] && t < mm) ? a.w[li[u][t]] : 0.0;
        r0[u] = on[u] ? (INIT ? a.b[li[u][0]] : a.r[li[u][0]]) : 0.0;
        if constexpr (PC) dv[u] = on[u] ? __ldg(a.dinv + li[u][0]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        if (!on[u]) continue;
        double s = v[u][0];
#pragma unroll
        for (int t = 1; t < MM; ++t)
            if (t < mm) s += v[u][t];                        // ascending local order
        const double rn = INIT ? r0[u] - s : r0[u] - alpha * s;
        const bool own = k2_owned(a, gstart + q0 + u * qstride);
#pragma unroll
        for (int t = 0; t < MM; ++t)
            if (t < mm) a.r[li[u][t]] = rn;
        if (own) part += rn * rn;
        if constexpr (PC) {
            const double zn = dv[u] * rn;
            if constexpr (ZS) {
#pragma unroll
                for (int t = 0; t < MM; ++t)
                    if (t < mm) a.z[li[u][t]] = zn;
            }
            if (own) partz += rn * zn;
        }
    }
}

// Element-interior nodes of one chunk (m = 1, never Dirichlet): local
// indices of this thread's U nodes (-1 past the end), i fastest.  Interior
// node t is node q = t mod (N-1)^3 of element e = t div (N-1)^3; its offset
// inside the element comes from a shared-memory table (ioff[q], filled once
// per block), which replaces the per-node (i, j, k) division chain (ncu r02i:
// 22% of K2's instructions).  Consecutive threads keep consecutive interior
// nodes, so the loads stay coalesced (a row-segment-per-thread layout that
// also cut the arithmetic measured 26% slower, r02k: a warp's loads then span
// 32 rows).
template <int N>
struct K2Int {
    static constexpr int ni = N - 1, NI3 = ni * ni * ni;
};
template <int N>
__device__ __forceinline__ void k2_interior_table(int32_t *ioff) {
    constexpr int n = N + 1, n2 = n * n, ni = N - 1, NI3 = ni * ni * ni;
    for (int q = threadIdx.x; q < NI3; q += kK2Threads) {
        const int ii = q % ni, jj = (q / ni) % ni, kk = q / (ni * ni);
        ioff[q] = (kk + 1) * n2 + (jj + 1) * n + (ii + 1);
    }
}
template <int N, int U>
__device__ __forceinline__ void k2_interior_idx(int64_t E, int chunk, const int32_t *ioff,
                                                int (&l)[U]) {
    constexpr int n = N + 1, n3 = n * n * n, ni = N - 1, NI3 = ni * ni * ni;
    const int nint = (int)(E * NI3);
    const int t0 = chunk * kK2Threads * U + threadIdx.x;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int t = t0 + u * kK2Threads;
        const int tt = t < nint ? t : 0;
        const int e = tt / NI3;
        const int q = tt - e * NI3;
        l[u] = (t < nint) ? e * n3 + ioff[q] : -1;
    }
}

// ZS (PC only): store z = dinv r at every copy; false when K1 forms z from r
// and dinv itself (pcg_z_in_k1: N = 7 tensor-core K1), the (r, z) partial stays
template <int N, bool INIT, bool PC, bool ZS = PC>
__global__ void __launch_bounds__(kK2Threads, kK2BlocksPerSM) k2_kernel(const __grid_constant__ K2Args a) {
    constexpr int ni = N - 1;
    constexpr int U = kK2IntU;
    __shared__ double sred[3 * (kK2Threads / 32)];
    __shared__ int32_t ioff[ni > 0 ? ni * ni * ni : 1];
    if constexpr (!INIT && !PDL_LATE_K2) pdl_trigger();
    if constexpr (!INIT) pdl_wait();
    if constexpr (ni > 0) {
        k2_interior_table<N>(ioff);
        __syncthreads();
    }

    // Chunks: [0, nich) element-interior nodes (kK2Threads * U each), then
    // [nich + cchunk[c], nich + cchunk[c+1]) the groups of class c
    // (kK2Threads * U_m each).  A block walks chunks blockIdx.x, +gridDim.x, ...
    // Its first chunk is interior whenever there are enough of them, and its
    // loads are issued right after the scalar prologue's loads, before the
    // prologue consumes them.
    const int nich = a.nich;
    int ch = blockIdx.x;
    int l[U];
    double rv[U], wv[U], dv[U];
    bool staged = false;
    // the scalar loads go out first (L2-resident, ahead of the staged chunk)
    K2Pre pre;
    if constexpr (!INIT) cg_k2_load<kK2Threads, PC>(a.st, a.red, pre);
    if constexpr (ni > 0) {
        if (ch < nich) {
            k2_interior_idx<N, U>(a.E, ch, ioff, l);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (l[u] >= 0) {
                    rv[u] = INIT ? a.b[l[u]] : a.r[l[u]];
                    wv[u] = __ldcs(a.w + l[u]);
                    if constexpr (PC) dv[u] = __ldg(a.dinv + l[u]);
                }
            }
            staged = true;
        }
    }

    double alpha = 0.0;
    int k = -1;               // INIT produces the partials of rho_0 as "iteration -1"
    if constexpr (!INIT) {
        const CgStep c = cg_k2_finish<kK2Threads, PC>(a.st, a.red, sred, pre, alpha);
        if (c.done) return;
        k = c.k;
    }

    double part = 0.0, partz = 0.0;
    for (; ch < a.nchunks; ch += gridDim.x) {
        if (ch < nich) {
            if constexpr (ni > 0) {
                if (!staged) {
                    k2_interior_idx<N, U>(a.E, ch, ioff, l);
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (l[u] >= 0) {
                            rv[u] = INIT ? a.b[l[u]] : a.r[l[u]];
                            wv[u] = __ldcs(a.w + l[u]);
                            if constexpr (PC) dv[u] = __ldg(a.dinv + l[u]);
                        }
                    }
                }
                staged = false;
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (l[u] >= 0) {
                        const double rn = INIT ? rv[u] - wv[u] : rv[u] - alpha * wv[u];
                        a.r[l[u]] = rn;
                        part += rn * rn;
                        if constexpr (PC) {
                            const double zn = dv[u] * rn;
                            if constexpr (ZS) a.z[l[u]] = zn;
                            partz += rn * zn;
                        }
                    }
                }
            }
            continue;
        }
        const int cg = ch - nich;
        int c = 0;
        while (cg >= a.cchunk[c + 1]) ++c;
        const int cnt = a.cls.start[c + 1] - a.cls.start[c];
        const int m = a.cls.m[c];
        const int32_t *ix = a.idx + a.cls.idxoff[c];
        const int gs0 = a.cls.start[c];
        const int base = (cg - a.cchunk[c]) * kK2Threads * k2_upb(m, PC, ZS) + threadIdx.x;
        if (a.cls.dir[c]) {
            // Dirichlet (INIT only): r0 = 0 at every copy (mask)
            for (int u = 0; u < k2_upb(m, PC, ZS); ++u) {
                const int q = base + u * kK2Threads;
                if (q < cnt)
                    for (int t = 0; t < m; ++t) {
                        a.r[__ldg(ix + t * cnt + q)] = 0.0;
                        if constexpr (PC && ZS) a.z[__ldg(ix + t * cnt + q)] = 0.0;
                    }
            }
            continue;
        }
        switch (m) {
        case 1: k2_groups<1, k2_upb(1, PC, ZS), INIT, PC, ZS>(a, ix, m, cnt, base, kK2Threads, alpha, gs0, part, partz); break;
        case 2: k2_groups<2, k2_upb(2, PC, ZS), INIT, PC, ZS>(a, ix, m, cnt, base, kK2Threads, alpha, gs0, part, partz); break;
        case 4: k2_groups<4, k2_upb(4, PC, ZS), INIT, PC, ZS>(a, ix, m, cnt, base, kK2Threads, alpha, gs0, part, partz); break;
        case 8: k2_groups<8, 1, INIT, PC, ZS>(a, ix, m, cnt, base, kK2Threads, alpha, gs0, part, partz); break;
        default: {
            const int q = base;
            if (q < cnt) {
                double s = a.w[__ldg(ix + q)];
                for (int t = 1; t < m; ++t) s += a.w[__ldg(ix + t * cnt + q)];
                const double r0 = INIT ? a.b[__ldg(ix + q)] : a.r[__ldg(ix + q)];
                const double rn = INIT ? r0 - s : r0 - alpha * s;
                for (int t = 0; t < m; ++t) a.r[__ldg(ix + t * cnt + q)] = rn;
                const bool own = k2_owned(a, gs0 + q);
                if (own) part += rn * rn;
                if constexpr (PC) {
                    const double zn = __ldg(a.dinv + __ldg(ix + q)) * rn;
                    if constexpr (ZS)
                        for (int t = 0; t < m; ++t) a.z[__ldg(ix + t * cnt + q)] = zn;
                    if (own) partz += rn * zn;
                }
            }
        } break;
        }
    }

    if constexpr (!INIT && PDL_LATE_K2) pdl_trigger();   // dependents launch during the tail
    // one deterministic partial per block; consumers reduce (cg_device.cuh)
    if constexpr (PC) {
        double v2[2] = {part, partz};
        block_sum_vec<kK2Threads, 2>(v2, sred);
        if (threadIdx.x == 0) {
            a.part2[(k & 1) * a.red.s2 + blockIdx.x] = v2[0];
            a.part3[(k & 1) * a.red.s2 + blockIdx.x] = v2[1];
        }
    } else {
        const double bs = block_sum<kK2Threads>(part, sred);
        if (threadIdx.x == 0) a.part2[(k & 1) * a.red.s2 + blockIdx.x] = bs;
    }
}

#define SEM_K2_DISPATCH(N_, ...)                                             \
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
    case 11: { constexpr int NN = 11; __VA_ARGS__; } break;                  \
    case 12: { constexpr int NN = 12; __VA_ARGS__; } break;                  \
    case 13: { constexpr int NN = 13; __VA_ARGS__; } break;                  \
    case 14: { constexpr int NN = 14; __VA_ARGS__; } break;                  \
    case 15: { constexpr int NN = 15; __VA_ARGS__; } break;                  \
    default: break;                                                          \
    }

// Same grid for the start and the iterations: it is the count of (r,r) partials.
int k2_blocks(const DevMesh &m, bool) { return m.nsm * kK2BlocksPerSM; }

cudaError_t launch_k2(const DevMesh &m, const CgVecs &v, bool init, cudaStream_t s) {
    // Jacobi PCG with a K1 that forms z itself (N = 7 tensor cores): no z stores
    const bool zs = !(v.dinv && pcg_z_in_k1(m) && m.N == 7);
    K2Args a{};
    a.cls = m.cls;
    a.idx = m.gs_idx;
    a.own = m.own;
    a.ngroups = m.ngroups;
    a.E = m.E;
    a.w = v.w;
    a.b = v.b;
    a.r = v.r;
    a.red = make_red(m, v);
    a.part2 = v.part2;
    a.dinv = v.dinv;
    a.z = v.z;
    a.part3 = v.part3;
    a.st = v.st;
    // chunk table: interior chunks first, then the group classes (Dirichlet
    // classes only at INIT)
    const int64_t nint = m.E * int64_t(m.N - 1) * (m.N - 1) * (m.N - 1);
    a.nich = (int)((nint + kK2IntU * kK2Threads - 1) / (kK2IntU * kK2Threads));
    int nch = 0;
    for (int c = 0; c < m.cls.n; ++c) {
        a.cchunk[c] = nch;
        const int cnt = m.cls.start[c + 1] - m.cls.start[c];
        const int per = kK2Threads * k2_upb(m.cls.m[c], v.dinv != nullptr, zs);
        if (!m.cls.dir[c] || init) nch += (cnt + per - 1) / per;
    }
    a.cchunk[m.cls.n] = nch;
    a.nchunks = a.nich + nch;
    const int nb = k2_blocks(m, init);
    cudaError_t e = cudaSuccess;
    const bool pc = v.dinv != nullptr;
    if (init && pc && !zs) {
        if (m.N == 7) k2_kernel<7, true, true, false><<<nb, kK2Threads, 0, s>>>(a), e = cudaGetLastError();
    } else if (pc && !zs) {
        if (m.N == 7) e = launch_pdl(k2_kernel<7, false, true, false>, nb, kK2Threads, 0, s, a);
    } else if (init && pc) {
        SEM_K2_DISPATCH(m.N, (k2_kernel<NN, true, true><<<nb, kK2Threads, 0, s>>>(a), e = cudaGetLastError()));
    } else if (init) {
        SEM_K2_DISPATCH(m.N, (k2_kernel<NN, true, false><<<nb, kK2Threads, 0, s>>>(a), e = cudaGetLastError()));
    } else if (pc) {
        SEM_K2_DISPATCH(m.N, e = launch_pdl(k2_kernel<NN, false, true>, nb, kK2Threads, 0, s, a));
    } else {
        SEM_K2_DISPATCH(m.N, e = launch_pdl(k2_kernel<NN, false, false>, nb, kK2Threads, 0, s, a));
    }
    return e;
}

}  // namespace sem
