// cg_sr.cu -- KB of the single-reduction (Chronopoulos-Gear) CG (NEXT-3,
// DESIGN.md reading R7; a latency-hiding variant of the PCG of
// PAPER.md:672-673), and its start / finish / multi-rank fold kernels.
//
// Iteration k = KA(k) [w = A_L r, (r, w) partials: ax_tma_sr.cu] then KB(k):
//   prologue: gamma_k = (r_k, r_k)_c (partials of KB(k-1)), delta_k = (r_k, w)_c
//             (partials of KA(k)) -> the stopping decision (the ONLY one of the
//             iteration) and alpha_k, beta_k
//   for every global node (surface group: copies summed in ascending local
//   order, Dirichlet groups skipped; element-interior node: itself):
//       w = (Q Q^T w_L)_g;  u = r_g
//       p = u + beta p;  s = w + beta s;  xinc += alpha p;  r_g = u - alpha s
//       r_g written to every copy; gamma_{k+1} partial += r_g^2 (owned)
// p, s and the x increment live in GLOBAL storage (one value per global node
// of the rank), so the extra recurrence of the variant costs no more bytes
// than K1's element-duplicated x / p updates: KA 64 B / local node, KB
// 16 B / surface copy + 56 B / group + 72 B / interior node.
#include <cstring>

#include "cg_device.cuh"
#include "p2p_dev.cuh"
#include "sem_internal.h"

namespace sem {

struct KbArgs {
    GsClasses cls;
    const int32_t *idx;       // class-transposed copies of every surface group
    const uint32_t *own;      // nranks > 1: groups counted in (r,r) on this rank
    int32_t ngroups;
    int64_t E;
    const double *w;
    double *r;
    double *pg, *sg, *xg;     // global storage: p, s, x increment
    CgRed red;
    double *part2;            // (r, r) partials of this kernel, [2][s2]
    const double *sr_all;     // nranks > 1: [kRing][nranks][2] (gamma, delta)
    CgState *st;
    int32_t nich;
    int32_t cchunk[kMaxClasses + 1];
    int32_t nchunks;
};

constexpr int kKbThreads = 256;
constexpr int kKbBlocksPerSM = 3;
constexpr int kKbIntU = 3;          // interior nodes per thread (4 spills: p, s, x ride along)

__host__ __device__ constexpr int kb_upb(int m) { return (m == 1 || m == 2) ? 4 : (m == 4 ? 2 : 1); }

__device__ __forceinline__ bool kb_owned(const KbArgs &a, int g) {
    return !a.own || ((__ldg(a.own + (g >> 5)) >> (g & 31)) & 1u);
}

// interior node t of the rank (element-major, i fastest) -> local index
template <int N>
__device__ __forceinline__ int kb_interior_local(int t) {
    constexpr int n = N + 1, n2 = n * n, n3 = n2 * n, ni = N - 1, NI3 = ni * ni * ni;
    const int e = t / NI3;
    const int q = t - e * NI3;
    const int ii = q % ni, jj = (q / ni) % ni, kk = q / (ni * ni);
    return e * n3 + (kk + 1) * n2 + (jj + 1) * n + (ii + 1);
}

template <int N>
__global__ void __launch_bounds__(kKbThreads, kKbBlocksPerSM) kb_sr_kernel(const __grid_constant__ KbArgs a) {
    constexpr int ni = N - 1, U = kKbIntU, T = kKbThreads;
    __shared__ double sred[2 * (T / 32)];
    const int tid = threadIdx.x;
    const int nint = (int)(a.E * ni * ni * ni);

    // ---- prologue: gamma_k, delta_k -> stop, alpha_k, beta_k (one reduction) ----
    const CgRed &R = a.red;
    const int done = ld_state(&a.st->done);
    const int k = ld_state(&a.st->k2);
    double v[2];
    if (R.nranks == 1) {
        const double g0 = thread_sum<T>(R.part2, R.nb2), g1 = thread_sum<T>(R.part2 + R.s2, R.nb2);
        const double d0 = thread_sum<T>(R.part1, R.nb1), d1 = thread_sum<T>(R.part1 + R.s1, R.nb1);
        v[0] = ((k - 1) & 1) ? g1 : g0;       // gamma_k: partials of KB(k-1) (the start: slot 1)
        v[1] = (k & 1) ? d1 : d0;             // delta_k: partials of KA(k)
    } else {
        v[0] = v[1] = 0.0;
        if (tid == 0) {
            const double *src = a.sr_all + (k & 3) * 2 * R.nranks;
            for (int q = 0; q < R.nranks; ++q) {     // ranks in ascending order
                v[0] += __ldcg(src + 2 * q);
                v[1] += __ldcg(src + 2 * q + 1);
            }
        }
    }
    if (done) return;
    block_sum_vec<T, 2>(v, sred);
    const double gamma = v[0], delta = v[1];
    const double rr0 = (k == 0) ? gamma : __ldcg(&a.st->rho0);
    const bool stop = cg_stop(k, gamma, rr0, a.st->maxit, a.st->tol);
    double alpha, beta;
    if (k == 0) {
        beta = 0.0;
        alpha = gamma / delta;
    } else {
        const double gold = __ldcg(&a.st->gamma_hist[(k - 1) & 1]);
        const double aold = __ldcg(&a.st->alpha_hist[(k - 1) & 1]);
        beta = gamma / gold;
        alpha = gamma / (delta - beta * gamma / aold);
    }
    if (blockIdx.x == 0 && tid == 0) {
        CgState *st = a.st;
        if (k == 0) st->rho0 = rr0;
        if (stop) {
            st->iters = k;
            st->rel_res = (rr0 == 0.0) ? 0.0 : sqrt(gamma) / sqrt(rr0);
            st->converged = (rr0 == 0.0) || !(sqrt(gamma) > st->tol * sqrt(rr0));
            __threadfence();
            st->done = 1;
        } else {
            st->gamma_hist[k & 1] = gamma;
            st->alpha_hist[k & 1] = alpha;
            st->k1 = k + 1;              // for KA of k+1
        }
    }
    if (stop) return;

    // ---- body: interior chunks, then the surface-group classes ----
    double part = 0.0;
    for (int ch = blockIdx.x; ch < a.nchunks; ch += gridDim.x) {
        if (ch < a.nich) {
            if constexpr (ni > 0) {
                int l[U], t[U];
                double u[U], wv[U], pv[U], sv[U], xv[U];
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    t[q] = (ch * U + q) * T + tid;
                    l[q] = (t[q] < nint) ? kb_interior_local<N>(t[q]) : -1;
                }
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    if (l[q] >= 0) {
                        const int sl = a.ngroups + t[q];
                        u[q] = a.r[l[q]];
                        wv[q] = __ldcs(a.w + l[q]);
                        pv[q] = a.pg[sl];
                        sv[q] = a.sg[sl];
                        xv[q] = a.xg[sl];
                    }
                }
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    if (l[q] >= 0) {
                        const int sl = a.ngroups + t[q];
                        const double p = u[q] + beta * pv[q];
                        const double s = wv[q] + beta * sv[q];
                        a.pg[sl] = p;
                        a.sg[sl] = s;
                        a.xg[sl] = xv[q] + alpha * p;
                        const double rn = u[q] - alpha * s;
                        a.r[l[q]] = rn;
                        part += rn * rn;
                    }
                }
            }
            continue;
        }
        const int cg = ch - a.nich;
        int c = 0;
        while (cg >= a.cchunk[c + 1]) ++c;
        const int cnt = a.cls.start[c + 1] - a.cls.start[c];
        const int m = a.cls.m[c];
        const int32_t *ix = a.idx + a.cls.idxoff[c];
        const int gs0 = a.cls.start[c];
        const int upb = kb_upb(m);
        const int base = (cg - a.cchunk[c]) * T * upb + tid;
        for (int q0 = 0; q0 < upb; ++q0) {
            const int q = base + q0 * T;
            if (q >= cnt) break;
            const int g = gs0 + q;
            const int l0 = __ldg(ix + q);
            double sw = a.w[l0];
            for (int t = 1; t < m; ++t) sw += a.w[__ldg(ix + t * cnt + q)];   // ascending local order
            const double u = a.r[l0];
            const double p = u + beta * a.pg[g];
            const double s = sw + beta * a.sg[g];
            a.pg[g] = p;
            a.sg[g] = s;
            a.xg[g] = a.xg[g] + alpha * p;
            const double rn = u - alpha * s;
            for (int t = 0; t < m; ++t) a.r[__ldg(ix + t * cnt + q)] = rn;
            if (kb_owned(a, g)) part += rn * rn;
        }
    }
    const double bs = block_sum<T>(part, sred);
    if (tid == 0) a.part2[(k & 1) * a.red.s2 + blockIdx.x] = bs;
}

// start: zero the global-storage p, s, x increment; reset the state (k = 0)
__global__ void sr_init_kernel(int64_t nslots, double *pg, double *sg, double *xg, CgState *st) {
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nslots;
         q += (int64_t)gridDim.x * blockDim.x) {
        pg[q] = 0.0;
        sg[q] = 0.0;
        xg[q] = 0.0;
    }
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

// finish: x += (x increment) at every copy of every non-Dirichlet global node
template <int N>
__global__ void sr_finish_kernel(const __grid_constant__ GsClasses cls, const int32_t *__restrict__ idx,
                                 int32_t ngroups, int64_t E, const double *__restrict__ xg, double *x) {
    constexpr int ni = N - 1;
    const int64_t nint = E * ni * ni * ni;
    const int64_t total = ngroups + nint;
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
         q += (int64_t)gridDim.x * blockDim.x) {
        if (q < ngroups) {
            const int g = (int)q;
            int c = 0;
            while (c + 1 < cls.n && g >= cls.start[c + 1]) ++c;
            if (cls.dir[c]) continue;
            const int m = cls.m[c], cnt = cls.start[c + 1] - cls.start[c], gl = g - cls.start[c];
            const int32_t *ix = idx + cls.idxoff[c];
            const double d = xg[g];
            for (int t = 0; t < m; ++t) x[ix[t * cnt + gl]] += d;
        } else if constexpr (ni > 0) {
            const int t = (int)(q - ngroups);
            x[kb_interior_local<N>(t)] += xg[q];
        }
    }
}

// nranks > 1: this rank's (gamma_k, delta_k) into sr_all[k & 3][rank] before
// the one all-gather of the iteration (k from KA(k): st->k2); with the
// peer-memory transport (p2p != nullptr) this kernel also performs the
// all-gather of the (gamma, delta) pair (warp 0), even after the stop
constexpr int kFoldThreads = 256;
__global__ void __launch_bounds__(kFoldThreads) sr_fold_kernel(CgRed R, double *sr_all, const CgState *st,
                                                               int rank, const P2PDev *p2p) {
    __shared__ double sred[2 * (kFoldThreads / 32)];
    const bool done = ld_state(&st->done);
    const int k = ld_state(&st->k2);
    if (!done) {
        double v[2];
        v[0] = thread_sum<kFoldThreads>(R.part2 + ((k - 1) & 1) * R.s2, R.nb2);
        v[1] = thread_sum<kFoldThreads>(R.part1 + (k & 1) * R.s1, R.nb1);
        block_sum_vec<kFoldThreads, 2>(v, sred);
        if (threadIdx.x == 0) {
            sr_all[(k & 3) * 2 * R.nranks + 2 * rank] = v[0];
            sr_all[(k & 3) * 2 * R.nranks + 2 * rank + 1] = v[1];
        }
    } else if (!p2p) {
        return;
    }
    if (p2p) {
        __syncthreads();
        if (threadIdx.x < 32) p2p_allgather_warp(*p2p, kSiteSr, sr_all + (k & 3) * 2 * R.nranks, 2);
    }
}

#define SEM_SR_DISPATCH(N_, ...)                                             \
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

static int grid_sr(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

static int64_t sr_slots(const DevMesh &m) {
    return m.ngroups + m.E * int64_t(m.N - 1) * (m.N - 1) * (m.N - 1);
}

cudaError_t launch_kb_sr(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    KbArgs a{};
    a.cls = m.cls;
    a.idx = m.gs_idx;
    a.own = m.own;
    a.ngroups = m.ngroups;
    a.E = m.E;
    a.w = v.w;
    a.r = v.r;
    a.pg = v.p;
    a.sg = v.z;
    a.xg = v.xw;
    a.red = make_red(m, v);
    a.red.nb1 = ka_blocks(m);            // delta's partials come from KA, not K1
    a.part2 = v.part2;
    a.sr_all = v.rr_all;
    a.st = v.st;
    const int64_t nint = m.E * int64_t(m.N - 1) * (m.N - 1) * (m.N - 1);
    a.nich = (int)((nint + kKbIntU * kKbThreads - 1) / (kKbIntU * kKbThreads));
    int nch = 0;
    for (int c = 0; c < m.cls.n; ++c) {
        a.cchunk[c] = nch;
        const int cnt = m.cls.start[c + 1] - m.cls.start[c];
        const int per = kKbThreads * kb_upb(m.cls.m[c]);
        if (!m.cls.dir[c]) nch += (cnt + per - 1) / per;
    }
    a.cchunk[m.cls.n] = nch;
    a.nchunks = a.nich + nch;
    // the same grid as K2: its (r,r) partial count nb2 (the start's K2 INIT
    // provides gamma_0's partials)
    const int nb = v.nb2;
    SEM_SR_DISPATCH(m.N, (kb_sr_kernel<NN><<<nb, kKbThreads, 0, s>>>(a)));
    return cudaGetLastError();
}

cudaError_t launch_sr_init(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    const int64_t n = sr_slots(m);
    sr_init_kernel<<<grid_sr(n), 256, 0, s>>>(n, v.p, v.z, v.xw, v.st);
    return cudaGetLastError();
}

cudaError_t launch_sr_finish(const DevMesh &m, const CgVecs &v, cudaStream_t s) {
    const int64_t n = sr_slots(m);
    SEM_SR_DISPATCH(m.N, (sr_finish_kernel<NN><<<grid_sr(n), 256, 0, s>>>(m.cls, m.gs_idx, m.ngroups,
                                                                          m.E, v.xw, v.x)));
    return cudaGetLastError();
}

cudaError_t launch_sr_fold(const DevMesh &m, const CgVecs &v, const P2PDev *p2p, cudaStream_t s) {
    CgRed R = make_red(m, v);
    R.nb1 = ka_blocks(m);
    sr_fold_kernel<<<1, kFoldThreads, 0, s>>>(R, v.rr_all, v.st, m.rank, p2p);
    return cudaGetLastError();
}

}  // namespace sem
