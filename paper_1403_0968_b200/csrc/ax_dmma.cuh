// ax_dmma.cuh -- N = 7 Ax / K1 with the r- and s-direction contractions on the
// FP64 tensor cores (mma.sync m8n8k4 f64, DMMA; tcgen05 has no f64 kind).
//
// Why: the CUDA-core kernel (ax_tma.cuh) is latency-bound at 6 warps per SM
// (ncu r01l: issue active 23%, ~1000 instructions per warp per element, 8-long
// dependent FMA chains).  A DMMA does 256 FMAs per warp instruction at the
// same FP64 peak (tools/micro/dmma_rate.cu: 37.2 vs 34.2 TFLOP/s), so the
// contractions that are genuine 8x8 x 8x8 matrix products move to it:
//   k-slice tile (fixed k), C[j][i]:
//     u_r = P_k  D^T      (A = P_k[j][m] from smem,  B[m][i] = D[i][m])
//     u_s = D    P_k      (A = D[j][m],              B = P_k[m][i] from smem)
//     w  += F_rk D        (A = F_r,k[j][m] from smem, B[m][i] = D[m][i])
//     w  += D^T F_sk      (A[j][m] = D[m][j],         B = F_s,k[m][i] from smem)
// The t-direction (a combination of whole slices) stays on FMAs with the
// lane's two columns loaded once per element.  All fragments of one tile map
// lane t to the nodes (i = 2(t%4) + {0,1}, j = t/4, k), so u_r, u_s, u_t meet
// G^ pointwise in registers and w_r + w_s accumulate in one fragment.
//
// Staging, pipeline, CG fusion, deferred reductions: as ax_tma_kernel
// (TMA bulk copies of r, p, x and G^ per element, double-buffered groups of
// 64 threads; here warp w of a group owns the k-slices 4w .. 4w+3).
#pragma once
#include "ax_tma.cuh"

namespace sem {

#ifndef SEM_PDL_LATE
#define SEM_PDL_LATE 1
#endif
constexpr bool PDL_LATE = SEM_PDL_LATE != 0;   // (only with SEM_PDL=1 launches)

#ifndef SEM_DMMA_W4_GROUPS
#define SEM_DMMA_W4_GROUPS 2
#endif

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Groups of W warps per element: warp w owns the k-slices (8/W) w ..
// (8/W)(w+1) - 1.  W = 2: three groups per SM (444 on 148 SMs: c3's 4096
// elements take 9.22 rounds, the last one 23% full); W = 4: two groups per
// SM (296: 13.84 rounds, the last one 84% full) with each element done in
// about half the time.  Stages: two per group, TMA-filled as ax_tma_kernel.
// PCZ (Jacobi PCG without a mass term): K1 stages r and dinv next to p, x and
// forms z = dinv r itself, so K2 need not store z at every copy (pcg_z_in_k1).
template <bool CG, int W, bool PCZ = false>
struct DmmaLayout {
    using C = TmaCfg<7>;
    static constexpr int GT = 32 * W;
    static constexpr int NV = CG ? (PCZ ? 4 : 3) : 1;           // r,p,x[,dinv] | u
    static constexpr int STAGE = NV * C::VL + 6 * C::n3;        // doubles
    static constexpr int SMEM_MAX = 227 * 1024 - 1024;
    static constexpr int NG_FIT = SMEM_MAX / (2 * STAGE * 8);
    static constexpr int NG_CAP = W == 2 ? 4 : SEM_DMMA_W4_GROUPS;   // W=4: 2 (3 measured slower, r02)
    static constexpr int NG = NG_FIT > NG_CAP ? NG_CAP : NG_FIT;  // groups per CTA
    static constexpr int NT = NG * GT;
    static constexpr size_t SMEM = size_t(NG) * 2 * STAGE * 8 + 128;
};

// elements-per-group layout chosen at run time (SEM_DMMA_W=2|4, default 4)
inline int dmma_w() {
    static const int w = [] {
        const char *e = getenv("SEM_DMMA_W");
        return (e && e[0] == '2') ? 2 : 4;
    }();
    return w;
}

// MASS: + h u with h = alpha w J (screened Coulomb, the h pointer in the field
// the variant does not use, as ax_tma_kernel); PC: Jacobi PCG scalars; DOT:
// KA of the single-reduction CG (plain apply + (u, w) partials).
template <bool CG, bool MASS = false, bool PC = false, bool DOT = false, int W = 2>
__global__ void __launch_bounds__(DmmaLayout<CG, W, PC && !MASS>::NT, 1) ax_dmma_kernel(TmaArgs a) {
    constexpr int N = 7;
    using C = TmaCfg<N>;
    constexpr bool PCZ = PC && !MASS;     // z = dinv r formed here (a.r = r, a.u = dinv)
    using Lo = DmmaLayout<CG, W, PCZ>;
    constexpr int n = C::n, n2 = C::n2, n3 = C::n3, GT = Lo::GT, VL = C::VL;
    constexpr int NG = Lo::NG, NV = Lo::NV, STAGE = Lo::STAGE;
    constexpr int KW = n / W;                 // k-slices per warp
    constexpr int KC = n * 64 / GT;           // k-values per column owner in phase 0
    constexpr int DO = d_off(N);
    static_assert(C::EPG == 1 && n == 8 && (W == 2 || W == 4), "DMMA kernel: N = 7, one element per group");
    extern __shared__ __align__(128) double smem[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + size_t(NG) * 2 * STAGE);
    __shared__ double sred[4 * ((Lo::NT + 31) / 32)];

    const int tid = threadIdx.x;
    const int g = tid / GT;
    const int gt = tid - g * GT;
    const int i = gt % n, j = (gt / n) % n;  // phase-0 column owner (the CG update)
    const int kc0 = (gt / n2) * KC;          // ... of k = kc0 .. kc0 + KC - 1
    const int warp = gt >> 5, lane = gt & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int i0 = 2 * tig;                  // the lane's node pair (i0, i0+1) of row gid
    const bool leader = (gt == 0);
    double *stage0 = smem + size_t(g) * 2 * STAGE;
    uint64_t *gbar = bars + 2 * g;

    const int64_t nunits = a.E;
    const int64_t TG = int64_t(gridDim.x) * NG;
    // group-major: the extra elements of the last round land on different SMs
    const int64_t u0 = int64_t(g) * gridDim.x + blockIdx.x;
    const int64_t L = a.E * n3;

    if (leader) {
        mbar_init(gbar + 0, 1);
        mbar_init(gbar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if constexpr (CG && !PDL_LATE) pdl_trigger();

    const uint64_t pol_g = policy_evict_first();
    const uint64_t pol_v = CG ? policy_evict_last() : policy_evict_first();

    auto issue_G = [&](int64_t e, int s) {
        const VecRange vr = vec_range(e * n3, n3, L);
        const uint32_t vb = (uint32_t)((vr.a1 - vr.a0) * 8), gb = (uint32_t)(6 * n3 * 8);
        double *sb = stage0 + size_t(s) * STAGE;
        mbar_expect_tx_only(gbar + s, NV * vb + gb);
        bulk_g2s(sb + NV * VL, a.G + e * 6 * n3, gb, gbar + s, pol_g);
    };
    auto issue_V = [&](int64_t e, int s) {
        const int64_t first = e * n3;
        const VecRange vr = vec_range(first, n3, L);
        const uint32_t vb = (uint32_t)((vr.a1 - vr.a0) * 8);
        double *sb = stage0 + size_t(s) * STAGE;
        const double *vsrc[4];
        if constexpr (CG) {
            vsrc[0] = a.r;
            vsrc[1] = a.p;
            vsrc[2] = a.x;
            if constexpr (PCZ) vsrc[3] = a.u;
        } else {
            vsrc[0] = a.u;
        }
        for (int v = 0; v < NV; ++v)
            for (int64_t q = vr.a1; q < first + n3; ++q) sb[v * VL + (q - vr.a0)] = __ldg(vsrc[v] + q);
        mbar_arrive(gbar + s);
        for (int v = 0; v < NV; ++v) bulk_g2s(sb + v * VL, vsrc[v] + vr.a0, vb, gbar + s, pol_v);
    };

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
        if (blockIdx.x == 0 && tid == 0) a.st->k2 = kit;
    }
    double beta = 0.0, alpha_prev = 0.0;
    if constexpr (CG) {
        const CgStep c = cg_k1_finish<Lo::NT, PC>(a.st, a.red, sred, pre);
        if (c.done) {
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

    // the lane's D fragments (both k-steps): dA[ks] = D[gid][4ks+tig], dB[ks] = D[4ks+tig][gid]
    double dA[2], dB[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
        dA[ks] = c_D[DO + gid * n + 4 * ks + tig];
        dB[ks] = c_D[DO + (4 * ks + tig) * n + gid];
    }
    const int kb = KW * warp;                 // this warp's k-slices kb .. kb+KW-1
    const int lq = gid * n + i0;              // the lane's first node within a slice
    // f_r is stored with its column halves swapped on rows 2, 3, 6, 7 (i ^ 4),
    // so the phase-B A-fragment loads F_r,k[gid][4ks + tig] of a warp hit all
    // 16 bank pairs (2 wavefronts) instead of 8 (4 wavefronts)
    // (not with the mass term: measured 9% slower there, r01az)
    constexpr bool SWZ = !MASS;
    const int swz = SWZ ? (((gid >> 1) & 1) << 2) : 0;
    const int lqr = gid * n + (i0 ^ swz);

    double pap = 0.0;
    int t = 0;
    for (int64_t e = u0; e < nunits; e += TG, ++t) {
        const int s = t & 1;
        double *sb = stage0 + size_t(s) * STAGE;
        const int sh = (int)((e * n3) & 1);
        mbar_wait(gbar + s, (t >> 1) & 1);
        double *su;
        if constexpr (CG) {
            // phase 0 (thread = column owner): x += alpha_{k-1} p_{k-1}; p = r + beta p
            double *sr = sb + 0 * VL + sh;
            double *sp = sb + 1 * VL + sh;
            double *sx = sb + 2 * VL + sh;
            su = sp;
            const int64_t gbase = e * n3 + (gt % n2);
#pragma unroll
            for (int kk = 0; kk < KC; ++kk) {
                const int k = kc0 + kk;
                const int q = k * n2 + (gt % n2);
                const double rl = PCZ ? sb[3 * VL + sh + q] * sr[q] : sr[q];   // z = dinv r
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
            }
            group_bar(1 + g, GT);
        } else {
            su = sb + sh;
        }
        double *sG = sb + NV * VL;
        (void)i;
        (void)j;

        // the lane's two columns (all m) of the input: the t-direction operand
        double c0v[n], c1v[n];
#pragma unroll
        for (int m = 0; m < n; ++m) {
            c0v[m] = su[m * n2 + lq];
            c1v[m] = su[m * n2 + lq + 1];
        }

        // ---- phase A: gradient (DMMA for r, s; FMA for t) and G^ ----
#pragma unroll
        for (int kt = 0; kt < KW; ++kt) {
            const int k = kb + kt;
            const double *uk = su + k * n2;
            double r0 = 0.0, r1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                dmma(r0, r1, uk[gid * n + 4 * ks + tig], dA[ks]);    // u_r = P_k D^T
                dmma(s0, s1, dA[ks], uk[(4 * ks + tig) * n + gid]);  // u_s = D P_k
            }
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                const double d = c_D[DO + k * n + m];
                t0 = fma(d, c0v[m], t0);
                t1 = fma(d, c1v[m], t1);
            }
            const int q = k * n2 + lq;
            double *G0 = sG + q;
            const double2 g0 = *reinterpret_cast<const double2 *>(G0 + 0 * n3);
            const double2 g1 = *reinterpret_cast<const double2 *>(G0 + 1 * n3);
            const double2 g2 = *reinterpret_cast<const double2 *>(G0 + 2 * n3);
            const double2 g3 = *reinterpret_cast<const double2 *>(G0 + 3 * n3);
            const double2 g4 = *reinterpret_cast<const double2 *>(G0 + 4 * n3);
            const double2 g5 = *reinterpret_cast<const double2 *>(G0 + 5 * n3);
            if constexpr (SWZ) __syncwarp();   // the slice's G^_0 pairs are read before the swizzled f_r lands
            *reinterpret_cast<double2 *>(sG + k * n2 + lqr) =
                make_double2(g0.x * r0 + g1.x * s0 + g2.x * t0, g0.y * r1 + g1.y * s1 + g2.y * t1);
            *reinterpret_cast<double2 *>(G0 + 1 * n3) =
                make_double2(g1.x * r0 + g3.x * s0 + g4.x * t0, g1.y * r1 + g3.y * s1 + g4.y * t1);
            *reinterpret_cast<double2 *>(G0 + 2 * n3) =
                make_double2(g2.x * r0 + g4.x * s0 + g5.x * t0, g2.y * r1 + g4.y * s1 + g5.y * t1);
        }
        group_bar(1 + g, GT);     // f_r, f_s, f_t of every slice in shared memory

        // ---- phase B: w = F_r D + D^T F_s (DMMA) + t-direction (FMA) ----
        double f0v[n], f1v[n];
#pragma unroll
        for (int m = 0; m < n; ++m) {
            f0v[m] = sG[2 * n3 + m * n2 + lq];
            f1v[m] = sG[2 * n3 + m * n2 + lq + 1];
        }
#pragma unroll
        for (int kt = 0; kt < KW; ++kt) {
            const int k = kb + kt;
            const double *frk = sG + 0 * n3 + k * n2;
            const double *fsk = sG + 1 * n3 + k * n2;
            double w0 = 0.0, w1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
                dmma(w0, w1, frk[gid * n + ((4 * ks + tig) ^ swz)], dB[ks]);   // F_r,k D
                dmma(w0, w1, dB[ks], fsk[(4 * ks + tig) * n + gid]); // D^T F_s,k
            }
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                const double d = c_D[DO + m * n + k];
                t0 = fma(d, f0v[m], t0);
                t1 = fma(d, f1v[m], t1);
            }
            w0 += t0;
            w1 += t1;
            const int q = k * n2 + lq;
            const double2 pv = *reinterpret_cast<const double2 *>(su + q);
            if constexpr (MASS) {
                const double2 hv = __ldg(reinterpret_cast<const double2 *>((CG ? a.u : a.r) + e * n3 + q));
                w0 = fma(hv.x, pv.x, w0);
                w1 = fma(hv.y, pv.y, w1);
            }
            *reinterpret_cast<double2 *>(a.w + e * n3 + q) = make_double2(w0, w1);
            if constexpr (CG || DOT) {
                pap = fma(w0, pv.x, pap);
                pap = fma(w1, pv.y, pap);
            }
        }
        fence_proxy_async();
        group_bar(1 + g, GT);     // stage s fully consumed
        if (leader && e + 2 * TG < nunits) {
            issue_G(e + 2 * TG, s);
            issue_V(e + 2 * TG, s);
        }
    }
    if constexpr (CG && PDL_LATE) pdl_trigger();   // dependents launch during the tail
    if constexpr (CG || DOT) {
        const double bs = block_sum<Lo::NT>(pap, sred);
        if (tid == 0) a.part1[(kit & 1) * a.red.s1 + blockIdx.x] = bs;
    }
}

// ---- launchers (instantiated by the translation unit of each variant) ----
template <bool CG, int W>
static int dmma_grid_w(int64_t E, int nsm) {
    const int64_t need = (E + DmmaLayout<CG, W>::NG - 1) / DmmaLayout<CG, W>::NG;
    return (int)(need < nsm ? (need < 1 ? 1 : need) : nsm);
}
template <bool CG>
static int dmma_grid(int64_t E, int nsm) {
    return dmma_w() == 4 ? dmma_grid_w<CG, 4>(E, nsm) : dmma_grid_w<CG, 2>(E, nsm);
}

template <bool CG, bool MASS, bool PC, bool DOT>
static cudaError_t dmma_attr() {
    constexpr bool PCZ = PC && !MASS;
    cudaError_t e = cudaFuncSetAttribute(ax_dmma_kernel<CG, MASS, PC, DOT, 2>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)DmmaLayout<CG, 2, PCZ>::SMEM);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(ax_dmma_kernel<CG, MASS, PC, DOT, 4>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)DmmaLayout<CG, 4, PCZ>::SMEM);
}

// plain apply (MASS: h in a.r)
template <bool MASS, bool DOT = false>
static cudaError_t launch_dmma_plain(const TmaArgs &a, int nsm, cudaStream_t s) {
    // small meshes (config c2: 512 elements): W = 2's three groups per SM need
    // fewer rounds than W = 4's two -- c2 Ax 8.2 vs 9.1 us (r02); the DOT
    // variant keeps dmma_w() (its grid is the partial count ka_blocks reads)
    static const bool w_env = getenv("SEM_DMMA_W") != nullptr;
    const bool w2 = DOT || w_env ? dmma_w() == 2 : a.E <= int64_t(4) * nsm;
    if (!w2)
        ax_dmma_kernel<false, MASS, false, DOT, 4>
            <<<dmma_grid_w<false, 4>(a.E, nsm), DmmaLayout<false, 4>::NT, DmmaLayout<false, 4>::SMEM, s>>>(a);
    else
        ax_dmma_kernel<false, MASS, false, DOT, 2>
            <<<dmma_grid_w<false, 2>(a.E, nsm), DmmaLayout<false, 2>::NT, DmmaLayout<false, 2>::SMEM, s>>>(a);
    return cudaGetLastError();
}

// K1 over the element range of a (cg_args)
template <bool MASS, bool PC>
static cudaError_t launch_dmma_cg(const TmaArgs &a, int nsm, cudaStream_t s) {
    // (the grid of the plain CG layout: it is the count of (p, A p) partials the
    // consumers sum, dmma_blocks; the persistent element loop covers any grid)
    constexpr bool PCZ = PC && !MASS;
    if (dmma_w() == 4)
        return launch_pdl(ax_dmma_kernel<true, MASS, PC, false, 4>, dmma_grid_w<true, 4>(a.E, nsm),
                          DmmaLayout<true, 4, PCZ>::NT, DmmaLayout<true, 4, PCZ>::SMEM, s, a);
    return launch_pdl(ax_dmma_kernel<true, MASS, PC, false, 2>, dmma_grid_w<true, 2>(a.E, nsm),
                      DmmaLayout<true, 2, PCZ>::NT, DmmaLayout<true, 2, PCZ>::SMEM, s, a);
}

}  // namespace sem
