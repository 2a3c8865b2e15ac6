// ax_dmmag.cuh -- the plain Ax apply for N = 8..14 with the r/s contractions on
// the FP64 tensor cores: the N = 7 recipe (ax_dmma.cuh) on n x n k-slices with
// 9 <= n <= 12, covered by a 2 x 2 grid of 8 x 8 DMMA tiles (nodes outside the
// slice masked) and ceil(n/4) k-steps of 4 (D fragments zero beyond n).
// Element-staged by TMA like ax_tma_kernel (P and G^ of one element per
// stage, double-buffered); a group of 8 warps works on one element: warp w owns
// tile (w & 3) of the k-slices of parity w >> 2.  The CUDA-core kernels at these
// orders are register/latency-bound (c4 fractions 0.68 / 0.70 / 0.44 / 0.43).
// SLICE: G^ in the slice-major layout [k][6][n^2] of the high-order kernel.
// DOT: the operator half of the split CG K1 at these orders (k1u_kernel does
// the x / p update first, sem_kernels.cu): w = A_L p plus per-CTA partials of
// (p, A_L p) into part1 at the iteration parity, a no-op after the stop.  The
// partial is accumulated in phase A as sum (D p)^T G^ (D p) = p^T D^T G^ D p
// (the same quantity as p . w, exactly, up to rounding), so p is not needed
// in phase B (its stage slot may hold the next element already).
#pragma once
#include "ax_tma.cuh"
#include "ax_dmma.cuh"

namespace sem {

#ifndef SEM_DMMAG_SWZ
#define SEM_DMMAG_SWZ 1
#endif

template <int N>
struct DgCfg {
    static constexpr int n = N + 1, n2 = n * n, n3 = n2 * n;
    static constexpr int KS = (n + 3) / 4;                  // k-steps of the contractions
    static constexpr int VL = ((n3 + 2 + 1) / 2) * 2;      // vector slot (doubles, even)
    static constexpr int STAGE = VL + 6 * n3;              // u + G^ of one element
    static constexpr int SMEM_MAX = 227 * 1024 - 1024;
    // two double-buffered groups while they fit (n <= 10), else single-stage
    // groups (two while they fit, n <= 12) whose next element's copies are
    // split around phase B (SPLIT below)
    static constexpr int NS = (4 * STAGE * 8 <= SMEM_MAX) ? 2 : 1;
    static constexpr int NG_FIT = SMEM_MAX / (NS * STAGE * 8);
    static constexpr int NG = NG_FIT > 2 ? 2 : NG_FIT;      // groups of 8 warps per CTA
    static constexpr int GT = 256;
    static constexpr int NT = NG * GT;
    static constexpr size_t SMEM = size_t(NG) * NS * STAGE * 8 + 128;
    static_assert(n >= 9 && n <= 16 && NG >= 1, "2 x 2 tiles of 8, one element per stage");
};

template <int N, bool SLICE, bool DOT = false>
__global__ void __launch_bounds__(DgCfg<N>::NT, 1) ax_dmmag_kernel(TmaArgs a) {
    using C = DgCfg<N>;
    constexpr int n = C::n, n2 = C::n2, n3 = C::n3, KS = C::KS, VL = C::VL, STAGE = C::STAGE;
    constexpr int NG = C::NG, GT = C::GT, NS = C::NS;
    constexpr int DO = d_off(N);
    // even n: a lane's node pair (i0, i0 + 1) is one 16-byte-aligned double2 in
    // every staged array (n^2, n^3, VL even, shift 0) -- one conflict-free
    // 128-bit access instead of two 4-way-conflicted 64-bit ones (ncu r01aw)
    constexpr bool VEC = (n % 2) == 0;
    // n = 16: rows of 128 bytes put a quarter-warp's node pairs (rows j, j+1)
    // and the DMMA fragments' rows on the same banks (ncu r02hi_n15: 64% of the
    // shared wavefronts were conflict excess, L1 82% busy).  Each staged row
    // (u and G^, row index j within its slice) is permuted in place once per
    // element: 16-byte chunk c -> c ^ sigma(j), sigma(j) = (j & 1) << 2 |
    // (j >> 1) & 3 -- node pairs, A- and B-fragment loads all conflict-free /
    // two wavefronts.  Element (row j, column c) then lives at column
    // c ^ 2 sigma(j) (sc below).
    constexpr bool SWZ = (n == 16) && SEM_DMMAG_SWZ;
    extern __shared__ __align__(128) double smem[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + size_t(NG) * NS * STAGE);

    const int tid = threadIdx.x;
    const int g = tid / GT;
    const int gt = tid - g * GT;
    const int warp = gt >> 5, lane = gt & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int tp = warp & 3, hpar = warp >> 2;
    const int jt = tp >> 1, it = tp & 1;
    const int j = jt * 8 + gid;                 // the lane's node row
    const int i0 = it * 8 + 2 * tig;            // and its node pair (i0, i0+1)
    const bool vj = j < n, v0 = vj && i0 < n, v1 = vj && i0 + 1 < n;
    const bool leader = (gt == 0);
    double *stage0 = smem + size_t(g) * NS * STAGE;
    uint64_t *gbar = bars + 2 * g;

    const int64_t nunits = a.E;
    const int64_t TG = int64_t(gridDim.x) * NG;
    const int64_t u0 = int64_t(blockIdx.x) * NG + g;
    const int64_t L = a.E * n3;

    if (leader) {
        mbar_init(gbar + 0, 1);
        mbar_init(gbar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t pol = policy_evict_first();
    auto issue = [&](int64_t e, int s) {
        const int64_t first = e * n3;
        const VecRange vr = vec_range(first, n3, L);
        const uint32_t vb = (uint32_t)((vr.a1 - vr.a0) * 8), gb = (uint32_t)(6 * n3 * 8);
        double *sb = stage0 + size_t(s) * STAGE;
        mbar_expect_tx_only(gbar + s, vb + gb);
        bulk_g2s(sb + VL, a.G + e * 6 * n3, gb, gbar + s, pol);
        for (int64_t q = vr.a1; q < first + n3; ++q) sb[q - vr.a0] = __ldg(a.u + q);
        mbar_arrive(gbar + s);
        bulk_g2s(sb, a.u + vr.a0, vb, gbar + s, pol);
    };
    // One stage, slice-major G^: the next element's copies in two halves --
    // u and the factors 3..5 of every slice (not read after phase A) as soon
    // as phase A is done, the factors 0..2 (f_r, f_s, f_t during phase B)
    // after phase B -- so half the load overlaps phase B.  Bulk copies need
    // 16-byte sizes and addresses: for odd n^2 the second half starts one
    // double late (3 n^2 - 1 doubles) and the first takes that double along
    // (3 n^2 + 1; it is factor 3 of node 0, not read in phase B).
    // element-major G^: one copy per half, [3n^3 + HO3, 6n^3) and [0, 3n^3 + HO3)
    constexpr bool SPLIT = NS == 1;
    constexpr int HO = n2 & 1;                  // 0 (even n) or 1 (odd n)
    constexpr int HO3 = n3 & 1;
    auto issue_a = [&](int64_t e) {
        const int64_t first = e * n3;
        const VecRange vr = vec_range(first, n3, L);
        const uint32_t vb = (uint32_t)((vr.a1 - vr.a0) * 8);
        const uint32_t hb = (uint32_t)((3 * n2 - HO) * 8);
        double *sb = stage0;
        mbar_expect_tx_only(gbar, vb + (uint32_t)(6 * n3 * 8));
        for (int64_t q = vr.a1; q < first + n3; ++q) sb[q - vr.a0] = __ldg(a.u + q);
        mbar_arrive(gbar);
        bulk_g2s(sb, a.u + vr.a0, vb, gbar, pol);
        if constexpr (SLICE) {
            for (int k = 0; k < n; ++k) {
                const int o = k * 6 * n2 + 3 * n2 + HO;
                bulk_g2s(sb + VL + o, a.G + e * 6 * n3 + o, hb, gbar, pol);
            }
        } else {
            const int o = 3 * n3 + HO3;
            bulk_g2s(sb + VL + o, a.G + e * 6 * n3 + o, (uint32_t)((3 * n3 - HO3) * 8), gbar, pol);
        }
    };
    auto issue_b = [&](int64_t e) {
        if constexpr (SLICE) {
            const uint32_t hb = (uint32_t)((3 * n2 + HO) * 8);
            for (int k = 0; k < n; ++k)
                bulk_g2s(stage0 + VL + k * 6 * n2, a.G + e * 6 * n3 + k * 6 * n2, hb, gbar, pol);
        } else {
            bulk_g2s(stage0 + VL, a.G + e * 6 * n3, (uint32_t)((3 * n3 + HO3) * 8), gbar, pol);
        }
    };
    if (leader) {
        if (u0 < nunits) issue(u0, 0);
        if (NS == 2 && u0 + TG < nunits) issue(u0 + TG, 1);
    }
    int kit = 0;
    if constexpr (DOT) {
        __shared__ int done_s;
        if (tid == 0) {
            done_s = ld_state(&a.st->done);
            kit = ld_state(&a.st->k1);
        }
        __syncthreads();
        if (done_s) {       // after the stop: drain the issued copies, no work
            if (leader) {
                if (u0 < nunits) mbar_wait(gbar + 0, 0);
                if (NS == 2 && u0 + TG < nunits) mbar_wait(gbar + 1, 0);
            }
            return;
        }
    }
    double pap = 0.0;

    // D fragments: B of u_r = D[i][m], A of u_s = D[j][m], B of w_r = D[m][i],
    // A of w_s = D[m][j]; rows / columns beyond n are zero
    double urB[KS], usA[KS], wrB[KS], wsA[KS];
    const int ib = it * 8 + gid, jb = jt * 8 + gid;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
        const int m = 4 * ks + tig;
        urB[ks] = (ib < n && m < n) ? c_D[DO + ib * n + m] : 0.0;
        usA[ks] = (jb < n && m < n) ? c_D[DO + jb * n + m] : 0.0;
        wrB[ks] = (ib < n && m < n) ? c_D[DO + m * n + ib] : 0.0;
        wsA[ks] = (jb < n && m < n) ? c_D[DO + m * n + jb] : 0.0;
    }
    // G^ factor f of node (k, jj, ii) within the staged element
    auto sc = [&](int jj, int ii) -> int {
        return SWZ ? ii ^ ((((jj & 1) << 2) | ((jj >> 1) & 3)) << 1) : ii;
    };
    auto gidx = [&](int f, int k, int jj, int ii) -> int {
        return SLICE ? k * 6 * n2 + f * n2 + jj * n + sc(jj, ii) : f * n3 + k * n2 + jj * n + sc(jj, ii);
    };

    int t = 0;
    for (int64_t e = u0; e < nunits; e += TG, ++t) {
        const int s = NS == 2 ? (t & 1) : 0;
        double *sb = stage0 + size_t(s) * STAGE;
        const int sh = (int)((e * n3) & 1);
        mbar_wait(gbar + s, NS == 2 ? (t >> 1) & 1 : t & 1);
        const double *su = sb + sh;
        double *sG = sb + VL;
        if constexpr (SWZ) {
            // in-place row permutation of u (n^2 rows) and G^ (6 n^2 rows):
            // lane = (row r = 4 warp' + lane / 8 of the step, chunk lane % 8)
            constexpr int ROWS = n2 + 6 * n2;
            const int c = lane & 7;
            for (int r = warp * 4 + (lane >> 3); r < ROWS; r += (GT / 32) * 4) {
                double *row = (r < n2) ? (sb + sh) + r * n : sG + (r - n2) * n;
                const int jj = (r < n2 ? r : r - n2) & (n - 1);
                const double2 v = *reinterpret_cast<const double2 *>(row + 2 * c);
                __syncwarp();
                *reinterpret_cast<double2 *>(row + 2 * (c ^ (((jj & 1) << 2) | ((jj >> 1) & 3)))) = v;
            }
            group_bar(1 + g, GT);
        }

        double c0v[n], c1v[n];                  // the lane's two input columns
#pragma unroll
        for (int m = 0; m < n; ++m) {
            if constexpr (VEC) {                // even n: node pairs are 16-byte aligned
                const double2 c = v0 ? *reinterpret_cast<const double2 *>(su + m * n2 + j * n + sc(j, i0))
                                     : make_double2(0.0, 0.0);
                c0v[m] = c.x;
                c1v[m] = c.y;
            } else {
                c0v[m] = v0 ? su[m * n2 + j * n + i0] : 0.0;
                c1v[m] = v1 ? su[m * n2 + j * n + i0 + 1] : 0.0;
            }
        }
        // ---- phase A on the warp's tile of its slices ----
        for (int k = hpar; k < n; k += 2) {
            const double *uk = su + k * n2;
            double r0 = 0.0, r1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int m = 4 * ks + tig;
                const double aa = (jb < n && m < n) ? uk[jb * n + sc(jb, m)] : 0.0;   // P_k[j][m]
                const double bb = (ib < n && m < n) ? uk[m * n + sc(m, ib)] : 0.0;   // P_k[m][i]
                dmma(r0, r1, aa, urB[ks]);
                dmma(s0, s1, usA[ks], bb);
            }
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                const double d = c_D[DO + k * n + m];
                t0 = fma(d, c0v[m], t0);
                t1 = fma(d, c1v[m], t1);
            }
            if constexpr (VEC) {
                if (v0) {
                    double2 g[6];
#pragma unroll
                    for (int f = 0; f < 6; ++f) g[f] = *reinterpret_cast<const double2 *>(sG + gidx(f, k, j, i0));
                    const double2 fr = make_double2(g[0].x * r0 + g[1].x * s0 + g[2].x * t0,
                                                    g[0].y * r1 + g[1].y * s1 + g[2].y * t1);
                    const double2 fs = make_double2(g[1].x * r0 + g[3].x * s0 + g[4].x * t0,
                                                    g[1].y * r1 + g[3].y * s1 + g[4].y * t1);
                    const double2 ft = make_double2(g[2].x * r0 + g[4].x * s0 + g[5].x * t0,
                                                    g[2].y * r1 + g[4].y * s1 + g[5].y * t1);
                    *reinterpret_cast<double2 *>(sG + gidx(0, k, j, i0)) = fr;
                    *reinterpret_cast<double2 *>(sG + gidx(1, k, j, i0)) = fs;
                    *reinterpret_cast<double2 *>(sG + gidx(2, k, j, i0)) = ft;
                    if constexpr (DOT) {   // p^T A p = (D p)^T G^ (D p), node by node (pairs valid: n even)
                        pap = fma(r0, fr.x, fma(s0, fs.x, fma(t0, ft.x, pap)));
                        pap = fma(r1, fr.y, fma(s1, fs.y, fma(t1, ft.y, pap)));
                    }
                }
                continue;
            }
            if (v0) {
                const double g0 = sG[gidx(0, k, j, i0)], g1 = sG[gidx(1, k, j, i0)];
                const double g2 = sG[gidx(2, k, j, i0)], g3 = sG[gidx(3, k, j, i0)];
                const double g4 = sG[gidx(4, k, j, i0)], g5 = sG[gidx(5, k, j, i0)];
                const double fr = g0 * r0 + g1 * s0 + g2 * t0;
                const double fs = g1 * r0 + g3 * s0 + g4 * t0;
                const double ft = g2 * r0 + g4 * s0 + g5 * t0;
                sG[gidx(0, k, j, i0)] = fr;
                sG[gidx(1, k, j, i0)] = fs;
                sG[gidx(2, k, j, i0)] = ft;
                if constexpr (DOT) pap = fma(r0, fr, fma(s0, fs, fma(t0, ft, pap)));
            }
            if (v1) {
                const double g0 = sG[gidx(0, k, j, i0 + 1)], g1 = sG[gidx(1, k, j, i0 + 1)];
                const double g2 = sG[gidx(2, k, j, i0 + 1)], g3 = sG[gidx(3, k, j, i0 + 1)];
                const double g4 = sG[gidx(4, k, j, i0 + 1)], g5 = sG[gidx(5, k, j, i0 + 1)];
                const double fr = g0 * r1 + g1 * s1 + g2 * t1;
                const double fs = g1 * r1 + g3 * s1 + g4 * t1;
                const double ft = g2 * r1 + g4 * s1 + g5 * t1;
                sG[gidx(0, k, j, i0 + 1)] = fr;
                sG[gidx(1, k, j, i0 + 1)] = fs;
                sG[gidx(2, k, j, i0 + 1)] = ft;
                if constexpr (DOT) pap = fma(r1, fr, fma(s1, fs, fma(t1, ft, pap)));
            }
        }
        if constexpr (SPLIT) fence_proxy_async();   // generic reads of u, G^ 3..5 done
        group_bar(1 + g, GT);
        if constexpr (SPLIT) {
            if (leader && e + TG < nunits) issue_a(e + TG);
        }

        // ---- phase B ----
        double f0v[n], f1v[n];
#pragma unroll
        for (int m = 0; m < n; ++m) {
            if constexpr (VEC) {
                const double2 f = v0 ? *reinterpret_cast<const double2 *>(sG + gidx(2, m, j, i0))
                                     : make_double2(0.0, 0.0);
                f0v[m] = f.x;
                f1v[m] = f.y;
            } else {
                f0v[m] = v0 ? sG[gidx(2, m, j, i0)] : 0.0;
                f1v[m] = v1 ? sG[gidx(2, m, j, i0 + 1)] : 0.0;
            }
        }
        for (int k = hpar; k < n; k += 2) {
            double w0 = 0.0, w1 = 0.0;
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                const int m = 4 * ks + tig;
                const double aa = (jb < n && m < n) ? sG[gidx(0, k, jb, m)] : 0.0;   // F_r,k[j][m]
                const double bb = (ib < n && m < n) ? sG[gidx(1, k, m, ib)] : 0.0;   // F_s,k[m][i]
                dmma(w0, w1, aa, wrB[ks]);
                dmma(w0, w1, wsA[ks], bb);
            }
            double t0 = 0.0, t1 = 0.0;
#pragma unroll
            for (int m = 0; m < n; ++m) {
                const double d = c_D[DO + m * n + k];
                t0 = fma(d, f0v[m], t0);
                t1 = fma(d, f1v[m], t1);
            }
            double *wo = a.w + e * n3 + k * n2 + j * n + i0;
            if (v0) wo[0] = w0 + t0;
            if (v1) wo[1] = w1 + t1;

        }
        fence_proxy_async();
        group_bar(1 + g, GT);
        if constexpr (SPLIT) {
            if (leader && e + TG < nunits) issue_b(e + TG);
        } else {
            if (leader && e + NS * TG < nunits) issue(e + NS * TG, s);
        }
    }
    if constexpr (DOT) {
        __shared__ double sred[DgCfg<N>::NT / 32];
        const double bs = block_sum<DgCfg<N>::NT>(pap, sred);
        if (tid == 0) a.part1[(kit & 1) * a.red.s1 + blockIdx.x] = bs;
    }
}

template <int N>
static int dmmag_grid(int64_t E, int nsm) {
    const int64_t need = (E + DgCfg<N>::NG - 1) / DgCfg<N>::NG;
    return (int)(need < nsm ? (need < 1 ? 1 : need) : nsm);
}

}  // namespace sem
