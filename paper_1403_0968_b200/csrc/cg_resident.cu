// cg_resident.cu -- the whole CG solve at N = 7 as ONE persistent cooperative
// kernel with the solver state on chip (DESIGN.md §6 "Resident CG").  Opt-in
// (SEM_CG_RESIDENT=1): correct (tests/test_gpu_resident.py) but measured
// SLOWER than the two-kernel schedule at c3 (57.8 vs 44.0 us per iteration);
// kept as the record of the experiment and for its tests.
//
// The method is the CG of PAPER.md:667-673 on the SEM operator of
// eq:semOperator, computed as the two-kernel schedule
// (K1 = ax_dmma_kernel<CG>, K2 = k2_kernel) computes it: the same DMMA
// operator arithmetic, the same ascending-order DSSUM sums, the same
// x / p / r update expressions and stopping rule (cg_device.cuh cg_stop); only
// the association of the two global dot products differs (per-CTA partials
// of the CTA's own elements, summed in CTA order -- identical in every CTA).
//
// Idea: at c3 (4096 elements, 2.1 M local nodes) r, p and w fit on chip
// (TMEM 256 KB + shared memory 227 KB per SM), so an iteration would stream
// only the static G^ (48 B per node) instead of 96 + 21 B per node.
// Layout (one CTA per SM, 256 threads = 2 groups of 4 warps):
//   * CTA b owns the contiguous elements [b E / P, (b+1) E / P) (<= 28);
//     group g owns its local elements g, g + 2, ... (<= 14); a thread owns
//     the four nodes of its DMMA fragments in each of them;
//   * TMEM: thread gt of group g owns lane gt, columns [256 g, 256 g + 256):
//     element slot i holds r (8 columns) and w (8 columns) of its four nodes,
//     column 224 + i their metadata (m | pos << 4);
//   * shared memory: p of all the CTA's elements (28 x 4 KB) + two TMA stages
//     per group (G^ and the element's push targets);
//   * global: x (updated in place), the receive slots X and push targets of
//     the DSSUM exchange, two partial slots per CTA, a barrier counter.
// Per iteration k (group g, for each of its elements):
//     P:  x += alpha_{k-1} p_{k-1};  p = r + beta_k p  (p = r at k = 0)
//     A:  w_e = A_e p_e (DMMA r/s contractions, FMA t), (p, w) partial; own w
//         into TMEM; each surface value pushed (plain stores) into the
//         receive slots of the other copies of its node
//   grid barrier 1 -> pap_k, alpha_k = rho_k / pap_k
//     R:  the element's receive slots bulk-copied (TMA ring over both
//         stages); r -= alpha_k (own w + received, ascending order) at every
//         non-Dirichlet copy; (r, r) partial over the first copy of each node
//   grid barrier 2 -> rho_{k+1}, the stopping rule, beta_{k+1}
// Why it loses (ncu + phase clocks): with 8 warps per SM every
// latency is exposed -- the push stores cost ~10 us per iteration, the
// receive phase ~17 us, the CTA imbalance at the two barriers ~8 us; the
// operator phase alone (22 us) is close to the G^ HBM floor (15.7 us).
#include "ax_tma.cuh"
#include "ax_dmma.cuh"

namespace sem {

cudaError_t upload_const_D_rcg(int N, const double *D_host) { return upload_D_this_tu(N, D_host); }

namespace {

constexpr int kN = 7, kn = 8, kn2 = 64, kn3 = 512;
constexpr int kW = 4;                 // warps per group
constexpr int kNG = 2;                // groups per CTA
constexpr int kGT = 32 * kW;          // threads per group
constexpr int kNT = kNG * kGT;        // 256
constexpr int kEPG = 14;              // elements per group (TMEM: 16 columns each, 224 of 256)
constexpr int kEPC = kNG * kEPG;      // elements per CTA
constexpr int kGd = 6 * kn3;          // doubles: G^ of one element
constexpr int kStage = kGd + kRcgMaxSlots / 2;   // + the element's push targets (S int32)
constexpr int kRBars = 16;            // receive-slot mbarriers per group
constexpr size_t kSmem = size_t(kEPC) * kn3 * 8 + size_t(kNG) * 2 * kStage * 8 +
                         size_t(kNG) * (2 + kRBars) * 8;
static_assert(kSmem <= 227 * 1024, "resident CG: shared memory");
constexpr int kNodes = kn3 / kGT;     // nodes per thread and element (4)
static_assert(kNodes == 4, "thread <-> node map assumes 4 nodes per thread");

struct RcgArgs {
    int64_t E;
    int32_t S;                // receive slots per element
    const double *G;          // [E][6][512]
    double *x;                // [L] x_0 in, the solution out (updated in place)
    const double *r0;         // [L] r_0 (K2's start)
    const uint8_t *meta;      // [L] m | pos << 4 (m = 0: Dirichlet)
    const int32_t *sbq;       // [512] first receive slot of each node position
    const int32_t *push;      // [E][S] destinations of the pushed values (index into X)
    double *X;                // [E][S] receive slots
    const double *rho0_part;  // K2-start partials of rho_0 (nb2 values, fixed order)
    int nb2;
    double *part;             // [2][P]: (p, A p) and (r, r) partials of each CTA
    uint32_t *bar;            // grid barrier counter (zeroed before the launch)
    uint64_t *phase;          // [4] CTA 0's ns in P+A, barrier 1, R, barrier 2 (summed)
    CgState *st;
};

// ---- TMEM as per-thread storage (tcgen05.ld / st, 32x32b shape: lane = thread) ----
__device__ __forceinline__ void tm_ld16(uint32_t ta, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(ta));
}
__device__ __forceinline__ void tm_ld8(uint32_t ta, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(ta));
}
__device__ __forceinline__ void tm_st8(uint32_t ta, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ uint32_t tm_ld1(uint32_t ta) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(ta));
    return v;
}
__device__ __forceinline__ void tm_st1(uint32_t ta, uint32_t v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(ta), "r"(v) : "memory");
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ double u2d(uint32_t lo, uint32_t hi) {
    return __hiloint2double((int)hi, (int)lo);
}
__device__ __forceinline__ void d2u(double d, uint32_t &lo, uint32_t &hi) {
    lo = (uint32_t)__double2loint(d);
    hi = (uint32_t)__double2hiint(d);
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
    return t;
}

// Grid-wide barrier over the co-resident CTAs (cooperative launch): arrive
// with a release add, spin with acquire loads.  A barrier that has not
// completed after 10 s sets the error word (a lost CTA: never expected under
// a cooperative launch) and lets every CTA leave.
__device__ __forceinline__ bool grid_sync(uint32_t *ctr, uint32_t target, CgState *st) {
    __shared__ int s_ok;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        int ok = 1;
        uint32_t v;
        const uint64_t t0 = globaltimer();
        for (int spin = 0;; ++spin) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if ((int32_t)(v - target) >= 0) break;
            if ((spin & 1023) == 1023 && globaltimer() - t0 > 10000000000ull) {
                atomicExch(&st->rcg_err, 1);
                ok = 0;
                break;
            }
        }
        if (ok && ld_state(&st->rcg_err)) ok = 0;
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        s_ok = ok;
    }
    __syncthreads();
    return s_ok != 0;
}

// ordered sum of cnt <= kNT values (one per thread, fixed tree): the same in
// every CTA
__device__ __forceinline__ double sum_slots(const double *src, int cnt, double *red) {
    double v = 0.0;
    for (int t = threadIdx.x; t < cnt; t += kNT) v += __ldcg(src + t);
    return block_sum<kNT>(v, red);
}

__global__ void __launch_bounds__(kNT, 1) rcg_kernel(const __grid_constant__ RcgArgs a) {
    constexpr int DO = d_off(kN);
    constexpr int KW = kn / kW;            // k-slices per warp (2)
    extern __shared__ __align__(128) double smem[];
    double *sp = smem;                                          // [kEPC][512] p
    double *stg = smem + size_t(kEPC) * kn3;                   // [kNG][2][kStage]
    uint64_t *bars = reinterpret_cast<uint64_t *>(stg + size_t(kNG) * 2 * kStage);
    __shared__ double sred[4 * (kNT / 32)];
    __shared__ uint32_t s_tbase;

    const int tid = threadIdx.x;
    const int g = tid / kGT, gt = tid - g * kGT;
    const int warp = gt >> 5, lane = gt & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const int i0 = 2 * tig;
    const bool leader = (gt == 0);
    const int P = gridDim.x, b = blockIdx.x;
    const int64_t e_lo = int64_t(b) * a.E / P, e_hi = int64_t(b + 1) * a.E / P;
    const int ne = (int)(e_hi - e_lo);
    const int neg = ne > g ? (ne - g + 1) / 2 : 0;             // elements of this group
    const int S = a.S;
    // receive ring of R: the group's two stages, S doubles per slot
    const int nslot = min(kRBars, (2 * kStage) / max(S, 2));
    uint64_t *gbar = bars + (2 + kRBars) * g;  // [0,1]: G^ stages, [2, 2 + nslot): receive slots
    double *stage0 = stg + size_t(g) * 2 * kStage;

    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (leader) {
        for (int q = 0; q < 2 + kRBars; ++q) mbar_init(gbar + q, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // this thread's lane (quarter = warp % 4 of the group) and column half
    const uint32_t tb = s_tbase + ((uint32_t)(32 * warp) << 16) + (uint32_t)(256 * g);

    // the thread's four nodes (the DMMA fragment layout): slices kk = 2 warp +
    // (u >> 1), row gid, columns i0 + (u & 1)
    int qn[kNodes], sb[kNodes];
#pragma unroll
    for (int u = 0; u < kNodes; ++u) {
        qn[u] = (KW * warp + (u >> 1)) * kn2 + gid * kn + i0 + (u & 1);
        sb[u] = __ldg(a.sbq + qn[u]);
    }

    const uint64_t pol_g = policy_evict_first();
    const uint64_t pol_v = policy_evict_last();
    // G^ and the push targets of the group's t-th element in the cyclic stream
    int tissue = 0;                          // next stream position to issue (leader)
    const uint32_t gbytes = (uint32_t)(kGd * 8), pbytes = (uint32_t)(S * 4 + 15) & ~15u;
    auto issue_G = [&]() {
        const int t = tissue++;
        const int64_t e = e_lo + g + 2 * (t % neg);
        const int s = t & 1;
        double *dst = stage0 + size_t(s) * kStage;
        mbar_expect_tx(gbar + s, gbytes + pbytes);
        bulk_g2s(dst, a.G + e * 6 * kn3, gbytes, gbar + s, pol_g);
        bulk_g2s(dst + kGd, a.push + e * S, pbytes, gbar + s, pol_v);
    };
    if (leader && neg > 0) {
        issue_G();
        if (neg > 1) issue_G();
    }

    // r_0 and the node metadata of the group's elements into TMEM
    for (int i = 0; i < neg; ++i) {
        const int64_t base = (e_lo + g + 2 * i) * kn3;
        uint32_t v[8];
        uint32_t mt = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const double2 rv = __ldcg(reinterpret_cast<const double2 *>(a.r0 + base + qn[2 * h]));
            d2u(rv.x, v[4 * h + 0], v[4 * h + 1]);
            d2u(rv.y, v[4 * h + 2], v[4 * h + 3]);
            mt |= (uint32_t)__ldg(a.meta + base + qn[2 * h]) << (16 * h);
            mt |= (uint32_t)__ldg(a.meta + base + qn[2 * h] + 1) << (16 * h + 8);
        }
        tm_st8(tb + 16 * i, v);
        tm_st1(tb + 224 + i, mt);
    }
    tm_wait_st();

    const int maxit = a.st->maxit;
    const double tol = a.st->tol;
    const double rho0 = sum_slots(a.rho0_part, a.nb2, sred);
    double rho = rho0, rho_prev = 0.0, alpha_prev = 0.0;
    int k = 0;
    uint32_t nbar = 0;
    int t = 0;                               // stream position of the next element consumed
    int trb = 0;                             // receive copies of earlier iterations
    bool ok = true;

    // the lane's D fragments: dA[ks] = D[gid][4ks+tig], dB[ks] = D[4ks+tig][gid]
    double dA[2], dB[2];
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
        dA[ks] = c_D[DO + gid * kn + 4 * ks + tig];
        dB[ks] = c_D[DO + (4 * ks + tig) * kn + gid];
    }
    const int kb = KW * warp;
    const int lq = gid * kn + i0;
    const int swz = ((gid >> 1) & 1) << 2;   // f_r column-half swizzle (ax_dmma.cuh)
    const int lqr = gid * kn + (i0 ^ swz);

    // CTA 0's phase clock (one thread): ns spent in P+A, barrier 1, R, barrier 2
    uint64_t ph[4] = {0, 0, 0, 0}, tph = globaltimer();
    auto lap = [&](int q) {
        if (b == 0 && tid == 0) {
            const uint64_t now = globaltimer();
            ph[q] += now - tph;
            tph = now;
        }
    };
    // receive copy c (= trb + i: the group's element i of this iteration) into
    // ring slot c % nslot
    const uint32_t xbytes = (uint32_t)(S * 8);
    auto issue_R = [&](int i) {
        const int c = trb + i, sl = c % nslot;
        mbar_expect_tx(gbar + 2 + sl, xbytes);
        bulk_g2s(stage0 + size_t(sl) * S, a.X + (e_lo + g + 2 * i) * S, xbytes, gbar + 2 + sl, pol_v);
    };

    while (true) {
        if (cg_stop(k, rho, rho0, maxit, tol)) break;
        const double beta = (k == 0) ? 0.0 : rho / rho_prev;
        double pap = 0.0;
        for (int i = 0; i < neg; ++i, ++t) {
            const int el = g + 2 * i;
            const int64_t e = e_lo + el;
            const int s = t & 1;
            double *pe = sp + size_t(el) * kn3;
            double *sG = stage0 + size_t(s) * kStage;
            const int32_t *sdst = reinterpret_cast<const int32_t *>(sG + kGd);
            // ---- P: x += alpha_{k-1} p_{k-1} (loads now, stores after B);
            //      p = r + beta p (p = r at k = 0) ----
            uint32_t mt;
            double2 xo[2], po[2];
            {
                uint32_t v[8];
                tm_ld8(tb + 16 * i, v);
                mt = tm_ld1(tb + 224 + i);
                if (k > 0) {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        xo[h] = __ldcg(reinterpret_cast<const double2 *>(a.x + e * kn3 + qn[2 * h]));
                }
                tm_wait_ld();
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    double2 *pp = reinterpret_cast<double2 *>(pe + qn[2 * h]);
                    const double r0 = u2d(v[4 * h + 0], v[4 * h + 1]);
                    const double r1 = u2d(v[4 * h + 2], v[4 * h + 3]);
                    if (k == 0) {
                        *pp = make_double2(r0, r1);
                    } else {
                        po[h] = *pp;
                        *pp = make_double2(r0 + beta * po[h].x, r1 + beta * po[h].y);
                    }
                }
            }
            group_bar(1 + g, kGT);
            mbar_wait(gbar + s, (t >> 1) & 1);
            const double *su = pe;

            // the lane's two columns (all m) of p: the t-direction operand
            double c0v[kn], c1v[kn];
#pragma unroll
            for (int m = 0; m < kn; ++m) {
                c0v[m] = su[m * kn2 + lq];
                c1v[m] = su[m * kn2 + lq + 1];
            }
            // ---- phase A: gradient (DMMA r, s; FMA t) and G^ ----
#pragma unroll
            for (int kt = 0; kt < KW; ++kt) {
                const int kk = kb + kt;
                const double *uk = su + kk * kn2;
                double r0 = 0.0, r1 = 0.0, s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    dmma(r0, r1, uk[gid * kn + 4 * ks + tig], dA[ks]);
                    dmma(s0, s1, dA[ks], uk[(4 * ks + tig) * kn + gid]);
                }
                double t0v = 0.0, t1v = 0.0;
#pragma unroll
                for (int m = 0; m < kn; ++m) {
                    const double d = c_D[DO + kk * kn + m];
                    t0v = fma(d, c0v[m], t0v);
                    t1v = fma(d, c1v[m], t1v);
                }
                const int q = kk * kn2 + lq;
                double *G0 = sG + q;
                const double2 g0 = *reinterpret_cast<const double2 *>(G0 + 0 * kn3);
                const double2 g1 = *reinterpret_cast<const double2 *>(G0 + 1 * kn3);
                const double2 g2 = *reinterpret_cast<const double2 *>(G0 + 2 * kn3);
                const double2 g3 = *reinterpret_cast<const double2 *>(G0 + 3 * kn3);
                const double2 g4 = *reinterpret_cast<const double2 *>(G0 + 4 * kn3);
                const double2 g5 = *reinterpret_cast<const double2 *>(G0 + 5 * kn3);
                __syncwarp();
                *reinterpret_cast<double2 *>(sG + kk * kn2 + lqr) =
                    make_double2(g0.x * r0 + g1.x * s0 + g2.x * t0v, g0.y * r1 + g1.y * s1 + g2.y * t1v);
                *reinterpret_cast<double2 *>(G0 + 1 * kn3) =
                    make_double2(g1.x * r0 + g3.x * s0 + g4.x * t0v, g1.y * r1 + g3.y * s1 + g4.y * t1v);
                *reinterpret_cast<double2 *>(G0 + 2 * kn3) =
                    make_double2(g2.x * r0 + g4.x * s0 + g5.x * t0v, g2.y * r1 + g4.y * s1 + g5.y * t1v);
            }
            group_bar(1 + g, kGT);
            // ---- phase B: w = F_r D + D^T F_s (DMMA) + t-direction (FMA) ----
            double f0v[kn], f1v[kn];
#pragma unroll
            for (int m = 0; m < kn; ++m) {
                f0v[m] = sG[2 * kn3 + m * kn2 + lq];
                f1v[m] = sG[2 * kn3 + m * kn2 + lq + 1];
            }
            uint32_t wv[8];
#pragma unroll
            for (int kt = 0; kt < KW; ++kt) {
                const int kk = kb + kt;
                const double *frk = sG + 0 * kn3 + kk * kn2;
                const double *fsk = sG + 1 * kn3 + kk * kn2;
                double w0 = 0.0, w1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    dmma(w0, w1, frk[gid * kn + ((4 * ks + tig) ^ swz)], dB[ks]);
                    dmma(w0, w1, dB[ks], fsk[(4 * ks + tig) * kn + gid]);
                }
                double t0v = 0.0, t1v = 0.0;
#pragma unroll
                for (int m = 0; m < kn; ++m) {
                    const double d = c_D[DO + m * kn + kk];
                    t0v = fma(d, f0v[m], t0v);
                    t1v = fma(d, f1v[m], t1v);
                }
                w0 += t0v;
                w1 += t1v;
                const int q = kk * kn2 + lq;
                const double2 pv = *reinterpret_cast<const double2 *>(su + q);
                pap = fma(w0, pv.x, pap);
                pap = fma(w1, pv.y, pap);
                // push the surface values into the other copies' receive slots
                const int u0 = 2 * kt;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = (mt >> (8 * (u0 + h))) & 15;
                    const double wq = h ? w1 : w0;
                    const int32_t *dq = sdst + sb[u0 + h];
                    if (m == 2) {                       // face node: one other copy
                        a.X[dq[0]] = wq;
                    } else if (m > 2) {                 // edge / vertex: all targets loaded first
                        int dd[kRcgMaxM - 1];
#pragma unroll
                        for (int q2 = 0; q2 < kRcgMaxM - 1; ++q2) dd[q2] = (q2 < m - 1) ? dq[q2] : 0;
#pragma unroll
                        for (int q2 = 0; q2 < kRcgMaxM - 1; ++q2)
                            if (q2 < m - 1) a.X[dd[q2]] = wq;
                    }
                }
                d2u(w0, wv[2 * u0 + 0], wv[2 * u0 + 1]);
                d2u(w1, wv[2 * u0 + 2], wv[2 * u0 + 3]);
            }
            tm_st8(tb + 16 * i + 8, wv);
            if (k > 0) {
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    *reinterpret_cast<double2 *>(a.x + e * kn3 + qn[2 * h]) =
                        make_double2(xo[h].x + alpha_prev * po[h].x, xo[h].y + alpha_prev * po[h].y);
            }
            fence_proxy_async();
            group_bar(1 + g, kGT);       // stage s consumed
            // the stream stops at the iteration's end: both stages serve the
            // receive ring of R, then the next iteration's first two elements
            if (leader && i + 2 < neg) issue_G();
        }

        // ---- barrier 1: pap_k -> alpha_k ----
        {
            const double bs = block_sum<kNT>(pap, sred);
            if (tid == 0) a.part[b] = bs;
        }
        lap(0);
        ++nbar;
        if (!(ok = grid_sync(a.bar, nbar * (uint32_t)P, a.st))) break;
        const double papk = sum_slots(a.part, P, sred);
        const double alpha = rho / papk;
        lap(1);

        // ---- R: r -= alpha Q Q^T w (own w + received copies, ascending);
        //      (r, r) over the first copies ----
        double rr = 0.0;
        if (neg > 0) {
            if (leader) {
                asm volatile("fence.proxy.async.global;" ::: "memory");
                for (int i = 0; i < min(neg, nslot); ++i) issue_R(i);
            }
            int sl = trb % nslot, use = trb / nslot;   // ring slot and its use count
            for (int i = 0; i < neg; ++i) {
                const double *Xs = stage0 + size_t(sl) * S;
                uint32_t v[16];
                tm_ld16(tb + 16 * i, v);
                const uint32_t mt = tm_ld1(tb + 224 + i);
                tm_wait_ld();
                mbar_wait(gbar + 2 + sl, use & 1);
#pragma unroll
                for (int u = 0; u < kNodes; ++u) {
                    const int m = (mt >> (8 * u)) & 15, pos = (mt >> (8 * u + 4)) & 15;
                    if (m == 0) continue;                  // Dirichlet: r stays 0
                    const double own = u2d(v[8 + 2 * u], v[8 + 2 * u + 1]);
                    const double *xq = Xs + sb[u];
                    double sum;
                    if (m == 1) {
                        sum = own;
                    } else if (m == 2) {
                        sum = own + xq[0];                 // (either order: a + b == b + a)
                    } else {                               // ascending, own at pos
                        double xv[kRcgMaxM - 1];
#pragma unroll
                        for (int q = 0; q < kRcgMaxM - 1; ++q) xv[q] = (q < m - 1) ? xq[q] : 0.0;
                        sum = (pos == 0) ? own : xv[0];
#pragma unroll
                        for (int q = 1; q < kRcgMaxM; ++q)
                            if (q < m) sum += (q == pos) ? own : (q < pos ? xv[q] : xv[q - 1]);
                    }
                    const double rn = u2d(v[2 * u], v[2 * u + 1]) - alpha * sum;
                    d2u(rn, v[2 * u], v[2 * u + 1]);
                    if (pos == 0) rr += rn * rn;
                }
                uint32_t rv8[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) rv8[q] = v[q];
                tm_st8(tb + 16 * i, rv8);
                if (i + nslot < neg) {
                    fence_proxy_async();
                    group_bar(1 + g, kGT);             // slot consumed
                    if (leader) issue_R(i + nslot);
                }
                if (++sl == nslot) {
                    sl = 0;
                    ++use;
                }
            }
            trb += neg;
            fence_proxy_async();
            group_bar(1 + g, kGT);                     // the ring is free again
            if (leader) {                              // the next iteration's first elements
                issue_G();
                if (neg > 1) issue_G();
            }
        }
        {
            const double bs = block_sum<kNT>(rr, sred);
            if (tid == 0) a.part[P + b] = bs;
        }
        lap(2);
        ++nbar;
        if (!(ok = grid_sync(a.bar, nbar * (uint32_t)P, a.st))) break;
        tm_wait_st();
        const double rho_next = sum_slots(a.part + P, P, sred);
        lap(3);
        rho_prev = rho;
        rho = rho_next;
        alpha_prev = alpha;
        ++k;
    }

    // x_it = x_{it-1} + alpha_{it-1} p_{it-1}
    if (ok && k > 0) {
        for (int i = 0; i < neg; ++i) {
            const int el = g + 2 * i;
            const int64_t e = e_lo + el;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double2 *xp = reinterpret_cast<double2 *>(a.x + e * kn3 + qn[2 * h]);
                const double2 xv = __ldcg(xp);
                const double2 pv = *reinterpret_cast<const double2 *>(sp + size_t(el) * kn3 + qn[2 * h]);
                *xp = make_double2(xv.x + alpha_prev * pv.x, xv.y + alpha_prev * pv.y);
            }
        }
    }
    if (ok && b == 0 && tid == 0) {
        CgState *st = a.st;
        st->rho0 = rho0;
        st->iters = k;
        st->rel_res = (rho0 == 0.0) ? 0.0 : sqrt(rho) / sqrt(rho0);
        st->converged = (rho0 == 0.0) || !(sqrt(rho) > tol * sqrt(rho0));
        st->alpha_km1 = alpha_prev;
        st->k1 = k;
        st->k2 = k;
        for (int q = 0; q < 4; ++q) a.phase[q] = ph[q];
        __threadfence();
        st->done = 1;
    }
    // drain the G^ copies still in flight before the CTA exits
    if (leader && neg > 0)
        for (int p = t; p < tissue; ++p) mbar_wait(gbar + (p & 1), (p >> 1) & 1);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(s_tbase));
}

}  // namespace

bool rcg_supported(const DevMesh &m) {
    return m.N == kN && m.nranks == 1 && !m.H && m.use_dmma && m.E >= 1 &&
           m.E <= int64_t(kEPC) * m.nsm;
}

int rcg_blocks(const DevMesh &m) {
    // enough CTAs that none holds more than kEPC elements; at most one per SM
    const int64_t need = (m.E + 1) / 2;            // >= 1 element per group where possible
    return (int)(need < m.nsm ? need : m.nsm);
}

cudaError_t rcg_prepare() {
    return cudaFuncSetAttribute(rcg_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
}

cudaError_t launch_rcg(const DevMesh &m, const CgVecs &v, const RcgBufs &rb, cudaStream_t s) {
    RcgArgs a{};
    a.E = m.E;
    a.S = rb.S;
    a.G = m.G;
    a.x = v.x;
    a.r0 = v.r;
    a.meta = rb.meta;
    a.sbq = rb.sbq;
    a.push = rb.push;
    a.X = rb.X;
    a.rho0_part = v.part2 + v.s2;          // K2's start writes rho_0's partials as "k = -1"
    a.nb2 = v.nb2;
    a.part = rb.part;
    a.bar = rb.bar;
    a.phase = reinterpret_cast<uint64_t *>(rb.bar + 16);
    a.st = v.st;
    const int P = rcg_blocks(m);
    if (int64_t(P) * kEPC < m.E || rb.S > kRcgMaxSlots || (rb.S & 3)) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaMemsetAsync(rb.bar, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    void *args[] = {(void *)&a};
    return cudaLaunchCooperativeKernel((const void *)rcg_kernel, dim3(P), dim3(kNT), args, kSmem, s);
}

}  // namespace sem
