// fd2d.cu -- the finite-difference wave-equation step of arXiv 1403.0968
// (Sec. "Finite Difference", lst:fdCode PAPER.md:418-449; SURVEY.md §8(f)
// NEXT-4) for sm_100a, behind include/fd.h.
//
// HBM-bound 2-D stencil (24 B per node: u1, u2 read, u3 written; the paper
// makes "no memory retrieval optimizations", this kernel is the
// Micikevicius-style design it points to at :395): a CTA owns a tile of
// kTW = 256 columns and marches down a strip of rows.  Rows of u1 (with an
// r-column halo, periodic wrap) and of u2 stream through shared-memory rings
// by cp.async, kP rows ahead; each thread owns two adjacent columns, keeps
// their 2r+1 u1 values of the column in registers (the y-neighbours) and
// reads the x-neighbours of the center row from shared memory as 16-byte
// pairs.  omega is a __grid_constant__ kernel parameter (uniform operands in
// the parameter bank; no process-wide __constant__ state, so concurrent calls
// with different weights on different streams cannot race).  The arithmetic
// is the listing's, operation by operation, with explicit round-to-nearest
// intrinsics (no FMA contraction), so every u3 is bit-identical to a plain C
// evaluation of lst:fdCode -- the default of fd2d_step / fd2d_run.  SYM
// (fd2d_run_ex with FD_REGROUPED; symmetric weights omega_{-k} = omega_k, as
// every central stencil has): the same sum regrouped by pairs,
//   lap = omega_0 (u + u) + sum_{k=1..r} omega_k ((u_{i-k} + u_{i+k}) + (u_{j-k} + u_{j+k}))
// with FMAs: 4r + 3 FP64 operations per node instead of 8r + 8 (the kernel is
// FP64-issue-bound at large r otherwise); equal to the listing up to rounding
// (reading R6c; tests bound the difference).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/fd.h"
#include "../../include/sem.h"

namespace sem_fd {

constexpr int kNT = 128;          // threads per CTA
constexpr int kTW = 2 * kNT;      // tile width (columns), two per thread
constexpr int kP = 4;             // rows in flight

struct Omega {
    double w[2 * FD_RMAX + 1];
};

template <int R>
struct FdCfg {
    static constexpr int LP = R + (R & 1);           // left halo, rounded up to even
    static constexpr int NB = R + kP + 1;            // ring rows: center .. newest in flight
    static constexpr int RW = kTW + 2 * LP;          // u1 row with halo (even: 16-byte rows)
    static constexpr int XO = LP - R;                // 0 or 1: window offset of u1(c - R)
    static constexpr size_t SMEM = size_t(NB) * (RW + kTW) * sizeof(double);
};

__device__ __forceinline__ void cp_async16(double *dst, const double *src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(double *dst, const double *src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// compile-time loop: f(std::integral_constant<int, i>) for i = 0 .. M-1
template <int I, int M, typename F>
__device__ __forceinline__ void static_for_impl(F &&f) {
    if constexpr (I < M) {
        f(std::integral_constant<int, I>{});
        static_for_impl<I + 1, M>(f);
    }
}
template <int M, typename F>
__device__ __forceinline__ void static_for(F &&f) { static_for_impl<0, M>(f); }

// Grid: x = tiles of kTW columns, y = strips of `ty` rows.
template <int R, bool SYM>
__global__ void __launch_bounds__(kNT, 3) fd2d_kernel(const double *__restrict__ u1,
                                                    const double *__restrict__ u2,
                                                    double *__restrict__ u3, int64_t w, int64_t h,
                                                    int ty, double dt2,
                                                    const __grid_constant__ Omega om_) {
    const double *c_omega = om_.w;
    using C = FdCfg<R>;
    constexpr int NB = C::NB, RW = C::RW, LP = C::LP, XO = C::XO;
    extern __shared__ __align__(16) double smem[];
    double *s1 = smem;                 // [NB][RW]  u1 rows, columns i0-LP .. i0+kTW+LP-1
    double *s2 = smem + NB * RW;       // [NB][kTW] u2 rows (center rows)

    const int tid = threadIdx.x;
    const int64_t i0 = int64_t(blockIdx.x) * kTW;
    const int64_t j0 = int64_t(blockIdx.y) * ty;
    const int64_t jend = (j0 + ty < h) ? j0 + ty : h;
    const int nl = int(jend - j0) + 2 * R;           // u1 rows j0-R .. jend+R-1
    // tiles away from the wrap-around with 16-byte aligned rows copy pairs
    const bool pairs = ((w & 1) == 0) && i0 >= LP && i0 + kTW + LP <= w;

    // issue the copies of pipeline row s: u1 row j0-R+s (wrapped), and u2 row
    // j0-2R+s (the center row when u1 row s arrives) if it is an output row
    auto issue = [&](int s) {
        if (s < nl) {
            const int slot = s % NB;
            int64_t y = j0 - R + s;
            y = (y < 0) ? y + h : (y >= h ? y - h : y);
            const double *row = u1 + y * w;
            double *d1 = s1 + slot * RW;
            const int64_t yc = j0 - 2 * R + s;
            if (pairs) {
                const double *src = row + (i0 - LP);
                for (int q = 2 * tid; q < RW; q += 2 * kNT) cp_async16(d1 + q, src + q);
                if (yc >= j0) cp_async16(s2 + slot * kTW + 2 * tid, u2 + yc * w + i0 + 2 * tid);
            } else {
                for (int q = tid; q < RW; q += kNT) {
                    int64_t x = i0 - LP + q;          // in [-LP, w + kTW + LP): wrap (w >= 2R+1)
                    if (x < 0) x += w;
                    while (x >= w) x -= w;
                    cp_async8(d1 + q, row + x);
                }
                if (yc >= j0) {
                    const double *row2 = u2 + yc * w;
                    for (int q = tid; q < kTW; q += kNT) {
                        const int64_t x = i0 + q;
                        if (x < w) cp_async8(s2 + slot * kTW + q, row2 + x);
                    }
                }
            }
        }
        cp_async_commit();   // (empty groups keep the wait count uniform)
    };

#pragma unroll
    for (int s = 0; s < kP; ++s) issue(s);

    const int c0 = 2 * tid;                       // this thread's columns c0, c0+1
    // register queues of the column values of rows s-2R .. s: row s lives in
    // slot s mod NQ; the row loop is unrolled by NQ so every slot index is a
    // compile-time constant (a rotating queue, no register moves)
    constexpr int NQ = 2 * R + 1;
    double q0[NQ], q1[NQ];
#pragma unroll
    for (int k = 0; k < NQ; ++k) q0[k] = q1[k] = 0.0;

    auto step = [&](const int s, auto uc) {
        constexpr int u = decltype(uc)::value;        // s mod NQ
        cp_async_wait<kP - 1>();
        __syncthreads();          // row s landed for all; step s-1's reads are done
        issue(s + kP);            // refills the slot of row s+kP-NB = s-R-1 (no longer read)
        const int slot = s % NB;
        const double2 nv = *reinterpret_cast<const double2 *>(s1 + slot * RW + LP + c0);
        q0[u] = nv.x;                                   // own columns of the new row
        q1[u] = nv.y;
        if (s < 2 * R) return;
        // center row s - R: x-neighbours from its smem row, u2 from the slot of row s
        const int64_t j = j0 + s - 2 * R;
        // window of the center row: xw[XO + R + k] = u1(c0 + k), 16-byte pairs
        const double *cr = s1 + ((s - R) % NB) * RW + c0;
        double xw[2 * R + 2 + 2 * XO];
#pragma unroll
        for (int t = 0; t < R + 1 + XO; ++t) {
            const double2 pv = *reinterpret_cast<const double2 *>(cr + 2 * t);
            xw[2 * t] = pv.x;
            xw[2 * t + 1] = pv.y;
        }
        const double *xv = xw + XO;                     // xv[R + k] = u1(c0 + k)
        // y[R + k] = u1 of row (center + k) = slot (u - R + k) mod NQ
        auto Y0 = [&](int k) -> double { return q0[(u - R + k + 2 * NQ) % NQ]; };
        auto Y1 = [&](int k) -> double { return q1[(u - R + k + 2 * NQ) % NQ]; };
        const double2 v2 = *reinterpret_cast<const double2 *>(s2 + slot * kTW + c0);
        double o0, o1;
        if constexpr (SYM) {
            double lap0 = c_omega[R] * (Y0(0) + Y0(0));
            double lap1 = c_omega[R] * (Y1(0) + Y1(0));
#pragma unroll
            for (int k = 1; k <= R; ++k) {
                const double om = c_omega[R + k];
                lap0 = fma(om, (xv[R - k] + xv[R + k]) + (Y0(-k) + Y0(k)), lap0);
                lap1 = fma(om, (xv[R - k + 1] + xv[R + k + 1]) + (Y1(-k) + Y1(k)), lap1);
            }
            o0 = fma(-dt2, lap0, fma(-2.0, Y0(0), v2.x));
            o1 = fma(-dt2, lap1, fma(-2.0, Y1(0), v2.y));
        } else {
            double lap0 = 0.0, lap1 = 0.0;
#pragma unroll
            for (int k = -R; k <= R; ++k) {
                const double om = c_omega[R + k];
                // lap += weight[r+k]*u1[j*w + nX] + weight[r+k]*u1[nY*w + i]
                lap0 = __dadd_rn(lap0, __dadd_rn(__dmul_rn(om, xv[R + k]), __dmul_rn(om, Y0(k))));
                lap1 = __dadd_rn(lap1, __dadd_rn(__dmul_rn(om, xv[R + k + 1]), __dmul_rn(om, Y1(k))));
            }
            // u3[id] = (-2*r_u1 + r_u2 - dt*dt*lap)
            o0 = __dsub_rn(__dadd_rn(__dmul_rn(-2.0, Y0(0)), v2.x), __dmul_rn(dt2, lap0));
            o1 = __dsub_rn(__dadd_rn(__dmul_rn(-2.0, Y1(0)), v2.y), __dmul_rn(dt2, lap1));
        }
        const int64_t x = i0 + c0;
        double *out = u3 + j * w + x;
        if (x + 1 < w) {
            if ((w & 1) == 0) {
                __stcs(reinterpret_cast<double2 *>(out), make_double2(o0, o1));
            } else {
                __stcs(out, o0);
                __stcs(out + 1, o1);
            }
        } else if (x < w) {
            __stcs(out, o0);
        }
    };
    for (int s0 = 0; s0 < nl; s0 += NQ) {
        static_for<NQ>([&](auto uc) {
            const int s = s0 + decltype(uc)::value;
            if (s < nl) step(s, uc);
        });
    }
    cp_async_wait<0>();
}

static thread_local std::string g_fd_err;

static int fd_fail(int code, const char *msg) {
    g_fd_err = msg;
    return code;
}

// rows per CTA strip (the 2r halo rows are re-read per strip); SEM_FD_STRIP
// overrides it for experiments
// (measured on 8192^2: 32 rows best up to r = 4, 64 above -- tools/gpu_r01q.sh)
static int strip_rows(int r) {
    static const int v = [] {
        const char *e = getenv("SEM_FD_STRIP");
        const int x = e ? atoi(e) : 0;
        return x >= 8 ? x : 0;
    }();
    return v ? v : (r <= 4 ? 32 : 64);
}

template <int R, bool SYM>
static cudaError_t launch_rs(const double *u1, const double *u2, double *u3, int64_t w, int64_t h,
                             double dt2, const Omega &om, cudaStream_t s) {
    using C = FdCfg<R>;
    // the shared-memory opt-in is per device: one bit per ordinal (set after a
    // successful call; a racing second call just repeats it)
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = dev < 64 ? (uint64_t(1) << dev) : 0;
    if (!bit || !(attr_set.load(std::memory_order_acquire) & bit)) {
        e = cudaFuncSetAttribute(fd2d_kernel<R, SYM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)C::SMEM);
        if (e != cudaSuccess) return e;
        attr_set.fetch_or(bit, std::memory_order_acq_rel);
    }
    const int ty = strip_rows(R);
    dim3 grid((unsigned)((w + kTW - 1) / kTW), (unsigned)((h + ty - 1) / ty));
    fd2d_kernel<R, SYM><<<grid, kNT, C::SMEM, s>>>(u1, u2, u3, w, h, ty, dt2, om);
    return cudaGetLastError();
}

template <int R>
static cudaError_t launch_r(bool sym, const double *u1, const double *u2, double *u3, int64_t w,
                            int64_t h, double dt2, const Omega &om, cudaStream_t s) {
    return sym ? launch_rs<R, true>(u1, u2, u3, w, h, dt2, om, s)
               : launch_rs<R, false>(u1, u2, u3, w, h, dt2, om, s);
}

static cudaError_t launch(int r, bool sym, const double *u1, const double *u2, double *u3,
                          int64_t w, int64_t h, double dt2, const Omega &om, cudaStream_t s) {
    switch (r) {
    case 1: return launch_r<1>(sym, u1, u2, u3, w, h, dt2, om, s);
    case 2: return launch_r<2>(sym, u1, u2, u3, w, h, dt2, om, s);
    case 3: return launch_r<3>(sym, u1, u2, u3, w, h, dt2, om, s);
    case 4: return launch_r<4>(sym, u1, u2, u3, w, h, dt2, om, s);
    case 5: return launch_r<5>(sym, u1, u2, u3, w, h, dt2, om, s);
    case 6: return launch_r<6>(sym, u1, u2, u3, w, h, dt2, om, s);
    case 7: return launch_r<7>(sym, u1, u2, u3, w, h, dt2, om, s);
    default: return cudaErrorInvalidValue;
    }
}

// FD_REGROUPED needs exactly symmetric weights (the pairs share one omega)
static bool symmetric(int r, const double *omega) {
    for (int k = 1; k <= r; ++k)
        if (!(omega[r - k] == omega[r + k])) return false;
    return true;
}

static int check(const double *u1, const double *u2, const double *u3, int64_t w, int64_t h, int r,
                 const double *omega, double dt) {
    if (r < 1 || r > FD_RMAX) return fd_fail(SEM_EINVAL, "fd2d: r must be in [1, FD_RMAX]");
    if (!u1 || !u2 || !u3 || !omega) return fd_fail(SEM_EINVAL, "fd2d: NULL pointer");
    if (w < 2 * r + 1 || h < 2 * r + 1) return fd_fail(SEM_EINVAL, "fd2d: w, h must be >= 2r+1");
    if (w > (int64_t(1) << 31) || h > (int64_t(1) << 31) || w * h >= (int64_t(1) << 62))
        return fd_fail(SEM_EINVAL, "fd2d: grid too large");
    if ((reinterpret_cast<uintptr_t>(u1) | reinterpret_cast<uintptr_t>(u2) |
         reinterpret_cast<uintptr_t>(u3)) & 15)
        return fd_fail(SEM_EINVAL, "fd2d: buffers must be 16-byte aligned");
    if (u1 == u2 || u1 == u3 || u2 == u3) return fd_fail(SEM_EINVAL, "fd2d: buffers must be distinct");
    if (!(dt == dt)) return fd_fail(SEM_EINVAL, "fd2d: dt is NaN");
    return SEM_OK;
}

static Omega pack(int r, const double *omega) {
    Omega o{};
    for (int k = 0; k <= 2 * r; ++k) o.w[k] = omega[k];
    return o;
}

}  // namespace sem_fd

using namespace sem_fd;

// Fornberg's recursion (Math. Comp. 51, 1988) for the weights of the second
// derivative at 0 on the nodes -r..r (times dx), then / dx^2.
extern "C" int fd_weights(int r, double dx, double *omega) {
    if (r < 1 || r > 16 || !(dx > 0.0) || !omega) return fd_fail(SEM_EINVAL, "fd_weights: bad arguments");
    const int n = 2 * r;          // nodes 0..n at x = (q - r)
    const int M = 2;
    std::vector<double> c((n + 1) * (M + 1), 0.0);
    auto C = [&](int q, int m) -> double & { return c[q * (M + 1) + m]; };
    auto X = [&](int q) { return double(q - r); };
    double c1 = 1.0, c4 = X(0);
    C(0, 0) = 1.0;
    for (int i = 1; i <= n; ++i) {
        const int mn = i < M ? i : M;
        double c2 = 1.0;
        const double c5 = c4;
        c4 = X(i);
        for (int j = 0; j < i; ++j) {
            const double c3 = X(i) - X(j);
            c2 *= c3;
            if (j == i - 1) {
                for (int m = mn; m >= 1; --m)
                    C(i, m) = c1 * (m * C(i - 1, m - 1) - c5 * C(i - 1, m)) / c2;
                C(i, 0) = -c1 * c5 * C(i - 1, 0) / c2;
            }
            for (int m = mn; m >= 1; --m) C(j, m) = (c4 * C(j, m) - m * C(j, m - 1)) / c3;
            C(j, 0) = c4 * C(j, 0) / c3;
        }
        c1 = c2;
    }
    // central stencil: mirror the k > 0 half so omega_{-k} == omega_k exactly
    // (the recursion's two halves can differ in the last bit)
    const double s = 1.0 / (dx * dx);
    omega[r] = C(r, 2) * s;
    for (int k = 1; k <= r; ++k) omega[r + k] = omega[r - k] = C(r + k, 2) * s;
    return SEM_OK;
}

extern "C" int fd2d_step(const double *u1, const double *u2, double *u3, int64_t w, int64_t h, int r,
                         const double *omega, double dt, void *stream) {
    int rc = check(u1, u2, u3, w, h, r, omega, dt);
    if (rc) return rc;
    cudaError_t e = launch(r, false, u1, u2, u3, w, h, dt * dt, pack(r, omega),
                           static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fd_fail(SEM_ECUDA, cudaGetErrorString(e));
    return SEM_OK;
}

extern "C" int fd2d_run_ex(double *u1, double *u2, double *u3, int64_t w, int64_t h, int r,
                           const double *omega, double dt, int steps, int flags, void *stream,
                           int *latest) {
    int rc = check(u1, u2, u3, w, h, r, omega, dt);
    if (rc) return rc;
    if (steps < 0) return fd_fail(SEM_EINVAL, "fd2d_run: steps < 0");
    if (flags & ~FD_REGROUPED) return fd_fail(SEM_EINVAL, "fd2d_run_ex: unknown flags");
    const bool sym = (flags & FD_REGROUPED) != 0;
    if (sym && !symmetric(r, omega))
        return fd_fail(SEM_EINVAL, "fd2d_run_ex: FD_REGROUPED needs omega_{-k} == omega_k");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Omega om = pack(r, omega);
    double *b[3] = {u1, u2, u3};
    int role[3] = {0, 1, 2};     // argument buffer playing u1, u2, u3
    for (int t = 0; t < steps; ++t) {
        cudaError_t e = launch(r, sym, b[role[0]], b[role[1]], b[role[2]], w, h, dt * dt, om, s);
        if (e != cudaSuccess) return fd_fail(SEM_ECUDA, cudaGetErrorString(e));
        const int n1 = role[2], n2 = role[0], n3 = role[1];   // (u1, u2, u3) <- (u3, u1, u2)
        role[0] = n1, role[1] = n2, role[2] = n3;
    }
    if (latest) *latest = role[0];
    return SEM_OK;
}

extern "C" int fd2d_run(double *u1, double *u2, double *u3, int64_t w, int64_t h, int r,
                        const double *omega, double dt, int steps, void *stream, int *latest) {
    return fd2d_run_ex(u1, u2, u3, w, h, r, omega, dt, steps, 0, stream, latest);
}
