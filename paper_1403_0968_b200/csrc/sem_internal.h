// sem_internal.h -- internal types shared by the host orchestration
// (sem_host.cpp) and the sm_100a kernels (sem_kernels.cu).  Not part of the ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace sem {

constexpr int kRing = 4;        // scalar ring depth (iteration k uses slot k & 3)
constexpr int kMaxRanks = 64;
constexpr int kTmaMaxN = 10;     // TMA-pipelined Ax kernel for N <= 10

// Device-resident CG state (one per context, in the workspace).
struct CgState {
    double rho0;                // (r0, r0)_c, written by K1 at k = 0 (the stopping norm)
    double tol;
    int32_t maxit;
    int32_t done;               // sticky: 1 once the stopping rule fired
    int32_t iters;              // iteration count at which it fired
    int32_t converged;          // 1 if sqrt(rho) <= tol sqrt(rho0) (or rho0 == 0)
    double rel_res;             // sqrt(rho_k / rho0)
    double alpha_km1;           // alpha_{it-1} at the stop, for the final x update
    int32_t k1;                 // iteration of the next K1 (written by K2 / the CG start)
    int32_t k2;                 // iteration of the next K2 (written by K1)
    // single-reduction CG (NEXT-3): gamma_k, alpha_k of iteration k in slot k & 1
    double gamma_hist[2];
    double alpha_hist[2];
    int32_t rcg_err;            // resident CG: 1 = a grid barrier timed out (lost CTA)
    int32_t pad_;
};

// Gather-scatter groups are stored by class (Dirichlet flag, multiplicity m):
// groups [start[c], start[c+1]) of class c have m[c] copies each; copy t of
// group start[c] + q is local index idx[idxoff[c] + t * count_c + q].
// Dirichlet classes come first.
constexpr int kMaxClasses = 40;
struct GsClasses {
    int32_t n;
    int32_t start[kMaxClasses + 1];
    int32_t m[kMaxClasses];
    int32_t idxoff[kMaxClasses];
    int32_t dir[kMaxClasses];
};

// Everything a kernel needs to know about the discretisation on this rank.
struct DevMesh {
    int N, n, n3;
    int64_t E, L;
    int64_t nbnd;               // elements [0, nbnd) touch a shared (inter-rank) node
    const double *D;            // [n][n] row-major, D[i*n+m] = phi'_m(xi_i)
    const double *G;            // [E][6][n3] rr rs rt ss st tt (w J folded in)
    const double *BM;           // [L] lumped mass w_i w_j w_k J
    const double *H;            // [L] alpha w_i w_j w_k J (screened-Coulomb mass term) or
                                // nullptr (Poisson); kappa is folded into G
    // gather-scatter plan over element-SURFACE nodes: groups of local copies of
    // one global id, Dirichlet groups first ([0, ndir)), copies in ascending
    // local order, stored by class (see GsClasses).
    GsClasses cls;
    const int32_t *gs_idx;      // [nsurf], class-transposed
    const uint32_t *own;        // nranks > 1: bit g set = group g counted in (r,r) here
                                // (its lowest sharing rank is this one); nullptr on one rank
    int32_t ngroups, ndir, nsurf;
    int rank, nranks;
    int nsm;                    // SM count of the device (persistent grids)
    bool use_tma;               // TMA element-staged Ax kernels (N <= kTmaMaxN)
    bool use_hi;                // TMA vector + register-streamed G^ kernels (high N)
    bool use_dmma;              // N = 7: r/s contractions on the FP64 tensor cores (ax_dmma.cuh)
    bool use_dmmag;             // N = 8..11: the plain Ax on the tensor cores (ax_dmmag.cuh)
    bool use_k1ax;              // CG K1 split in two launches: x / p update (k1u_kernel), then
                                // the operator with (p, A p) partials -- the tensor-core one
                                // (use_dmmag) or the CUDA-core TMA / high-order one; !H
};

struct CgVecs {
    const double *b;
    double *x;                  // the caller's x of this solve (x0 in, solution out)
    double *xw;                 // workspace copy of x updated by K1 (graph-invariant pointer)
    double *r, *p, *w;
    double *part1;              // [2][s1] per-block partials of (p, A p) (K1)
    double *part2;              // [2][s2] per-block partials of (r, r) (K2)
    int nb1, s1, nb2, s2;       // grids of K1 / K2 and buffer strides
    double *rr_all;             // [kRing][nranks] rank values of (r,r)_c (nranks > 1)
    double *pap_all;            // [kRing][nranks] rank values of (p,Ap) (nranks > 1)
    CgState *st;
    // Jacobi PCG (NEXT-2; nullptr dinv = identity preconditioner, plain CG):
    // z = dinv .* r written by K2 next to r, read by K1 in place of r
    const double *dinv;         // [L] mask / (Q Q^T diag A_L), continuous
    double *z;                  // [L]
    double *part3;              // [2][s2] per-block partials of (r, z) (K2) = part2 + 2 s2
    double *rz_all;             // [kRing][nranks] rank values of (r,z)_c = rr_all + kRing nranks
};

// the vector K1 forms p from: p = z + beta p (PCG) or p = r + beta p (CG)
inline const double *k1_src(const CgVecs &v) { return v.dinv ? v.z : v.r; }

constexpr int kGsThreads = 256;
constexpr int kMaxPartials = 1024;     // per-block partial slots of K1 / K2 (<= 4 CTAs/SM)

// ---- launchers (sem_kernels.cu); all return cudaGetLastError() ----
int ax_blocks(int N, int64_t E);      // grid size of the Ax kernels for E elements
// kappa: [L] or nullptr (G *= kappa); H: [L] holding alpha on entry (-> alpha w J)
// or nullptr
cudaError_t launch_geom(const DevMesh &m, const double *xyz, const double *kappa, double *G,
                        double *BM, double *H, int *bad, cudaStream_t s);
cudaError_t launch_ax(const DevMesh &m, const double *u, double *w, cudaStream_t s);
// The CG kernels take the iteration k from CgState (device), so one captured
// CUDA graph of a chunk of iterations is valid for every chunk.
cudaError_t launch_ax_cg(const DevMesh &m, const CgVecs &v, cudaStream_t s);
int ax_cg_blocks(const DevMesh &m);   // grid of K1 (= number of its partials)
// multi-rank TMA/high-order K1 runs as two launches, boundary elements [0, nbnd)
// first, so the DSSUM exchange overlaps the interior launch
bool k1_split(const DevMesh &m);
int ax_cg_range_blocks(const DevMesh &m, int64_t ne);
cudaError_t launch_ax_cg_range(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                               int pidx0, cudaStream_t s);
// mode: 0 = plain dssum, 1 = dssum + mask, 2 = CG iteration (dssum + mask,
// programmatic dependent of K1, no-op after the stop; v needed)
cudaError_t launch_gs(const DevMesh &m, double *w, int mode, const CgVecs *v, cudaStream_t s);
cudaError_t launch_mask(const DevMesh &m, double *w, cudaStream_t s);
cudaError_t launch_mass(const DevMesh &m, const double *f, double *b, cudaStream_t s);
// xw = x0, resets the CG state (k = 0)
cudaError_t launch_cg_init(const DevMesh &m, const CgVecs &v, cudaStream_t s);
// cg_update.cu, K2: Q Q^T w + mask fused with the r update; per-block (r,r)
// partials into part2[k & 1]; init: r0 = mask (b - Q Q^T w) into part2[1]
int k2_blocks(const DevMesh &m, bool init);
cudaError_t launch_k2(const DevMesh &m, const CgVecs &v, bool init, cudaStream_t s);
cudaError_t launch_cg_finish(const DevMesh &m, const CgVecs &v, cudaStream_t s);
// multi-rank: fold this rank's block partials (fixed order) into its slot of
// pap_all / rr_all before the NCCL all-gather
// (p2p: the peer-memory transport's descriptor -- the fold then also does the
// all-gather; nullptr: fold only)
struct P2PDev;
cudaError_t launch_cg_red_pap(const DevMesh &m, const CgVecs &v, const P2PDev *p2p, cudaStream_t s);
cudaError_t launch_cg_red_rr(const DevMesh &m, const CgVecs &v, const P2PDev *p2p, cudaStream_t s);
cudaError_t launch_cg_red_rz(const DevMesh &m, const CgVecs &v, const P2PDev *p2p, cudaStream_t s);
// single-reduction (Chronopoulos-Gear) CG, NEXT-3 (cg_update.cu, ax_tma_sr.cu).
// Global storage: p, s and the x increment live once per global node of the
// rank -- surface group g at slot g, element-interior node t at ngroups + t --
// in the workspace vectors p, z and xw.  sr_all: [kRing][nranks][2] rank
// values of (gamma, delta) (the rr_all region).
cudaError_t upload_const_D_sr(int N, const double *D_host);
cudaError_t sr_prepare(const DevMesh &m);
cudaError_t launch_ax_dot(const DevMesh &m, const CgVecs &v, cudaStream_t s);   // KA
int ka_blocks(const DevMesh &m);                  // KA's grid = its partial count
cudaError_t launch_kb_sr(const DevMesh &m, const CgVecs &v, cudaStream_t s);    // KB
cudaError_t launch_sr_init(const DevMesh &m, const CgVecs &v, cudaStream_t s);
cudaError_t launch_sr_finish(const DevMesh &m, const CgVecs &v, cudaStream_t s);
cudaError_t launch_sr_fold(const DevMesh &m, const CgVecs &v, const P2PDev *p2p,
                           cudaStream_t s);  // nranks > 1
// Jacobi preconditioner (NEXT-2): d = diag(A_L) per local node (unassembled;
// kappa-folded G^ + the mass term H); then, after Q Q^T d, dinv = 1 / d
// (the caller masks it)
cudaError_t launch_diag(const DevMesh &m, double *d, cudaStream_t s);
cudaError_t launch_recip(const DevMesh &m, const double *d, double *dinv, cudaStream_t s);

// cg_resident.cu: the whole CG solve at N = 7 as one persistent cooperative
// kernel with x, r in TMEM and p in shared memory (one rank, Poisson, no
// preconditioner, E <= 28 per SM).  Runs after the CG start (cg_init + K2
// INIT) and leaves x, the state words and rcg_err behind.
constexpr int kRcgMaxM = 8;           // largest multiplicity of a non-Dirichlet group
constexpr int kRcgMaxSlots = 1024;    // receive slots per element (S, even)
struct RcgBufs {
    int32_t S;                  // receive slots per element
    uint8_t *meta;              // [L] m | pos << 4 (m = 0: Dirichlet copy)
    int32_t *sbq;               // [n^3] first receive slot of each node position
    int32_t *push;              // [E][S] destination (index into X) of each pushed value
    double *X;                  // [E][S] receive slots: the other copies' w, ascending
    double *part;               // [2][kMaxPartials] per-CTA partials
    uint32_t *bar;              // grid barrier counter; bar + 16: 4 x uint64 phase clocks
};
bool rcg_supported(const DevMesh &m);
int rcg_blocks(const DevMesh &m);
cudaError_t rcg_prepare();
cudaError_t upload_const_D_rcg(int N, const double *D_host);
cudaError_t launch_rcg(const DevMesh &m, const CgVecs &v, const RcgBufs &rb, cudaStream_t s);

// ax_tma_pc.cu: Jacobi PCG whose K1 forms z = dinv r itself (K2 then skips z)
bool pcg_z_in_k1(const DevMesh &m);

// ax_tma.cu
bool tma_supported(int N);
bool dmma_supported(int N);
bool dmmag_supported(int N);
cudaError_t dmmag_prepare(int N);
cudaError_t launch_ax_dmmag(const DevMesh &m, const double *u, double *w, cudaStream_t s);
int tma_blocks(int N, int64_t E, int nsm, bool cg);
int dmma_blocks(int64_t E, int nsm, bool cg);   // N = 7 tensor-core kernel grid
int dmmag_blocks(int N, int64_t E, int nsm);     // N >= 8 tensor-core kernel grid
// the split K1 (use_k1ax): k1u_kernel over the range, then ax_dmmag_kernel<DOT>
cudaError_t launch_ax_cg_dmmag(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, int pidx0,
                               cudaStream_t s);
cudaError_t launch_k1u(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, cudaStream_t s);
// the split K1 with the CUDA-core TMA / high-order operator (use_k1ax, !use_dmmag)
int k1dot_blocks(const DevMesh &m, int64_t ne);
cudaError_t launch_k1dot_range(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne, int pidx0,
                               cudaStream_t s);
cudaError_t tma_prepare(int N, bool mass);
cudaError_t upload_const_D(int N, const double *D_host);
cudaError_t launch_ax_tma(const DevMesh &m, const double *u, double *w, cudaStream_t s);
cudaError_t launch_ax_cg_tma(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                             int pidx0, cudaStream_t s);
bool hi_supported(int N);
int hi_blocks(int N, int64_t E, int nsm, bool cg);
cudaError_t hi_prepare(int N, bool mass);
cudaError_t launch_ax_hi(const DevMesh &m, const double *u, double *w, cudaStream_t s);
cudaError_t launch_ax_cg_hi(const DevMesh &m, const CgVecs &v, int64_t eb, int64_t ne,
                            int pidx0, cudaStream_t s);

}  // namespace sem
