/*
 * sem.h -- C ABI of libsem, the B200-native (sm_100a) hot path of the
 * spectral-element Poisson benchmark of arXiv 1403.0968 (OCCA), Sec.
 * "Spectral Element Methods", PAPER.md:578-784:
 *
 *   sem_ax     local matrix-free stiffness operator w = A_L u on order-N hexahedra
 *              (eq:semOperator, with kappa = 1, alpha = 0;
 *              tensor-product GLL basis :599-604; derivative sparsity :615-625;
 *              chain rule and G^ = G^T G "precomputed for each elemental node"
 *              :627-665)
 *   sem_dssum  direct-stiffness summation w <- Q Q^T w over the global-local
 *              numbering (Fischer 1991)
 *   sem_mask   homogeneous Dirichlet mask (paper silent; reading G7)
 *   sem_mass   lumped diagonal mass b = J w_abc f (discrete orthogonality,
 *              PAPER.md:605-614) -- used to assemble right-hand sides
 *   sem_cg     the (P)CG iteration that drives them (identity
 *              preconditioner, reading G8)
 *
 * Conventions (all entry points):
 *  - Every function returns an int status (SEM_OK = 0) and never throws or
 *    aborts across the ABI.  sem_last_error() gives a message for the last
 *    failure on a context; sem_strerror() names a status code.
 *  - Vectors u, w, b, x, f are DEVICE pointers (CUDA global memory on the
 *    context's device) of nlocal = E * (N+1)^3 doubles in "local" (E-vector)
 *    storage: node (i,j,k) of element e at e*(N+1)^3 + i + (N+1)*j + (N+1)^2*k,
 *    i (the r direction) fastest.  They must be 16-byte aligned (the kernels
 *    stage them with bulk copies and 128-bit accesses).  The caller owns
 *    them (PyTorch tensors in the Python binding).
 *  - All device work is enqueued on the CUDA stream given to sem_setup and the
 *    call returns without a host synchronisation, except sem_setup and sem_cg,
 *    which synchronise that stream before returning.
 *  - The caller owns the device workspace passed to sem_setup (size from
 *    sem_workspace_bytes); it must stay allocated until sem_free.  The library
 *    allocates no device memory of its own on one rank; with nranks > 1 it
 *    allocates its small interface-exchange buffers and NCCL does its own.
 *  - sem_setup, sem_dssum and sem_cg are COLLECTIVE when nranks > 1: every rank
 *    must call them in the same order.
 *  - Errors: SEM_EINVAL for a NULL pointer, N outside [1, SEM_NMAX], an empty or
 *    malformed mesh (non-positive Jacobian, inconsistent Dirichlet flags across
 *    copies of a global node, an element-interior node that is shared or
 *    Dirichlet), or a misaligned pointer; SEM_ECUDA for a CUDA runtime failure
 *    (the context is then unusable); SEM_ENCCL for an NCCL failure, including
 *    an asynchronous one (ncclCommGetAsyncError, polled while sem_cg waits for
 *    the device; the communicator is then aborted and the context unusable);
 *    SEM_ENOCONV when sem_cg reached maxit with tol > 0 (x holds the last
 *    iterate; not a failure for tol == 0); SEM_ESTATE for a NULL/freed context.
 */
#ifndef SEM_H
#define SEM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SEM_NMAX 15

enum sem_status {
    SEM_OK = 0,
    SEM_EINVAL = 1,
    SEM_ECUDA = 2,
    SEM_ENCCL = 3,
    SEM_ENOCONV = 4,
    SEM_ESTATE = 5
};

/* Host-side all-gather used ONLY during sem_setup when nranks > 1 (to find the
 * global ids shared with each peer).  Must place the `bytes` bytes of every
 * rank's `send` buffer into `recv` in rank order (recv holds nranks*bytes).
 * Returns 0 on success.  The Python binding implements it with
 * torch.distributed (gloo or nccl). */
typedef int (*sem_allgather_fn)(void *user, const void *send, size_t bytes, void *recv);

typedef struct {
    int32_t nelem;             /* E, elements owned by this rank (> 0)                      */
    const double *xyz;         /* HOST [E][3][(N+1)^3] coordinates of the GLL nodes
                                  (isoparametric map x(r,s,t)), i fastest      */
    const int64_t *glo;        /* HOST [E][(N+1)^3] global node ids (global-local numbering,
                                  PAPER.md:667), consistent across ranks, >= 0               */
    const uint8_t *dirichlet;  /* HOST [E][(N+1)^3] 1 = homogeneous Dirichlet node           */
    int32_t nboundary;         /* the first nboundary elements touch a partition interface
                                  (ordering hint for overlap; 0 = unknown)                   */
    int32_t rank, nranks;      /* 0, 1 on one GPU                                            */
    const void *nccl_id;       /* 128-byte ncclUniqueId (rank 0's), required if nranks > 1   */
    sem_allgather_fn allgather;/* setup-time host all-gather, required if nranks > 1         */
    void *allgather_user;
    int32_t device;            /* CUDA device ordinal                                        */
    /* Screened-Coulomb coefficients (eq:semPDE -div(kappa grad u) + alpha u = f,
     * PAPER.md:580-586).  HOST [E][(N+1)^3] values at the
     * GLL nodes, read during sem_setup only.  NULL: kappa = 1 / alpha = 0 (the
     * Poisson operator).  kappa must be > 0 and finite, alpha >= 0 and finite,
     * else SEM_EINVAL.  kappa weights the flux pointwise (folded into G^ at setup,
     * DESIGN.md reading G2); alpha adds the lumped mass alpha w_i w_j w_k J
     * to the local operator (+8 B per node per apply).      */
    const double *kappa;
    const double *alpha;
} sem_mesh;

typedef struct sem_ctx sem_ctx;  /* opaque; created by sem_setup, destroyed by sem_free */

/* Library version string. */
const char *sem_version(void);

/* The library's own 1-D GLL nodes xi[N+1] (ascending, xi_0 = -1, xi_N = 1) and
 * weights w[N+1].  HOST arrays.  Pure function; no
 * GPU needed.  Mesh generators use xi to place the GLL nodes. */
int sem_gll(int N, double *xi, double *w);

/* Bytes of device workspace sem_setup needs for this mesh and order.  Pure
 * host query (looks only at nelem); no GPU needed. */
int sem_workspace_bytes(const sem_mesh *mesh, int N, size_t *bytes);

/* Build a context: GLL nodes and D (a0), geometric factors G^ with w J folded in
 * on the GPU (a1), gather-scatter plan from glo (a2, :667),
 * and for nranks > 1 the NCCL communicator and interface exchange lists.
 * `workspace` is a DEVICE buffer of at least sem_workspace_bytes bytes, 256-byte
 * aligned.  `cuda_stream` is a cudaStream_t (NULL = legacy default stream).
 * L2 (opt-in): with the environment variable SEM_L2_PERSIST=1, sem_setup raises the
 * device's persisting-L2 limit (cudaLimitPersistingL2CacheSize, never lowered)
 * to cover the four CG work vectors r, p, w, x-copy (contiguous in the
 * workspace, 32 nlocal bytes) and sem_cg's CUDA-graph kernels mark their
 * accesses to them persisting; sem_free resets the persisting lines.
 * Collective.  Synchronises the stream before returning. */
int sem_setup(const sem_mesh *mesh, int N, void *workspace, size_t bytes,
              void *cuda_stream, sem_ctx **out);

/* nlocal = E (N+1)^3 on this rank; nglobal = number of distinct global ids on
 * ALL ranks. */
int sem_sizes(const sem_ctx *ctx, int64_t *nlocal, int64_t *nglobal);

/* w = A_L u: local, unassembled, unmasked stiffness apply (eq:semOperator).
 * u and w are DEVICE [nlocal] and must not alias.  Asynchronous. */
int sem_ax(sem_ctx *ctx, const double *u, double *w);

/* In place w <- Q Q^T w (copies of each global id summed in ascending local
 * order, then summed across ranks in ascending rank order).  No mask.
 * Collective.  Asynchronous. */
int sem_dssum(sem_ctx *ctx, double *w);

/* In place w <- mask .* w (zero at Dirichlet nodes).  Asynchronous. */
int sem_mask(sem_ctx *ctx, double *w);

/* b = B_L f with B_L = diag(w_i w_j w_k J) the lumped local mass
 * (PAPER.md:605-614).  Unassembled; follow with sem_dssum / sem_mask to form a
 * right-hand side.  f and b may alias.  Asynchronous. */
int sem_mass(sem_ctx *ctx, const double *f, double *b);

/* Solve mask Q Q^T A_L x = mask b by CG (recurrence and
 * stopping rule in DESIGN.md / SURVEY.md §8(c) O7):
 *   inner product (a,b)_c = sum over distinct non-Dirichlet global nodes;
 *   stop before iteration k when k == maxit or sqrt(rho_k) <= tol sqrt(rho_0).
 * b: DEVICE, continuous (already assembled); x: DEVICE, in = x0, out = solution.
 * iters / rel_res (HOST, may be NULL) receive the iteration count and
 * sqrt(rho_k / rho_0).  Collective.  Synchronises the stream.  Returns
 * SEM_ENOCONV if maxit was reached with tol > 0. */
int sem_cg(sem_ctx *ctx, const double *b, double *x, double tol, int maxit,
           int *iters, double *rel_res);

/* Preconditioners of sem_pcg ("PCG ... Besides the
 * preconditioner choice"). */
enum sem_precond {
    SEM_PC_NONE = 0,    /* identity: exactly sem_cg                                    */
    SEM_PC_JACOBI = 1   /* M = diag of the assembled masked operator, M^-1 = mask / QQ^T d */
};

/* Preconditioned CG, same contract as sem_cg (b, x, tol, maxit, iters, rel_res,
 * collective, synchronises the stream), with the preconditioned
 * Hestenes-Stiefel recurrence (reading R4):
 *   z = M^-1 r;  rho = (r, z)_c;  p = z + (rho / rho_old) p;  alpha = rho / (p, A p)_c
 * while the stopping rule stays on the residual norm sqrt((r,r)_c) <= tol
 * sqrt((r0,r0)_c), so iteration counts compare directly with sem_cg.  The
 * Jacobi diagonal is formed on the first SEM_PC_JACOBI call (one extra
 * diag + DSSUM pass) and kept in the workspace.  SEM_EINVAL for an unknown
 * precond. */
int sem_pcg(sem_ctx *ctx, int precond, const double *b, double *x, double tol, int maxit,
            int *iters, double *rel_res);

/* Single-reduction CG (reading R7): the
 * Chronopoulos-Gear recurrence of the same CG (identity preconditioner,
 * Poisson operator): A is applied to the residual, A p is carried by
 * s = w + beta s, and both inner products of an iteration, (r,r)_c and
 * (r, A r)_c, are reduced at ONE point (one all-gather per iteration with
 * nranks > 1 instead of two).  Same contract as sem_cg (b, x, tol, maxit,
 * iters, rel_res, stopping rule, collective, synchronises).  x may hold a
 * discontinuous x0: the solution is x0 + the accumulated increment at every
 * copy.  SEM_EINVAL with a screened (alpha) operator or the simple Ax kernel. */
int sem_cg_sr(sem_ctx *ctx, const double *b, double *x, double tol, int maxit, int *iters,
              double *rel_res);

/* d = Q Q^T diag(A_L): the diagonal of the assembled (unmasked) operator in
 * local storage, diag(A^e)_q = sum over the three GLL lines through q
 * (DESIGN.md "Jacobi").  d: DEVICE [nlocal].  Collective.  Asynchronous. */
int sem_diag(sem_ctx *ctx, double *d);

/* Size of an ncclUniqueId (128) and a fresh one, for rank 0 to broadcast to
 * the other ranks before sem_setup (HOST buffer of sem_nccl_id_bytes()). */
int sem_nccl_id_bytes(void);
int sem_nccl_get_unique_id(void *id_out);

/* TEST-ONLY in-process transport (no NCCL): an id (HOST buffer of
 * sem_nccl_id_bytes() bytes) that, passed as sem_mesh.nccl_id to the nranks
 * contexts of ONE process -- one host thread per rank, all on one device, each
 * with its own stream -- makes their interface exchange and scalar all-gathers
 * device-to-device copies between the ranks' buffers, ordered by CUDA events
 * and a host rendezvous (a7 on a single GPU, where NCCL
 * refuses two ranks).  Everything else -- the exchange plan, pack/combine
 * kernels, rank-ordered sums, boundary/interior K1 split, the multi-rank CG
 * prologues -- runs exactly as with NCCL.  CUDA-graph capture of the CG chunks
 * is disabled for such contexts.  A rank that fails or stops calling the
 * collectives makes its peers fail with SEM_ENCCL after
 * SEM_LOOPBACK_TIMEOUT_MS (default 120000) instead of hanging. */
int sem_loopback_unique_id(void *id_out);

/* Transport selection (environment, read by sem_setup; all ranks must agree):
 * SEM_COMM=p2p selects the PEER-MEMORY transport instead of NCCL / the
 * host-rendezvous loopback: every rank owns a device window (exchange receive
 * areas, all-gather slots, per-site epoch flags); the interface exchange
 * stores each partial sum straight into the neighbour's window and the scalar
 * all-gathers are one-warp kernels that store into every peer's slots,
 * release a flag at system scope and acquire the peers' -- device work only,
 * captured into the CUDA graphs (the one-shot
 * device-side reduction).  Windows are shared as raw pointers inside one
 * process (the loopback world) and through CUDA IPC across processes
 * (peer access over NVLink).  Spins time out after SEM_P2P_TIMEOUT_MS
 * (default 20000) and make the context report SEM_ENCCL.  Caveat for several
 * ranks on ONE device (the loopback world): a rank that calls a
 * device-synchronising CUDA function (first allocations, lazy module loading)
 * while a peer's kernel spins stalls that peer until the timeout; warm up
 * first (CUDA_MODULE_LOADING=EAGER, allocate before the first collective). */

/* Device timing per kernel class, for the benchmark's roofline report.
 * sem_profile(ctx, 1) resets the accumulators and brackets every later launch
 * with a pair of CUDA events on the context stream (host-side cost only);
 * sem_profile(ctx, 0) stops.  sem_profile_read synchronises the stream and
 * returns, for class `which` (0 = sem_ax kernel, 1 = CG kernel K1: x/p update
 * + Ax + (w,p), 2 = CG kernel K2: DSSUM + mask fused with the r update and
 * (r,r), 3 = sem_dssum gather-scatter, 4 = other, 5 = the resident CG kernel:
 * the whole iteration loop of a one-rank N = 7 Poisson sem_cg as one launch,
 * bytes reported as 0 -- the caller knows the iteration count), the summed device
 * milliseconds, the number of launches that did work (CG launches after the
 * stopping decision are excluded) and their ALGORITHMIC bytes (DESIGN.md:
 * Ax 64 B/node; K1 96 B/node, 72 at k = 0; K2 16 B per surface copy + 8 B per
 * non-Dirichlet surface group + 24 B per element-interior node; gather-scatter
 * 16 B per surface copy). */
int sem_profile(sem_ctx *ctx, int enable);

/* Benchmark helper (one rank): enqueue, as ONE CUDA graph on the context
 * stream, `reps` back-to-back launches of one kernel of the CG iteration on the
 * context's internal work vectors (which = 1: K1, 2: K2, 0: the Ax kernel,
 * 3: the Ax kernel followed by the sem_dssum gather-scatter, config c2),
 * from a mid-solve state, so the caller can time the kernel with CUDA events
 * around the call.  The caller's vectors are untouched; the internal CG state
 * is left undefined until the next sem_cg.  Asynchronous. */
int sem_kernel_replay(sem_ctx *ctx, int which, int reps);
int sem_profile_read(sem_ctx *ctx, int which, double *ms, int64_t *launches, double *bytes);

/* Phase clock of the last sem_cg when it ran as the resident kernel (opt-in
 * with the environment variable SEM_CG_RESIDENT=1, set when the workspace is
 * sized (its tables add ~12 KB per element) and at sem_cg; one rank, N = 7, Poisson,
 * no preconditioner, E <= 28 per SM, non-Dirichlet multiplicities <= 8;
 * DESIGN.md §6 "Resident CG"): us[0..3] =
 * microseconds per iteration that CTA 0 spent in (0) the x / p update and the
 * operator of its elements, (1) the first grid barrier and the (p, A p) sum,
 * (2) the DSSUM + r update of its elements, (3) the second grid barrier and the
 * (r, r) sum (device %globaltimer).  Synchronises the context stream.
 * SEM_EINVAL if the last solve did not run resident. */
int sem_cg_phases(sem_ctx *ctx, double *us);

/* Host-only and collective over mesh->allgather: the interface exchange plan
 * sem_setup builds for nranks > 1, without touching a GPU.
 * counts[q] (HOST, [nranks]) = number of global ids this rank shares with rank
 * q; ids (HOST, [cap]) = those ids, peers in ascending rank order, ids
 * ascending within a peer (the order both sides pack and unpack in);
 * *nslot = total; *nglobal = distinct global ids over all ranks.  Returns
 * SEM_EINVAL (with *nslot set) if cap < *nslot.  For tests and tooling. */
int sem_exchange_plan(const sem_mesh *mesh, int N, int64_t *counts, int64_t *ids, int64_t cap,
                      int64_t *nslot, int64_t *nglobal);

/* SEM_OK, or the sticky error of the context: SEM_ENCCL after a collective
 * of the peer-memory transport timed out (a peer never arrived; the
 * asynchronous work of that collective used stale data), SEM_ECUDA after a
 * CUDA failure.  Does not synchronise.  Every collective entry point also
 * reports such an error. */
int sem_status(sem_ctx *ctx);

/* Number of kernels this context has launched so far (all entry points). */
int64_t sem_launch_count(const sem_ctx *ctx);

/* Destroy the context (the caller still owns workspace and vectors). */
void sem_free(sem_ctx *ctx);

const char *sem_strerror(int code);
const char *sem_last_error(const sem_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* SEM_H */
