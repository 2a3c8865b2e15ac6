/*
 * fd.h -- C ABI of the finite-difference wave-equation example of arXiv
 * 1403.0968 (Sec. "Finite Difference"; SURVEY.md §8(f)
 * NEXT-4), exported by libsem.so next to sem.h:
 *
 *   fd_weights  the 2r+1 stencil weights omega_{-r..r} (the paper gives none:
 *               DESIGN.md reading R6 -- central second-derivative weights of
 *               order 2r, / dx^2; this library derives them by Fornberg's
 *               recursion)
 *   fd2d_step   one step of lst:fdCode (alg:fdPseudocode
 *               :397-412) on a periodic w x h grid:
 *                 lap = sum_{k=-r..r} (omega_k u1(i+k, j) + omega_k u1(i, j+k))
 *                 u3  = -2 u1 + u2 - dt^2 lap
 *               in exactly the listing's operation order (no FMA contraction),
 *               so results are bit-identical to a plain C evaluation
 *   fd2d_run    `steps` steps with the buffer rotation of reading R6b
 *               (u_{n+1} -> u_n -> u_{n-1}: (u1, u2, u3) <- (u3, u1, u2))
 *
 * Conventions: u1, u2, u3 are DEVICE pointers to w*h doubles, node (i, j) at
 * j*w + i (i fastest), 16-byte aligned, pairwise distinct.  omega is a HOST
 * array of 2r+1 doubles.  1 <= r <= FD_RMAX; w, h >= 2r+1 (the listing's
 * wrap-around), w*h < 2^62.  Work is enqueued on `stream` (a cudaStream_t,
 * NULL = legacy default) without a host synchronisation.  Return codes are
 * sem.h's: SEM_OK, SEM_EINVAL (bad argument), SEM_ECUDA (CUDA failure; message
 * in sem_last_error(NULL)).
 */
#ifndef FD_H
#define FD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FD_RMAX 7   /* stencil sizes 3..15, the paper's sweep (fig:fdTable) */

/* omega[0..2r] = omega_{-r..r} for spacing dx > 0.  Pure host function. */
int fd_weights(int r, double dx, double *omega);

/* u3 = -2 u1 + u2 - dt^2 lap(u1).  Asynchronous. */
int fd2d_step(const double *u1, const double *u2, double *u3, int64_t w, int64_t h, int r,
              const double *omega, double dt, void *stream);

/* `steps` >= 0 steps starting from u1 = u_n, u2 = u_{n-1}; after each step the
 * roles rotate (u1, u2, u3) <- (u3, u1, u2).  *latest (HOST, may be NULL)
 * receives which argument buffer holds the newest solution at the end
 * (0 = u1, 1 = u2, 2 = u3); the previous one is the next in the rotation
 * ((latest + 1) mod 3 holds u_{n-1} of the final state).  Asynchronous. */
int fd2d_run(double *u1, double *u2, double *u3, int64_t w, int64_t h, int r, const double *omega,
             double dt, int steps, void *stream, int *latest);

/* fd2d_run with options.  flags = 0: exactly fd2d_run (the listing's operation
 * order, bit-identical to a plain C evaluation).  FD_REGROUPED: the
 * pair-regrouped FMA form (reading R6c)
 *   lap = omega_0 (u + u) + sum_k omega_k ((u_{i-k} + u_{i+k}) + (u_{j-k} + u_{j+k}))
 * -- 4r+3 FP64 operations per node instead of 8r+8, equal to the listing up
 * to rounding; requires exactly symmetric weights (omega_{-k} == omega_k, as
 * fd_weights returns), else SEM_EINVAL.  Unknown flags: SEM_EINVAL. */
#define FD_REGROUPED 1
int fd2d_run_ex(double *u1, double *u2, double *u3, int64_t w, int64_t h, int r,
                const double *omega, double dt, int steps, int flags, void *stream, int *latest);

#ifdef __cplusplus
}
#endif
#endif /* FD_H */
