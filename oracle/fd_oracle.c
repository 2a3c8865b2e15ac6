/*
 * fd_oracle.c -- plain CPU ORACLE for the finite-difference wave-equation
 * example of arXiv 1403.0968 (Sec. "Finite Difference", PAPER.md:362-576;
 * SURVEY.md §8(f) NEXT-4).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE (same rules as sem_oracle.c):
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it; it shares nothing with
 * paper_1403_0968_b200/csrc.  FP64, no FMA contraction (-ffp-contract=off).
 *
 * Notation (alg:fdPseudocode, lst:fdCode):
 *   w x h structured grid, node (i,j) at j*w + i (i fastest), periodic wrap
 *   (the listing's nX = (i + k + w) mod w, nY = (j + k + h) mod h);
 *   stencil radius r, 2r+1 weights omega_{-r..r}; u1 = u_n, u2 = u_{n-1},
 *   u3 = u_{n+1}.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#define ORA_OK 0
#define ORA_EINVAL 1

/* Reading R6: the paper gives no numerical omega_k ("a stencil of
 * size 2r+1").  omega = the central
 * second-derivative weights of order 2r scaled by 1/dx^2, the closed form
 *   omega_{+-k} = 2 (-1)^{k+1} (r!)^2 / (k^2 (r-k)! (r+k)!) / dx^2,  k = 1..r
 *   omega_0    = -2 sum_{k=1}^r omega_k
 * written to w[0..2r] = omega_{-r..r}.                                      */
int ora_fd_weights(int r, double dx, double *w)
{
    if (r < 1 || r > 16 || !(dx > 0.0) || !w) return ORA_EINVAL;
    double s = 0.0;
    for (int k = 1; k <= r; ++k) {
        /* (r!)^2 / ((r-k)! (r+k)!) = prod_{q=1}^{k} (r-q+1)/(r+q) */
        double ratio = 1.0;
        for (int q = 1; q <= k; ++q) ratio = ratio * (double)(r - q + 1) / (double)(r + q);
        double c = 2.0 * ratio / ((double)k * (double)k);
        if ((k & 1) == 0) c = -c;
        c = c / (dx * dx);
        w[r + k] = c;
        w[r - k] = c;
        s += c;
    }
    w[r] = -2.0 * s;
    return ORA_OK;
}

/* One time step, lst:fdCode line by line (alg:fdPseudocode
 * :397-412):
 *   lap = 0
 *   for k = -r..r:  lap += weight[r+k]*u1[j*w + nX] + weight[r+k]*u1[nY*w + i]
 *   u3[id] = (-2*u1[id] + u2[id] - dt*dt*lap)
 * with the sum of the two products formed first, then added to lap (the
 * listing's expression order).                                              */
int ora_fd_step(int64_t w, int64_t h, int r, const double *weight, double dt, const double *u1,
                const double *u2, double *u3)
{
    if (w < 2 * r + 1 || h < 2 * r + 1 || r < 1 || !weight || !u1 || !u2 || !u3)
        return ORA_EINVAL;
    for (int64_t j = 0; j < h; ++j)
        for (int64_t i = 0; i < w; ++i) {
            const int64_t id = j * w + i;
            double lap = 0.0;
            const double r_u1 = u1[id];
            const double r_u2 = u2[id];
            for (int k = -r; k <= r; ++k) {
                const int64_t nX = (i + k + w) % w;
                const int64_t nY = (j + k + h) % h;
                lap += weight[r + k] * u1[j * w + nX] + weight[r + k] * u1[nY * w + i];
            }
            u3[id] = (-2 * r_u1 + r_u2 - dt * dt * lap);
        }
    return ORA_OK;
}
