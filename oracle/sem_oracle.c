/*
 * sem_oracle.c -- plain, slow, obviously-correct CPU ORACLE for the SEM Poisson
 * hot path of arXiv 1403.0968 (OCCA), Sec. "Spectral Element Methods"
 * (PAPER.md:578-784).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
 * load it.  It shares no code, header, table or constant generator with the CUDA
 * library under paper_1403_0968_b200/csrc; neither includes or links the other.
 *
 * Every function follows the plain definition (or the algorithm, step by step)
 * of the passage it cites.  FP64, no blocking, no fusion, no reordering; build
 * without -ffast-math (FMA contraction is disabled with -ffp-contract=off).
 *
 * Notation:
 *   N      polynomial order, n = N+1 GLL nodes per direction
 *   xi_i   1-D Gauss-Lobatto-Legendre nodes, w_i the GLL weights (i = 0..N)
 *   D_im   = phi'_m(xi_i), the 1-D differentiation matrix (row-major D[i*n+m])
 *   local node (i,j,k) of element e is stored at e*n^3 + i + n*j + n*n*k
 *   (i = r direction fastest; SURVEY.md §8(c) reading G6)
 *   G      geometric factors [E][6][n^3] ordered rr, rs, rt, ss, st, tt with
 *          w_i w_j w_k J folded in (reading G3/G4)
 *
 * Pins (tests/test_oracle_*.py): GLL closed forms, sum w = 2, D exact on P_N,
 * SBP, affine closed-form factors, Kronecker closed form of A^e, A^e 1 = 0,
 * symmetry/PSD, assembled K against an independent Vandermonde route, exact
 * polynomial reproduction by CG, dense-matrix CG iteration counts.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_OK 0
#define ORA_EINVAL 1
#define ORA_ENOCONV 4

/* ------------------------------------------------------------------------- */
/* Legendre polynomial P_N(x) and P_{N-1}(x) by the three-term recurrence     */
/* (k+1) P_{k+1} = (2k+1) x P_k - k P_{k-1}.                                  */
static void legendre(int N, double x, double *pN, double *pNm1)
{
    double p0 = 1.0, p1 = x;
    if (N == 0) { *pN = 1.0; *pNm1 = 0.0; return; }
    for (int k = 1; k < N; ++k) {
        double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
        p0 = p1;
        p1 = p2;
    }
    *pN = p1;
    *pNm1 = p0;
}

/* O1.  GLL nodes and weights ("Gauss-Lobatto-Legendre nodes";
 * quadrature weights w_abc = w_a w_b w_c).
 * xi_0 = -1, xi_N = +1; interior nodes are the roots of P'_N, found by Newton's
 * method from -cos(pi i / N) on P'_N with P''_N from Legendre's ODE
 * (1-x^2) P'' = 2x P' - N(N+1) P.  Weights w_i = 2 / (N(N+1) P_N(xi_i)^2).   */
int ora_gll(int N, double *xi, double *w)
{
    if (N < 1 || N > 32 || !xi || !w) return ORA_EINVAL;
    xi[0] = -1.0;
    xi[N] = 1.0;
    for (int i = 1; i < N; ++i) {
        double x = -cos(M_PI * (double)i / (double)N);
        for (int it = 0; it < 100; ++it) {
            double p, pm1;
            legendre(N, x, &p, &pm1);
            double dp = N * (x * p - pm1) / (x * x - 1.0);          /* P'_N  */
            double d2p = (2.0 * x * dp - N * (N + 1.0) * p) / (1.0 - x * x); /* P''_N */
            double dx = dp / d2p;
            x -= dx;
            if (fabs(dx) < 1e-16) break;
        }
        xi[i] = x;
    }
    /* symmetrise: xi_{N-i} = -xi_i, and xi_{N/2} = 0 for even N */
    for (int i = 0; i < (N + 1) / 2; ++i) {
        double a = 0.5 * (xi[N - i] - xi[i]);
        xi[i] = -a;
        xi[N - i] = a;
    }
    if (N % 2 == 0) xi[N / 2] = 0.0;
    for (int i = 0; i <= N; ++i) {
        double p, pm1;
        legendre(N, xi[i], &p, &pm1);
        w[i] = 2.0 / (N * (N + 1.0) * p * p);
    }
    return ORA_OK;
}

/* O2.  Differentiation matrix D_im = phi'_m(xi_i) of the GLL Lagrange basis
 * (the phi' of PAPER.md:618-625).  Off-diagonal (textbook Lagrange-on-GLL):
 *   D_im = P_N(xi_i) / (P_N(xi_m) (xi_i - xi_m)),  i != m
 * Diagonal by the negative-sum rule D_ii = -sum_{m != i} D_im, so D 1 = 0
 * (reading G11).                                                              */
int ora_deriv(int N, const double *xi, double *D)
{
    if (N < 1 || N > 32 || !xi || !D) return ORA_EINVAL;
    int n = N + 1;
    double PN[33];
    for (int i = 0; i < n; ++i) {
        double pm1;
        legendre(N, xi[i], &PN[i], &pm1);
    }
    for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int m = 0; m < n; ++m) {
            if (m == i) continue;
            D[i * n + m] = PN[i] / (PN[m] * (xi[i] - xi[m]));
            s += D[i * n + m];
        }
        D[i * n + i] = -s;
    }
    return ORA_OK;
}

/* O3.  Geometric factors (PAPER.md:604 reference map x(r,s,t); :613 Jacobian;
 * :627-665 chain rule, G^ = G^T G "precomputed for each elemental node").
 * Isoparametric: X_r = (I x I x D) x, X_s = (I x D x I) x, X_t = (D x I x I) x at
 * each GLL node; J = det dX/dr; dr/dx = (dX/dr)^{-1} by the adjugate;
 * G_ab = w_i w_j w_k J sum_c (dr_a/dx_c)(dr_b/dx_c), a,b in {r,s,t}.
 * xyz is [E][3][n^3]; G is [E][6][n^3] (rr, rs, rt, ss, st, tt); J is [E][n^3]
 * (may be NULL).  Returns ORA_EINVAL if any J <= 0.                          */
int ora_geom(int N, int64_t E, const double *xyz, double *G, double *Jout)
{
    if (N < 1 || N > 32 || E < 0 || (E > 0 && (!xyz || !G))) return ORA_EINVAL;
    int n = N + 1, n3 = n * n * n;
    double xi[33], w[33];
    double *D = (double *)malloc(sizeof(double) * n * n);
    ora_gll(N, xi, w);
    ora_deriv(N, xi, D);
    int bad = 0;
    for (int64_t e = 0; e < E; ++e) {
        const double *X = xyz + e * 3 * n3;
        for (int k = 0; k < n; ++k)
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    int q = i + n * j + n * n * k;
                    double a[3][3]; /* a[c][d] = d x_c / d r_d */
                    for (int c = 0; c < 3; ++c) {
                        const double *Xc = X + c * n3;
                        double dr = 0.0, ds = 0.0, dt = 0.0;
                        for (int m = 0; m < n; ++m) {
                            dr += D[i * n + m] * Xc[m + n * j + n * n * k];
                            ds += D[j * n + m] * Xc[i + n * m + n * n * k];
                            dt += D[k * n + m] * Xc[i + n * j + n * n * m];
                        }
                        a[c][0] = dr;
                        a[c][1] = ds;
                        a[c][2] = dt;
                    }
                    double J = a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1])
                             - a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0])
                             + a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
                    if (!(J > 0.0)) bad = 1;
                    /* inverse: inv[d][c] = d r_d / d x_c = adj(a)[d][c] / J */
                    double inv[3][3];
                    inv[0][0] = (a[1][1] * a[2][2] - a[1][2] * a[2][1]) / J;
                    inv[0][1] = (a[0][2] * a[2][1] - a[0][1] * a[2][2]) / J;
                    inv[0][2] = (a[0][1] * a[1][2] - a[0][2] * a[1][1]) / J;
                    inv[1][0] = (a[1][2] * a[2][0] - a[1][0] * a[2][2]) / J;
                    inv[1][1] = (a[0][0] * a[2][2] - a[0][2] * a[2][0]) / J;
                    inv[1][2] = (a[0][2] * a[1][0] - a[0][0] * a[1][2]) / J;
                    inv[2][0] = (a[1][0] * a[2][1] - a[1][1] * a[2][0]) / J;
                    inv[2][1] = (a[0][1] * a[2][0] - a[0][0] * a[2][1]) / J;
                    inv[2][2] = (a[0][0] * a[1][1] - a[0][1] * a[1][0]) / J;
                    double scale = w[i] * w[j] * w[k] * J;
                    static const int pa[6] = {0, 0, 0, 1, 1, 2};
                    static const int pb[6] = {0, 1, 2, 1, 2, 2};
                    for (int f = 0; f < 6; ++f) {
                        double s = 0.0;
                        for (int c = 0; c < 3; ++c) s += inv[pa[f]][c] * inv[pb[f]][c];
                        G[e * 6 * n3 + f * n3 + q] = scale * s;
                    }
                    if (Jout) Jout[e * n3 + q] = J;
                }
    }
    free(D);
    return bad ? ORA_EINVAL : ORA_OK;
}

/* O4.  Local (unassembled, unmasked) stiffness apply w = A_L u (eq:semOperator,
 * PAPER.md:593-596, kappa = 1, alpha = 0; derivative sparsity :615-625; chain
 * rule and G^ :627-665; reading G4 A^e = D^T G^ D):
 *   u_r[ijk] = sum_m D_im u[mjk],  u_s[ijk] = sum_m D_jm u[imk],
 *   u_t[ijk] = sum_m D_km u[ijm]
 *   (f_r, f_s, f_t) = G^ (u_r, u_s, u_t)      (G^ symmetric, 6 factors)
 *   w[ijk] = sum_m D_mi f_r[mjk] + sum_m D_mj f_s[imk] + sum_m D_mk f_t[ijm]
 *
 * NEXT-1, the full screened-Coulomb operator of eq:semPDE (PAPER.md:580-586,
 * -div(kappa grad u) + alpha u = f) in the weak form eq:semOperator
 * (:593-596) = stiffness + mass:
 *   - kappa(x) weights the flux at each quadrature node (reading G2: the
 *     paper's u^ = kappa u at :664 is read as kappa multiplying G^ pointwise):
 *       (f_r, f_s, f_t) = kappa_ijk G^ (u_r, u_s, u_t)
 *   - the mass operator is the lumped diagonal J w_abc of :605-614, scaled by
 *     alpha(x) at the node:  w[ijk] += alpha_ijk w_i w_j w_k J_ijk u[ijk]
 * kappa == NULL means kappa = 1; alpha == NULL means alpha = 0 (J unused).  */
/* Host threads of the element loop of ora_ax_screened (default 1).  Only
 * the timing of the CPU baseline changes; results are bit-identical. */
static int ora_threads = 1;
int ora_set_threads(int nthreads)
{
    if (nthreads < 1) return ORA_EINVAL;
    ora_threads = nthreads;
    return ORA_OK;
}
int ora_get_threads(void) { return ora_threads; }

int ora_ax_screened(int N, int64_t E, const double *G, const double *J, const double *kappa,
                    const double *alpha, const double *u, double *w)
{
    if (N < 1 || N > 32 || E < 0 || (E > 0 && (!G || !u || !w))) return ORA_EINVAL;
    if (E > 0 && alpha && !J) return ORA_EINVAL;
    int n = N + 1, n3 = n * n * n;
    double xi[33], wq[33];
    double *D = (double *)malloc(sizeof(double) * n * n);
    ora_gll(N, xi, wq);
    ora_deriv(N, xi, D);
    /* Elements are independent (each w_e depends on u_e only), so the element
     * loop may run on several host threads (ora_set_threads; the CPU baseline
     * of bench.py): every w value is computed by the same operations in the
     * same order whatever the thread count -- bit-identical results. */
#pragma omp parallel num_threads(ora_threads)
    {
    double *fr = (double *)malloc(sizeof(double) * n3);
    double *fs = (double *)malloc(sizeof(double) * n3);
    double *ft = (double *)malloc(sizeof(double) * n3);
#pragma omp for schedule(static)
    for (int64_t e = 0; e < E; ++e) {
        const double *ue = u + e * n3;
        const double *Ge = G + e * 6 * n3;
        double *we = w + e * n3;
        for (int k = 0; k < n; ++k)
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    int q = i + n * j + n * n * k;
                    double ur = 0.0, us = 0.0, ut = 0.0;
                    for (int m = 0; m < n; ++m) {
                        ur += D[i * n + m] * ue[m + n * j + n * n * k];
                        us += D[j * n + m] * ue[i + n * m + n * n * k];
                        ut += D[k * n + m] * ue[i + n * j + n * n * m];
                    }
                    double grr = Ge[0 * n3 + q], grs = Ge[1 * n3 + q], grt = Ge[2 * n3 + q];
                    double gss = Ge[3 * n3 + q], gst = Ge[4 * n3 + q], gtt = Ge[5 * n3 + q];
                    fr[q] = grr * ur + grs * us + grt * ut;
                    fs[q] = grs * ur + gss * us + gst * ut;
                    ft[q] = grt * ur + gst * us + gtt * ut;
                    if (kappa) {
                        double kq = kappa[e * n3 + q];
                        fr[q] = kq * fr[q];
                        fs[q] = kq * fs[q];
                        ft[q] = kq * ft[q];
                    }
                }
        for (int k = 0; k < n; ++k)
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    double s = 0.0;
                    for (int m = 0; m < n; ++m) s += D[m * n + i] * fr[m + n * j + n * n * k];
                    for (int m = 0; m < n; ++m) s += D[m * n + j] * fs[i + n * m + n * n * k];
                    for (int m = 0; m < n; ++m) s += D[m * n + k] * ft[i + n * j + n * n * m];
                    int q = i + n * j + n * n * k;
                    if (alpha)
                        s += alpha[e * n3 + q] * (wq[i] * wq[j] * wq[k] * J[e * n3 + q]) * ue[q];
                    we[q] = s;
                }
    }
    free(fr);
    free(fs);
    free(ft);
    }
    free(D);
    return ORA_OK;
}

int ora_ax(int N, int64_t E, const double *G, const double *u, double *w)
{
    return ora_ax_screened(N, E, G, NULL, NULL, NULL, u, w);
}

/* ------------------------------------------------------------------------- */
/* NEXT-2.  Diagonal of the local operator, d[q] = (A^e)_qq
 * = e_q^T A^e e_q, for the Jacobi preconditioner of the PCG at PAPER.md:672-673
 * ("Besides the preconditioner choice").  Written from the definition of A^e
 * (eq:semOperator :593-596, reading G4, kappa / alpha as ora_ax_screened):
 * the reference gradient of the unit vector e_q, q = (i,j,k), at node p = (a,b,c)
 *     g_r(p) = sum_m D_am e_q[m,b,c] = D_ai  if (b,c) == (j,k), else 0
 *     g_s(p) = sum_m D_bm e_q[a,m,c] = D_bj  if (a,c) == (i,k), else 0
 *     g_t(p) = sum_m D_cm e_q[a,b,m] = D_ck  if (a,b) == (i,j), else 0
 * and (A^e)_qq = sum_p kappa_p g(p)^T G^(p) g(p) + alpha_q w_i w_j w_k J_q.
 * Nodes p off the three GLL lines through q have g(p) = 0 and are skipped.  */
int ora_diag_screened(int N, int64_t E, const double *G, const double *J, const double *kappa,
                      const double *alpha, double *d)
{
    if (N < 1 || N > 32 || E < 0 || (E > 0 && (!G || !d))) return ORA_EINVAL;
    if (E > 0 && alpha && !J) return ORA_EINVAL;
    int n = N + 1, n3 = n * n * n;
    double xi[33], wq[33];
    double *D = (double *)malloc(sizeof(double) * n * n);
    ora_gll(N, xi, wq);
    ora_deriv(N, xi, D);
    for (int64_t e = 0; e < E; ++e) {
        const double *Ge = G + e * 6 * n3;
        for (int k = 0; k < n; ++k)
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < n; ++i) {
                    double s = 0.0;
                    for (int c = 0; c < n; ++c)
                        for (int b = 0; b < n; ++b)
                            for (int a = 0; a < n; ++a) {
                                int onr = (b == j && c == k), ons = (a == i && c == k);
                                int ont = (a == i && b == j);
                                if (!onr && !ons && !ont) continue;
                                double gr = onr ? D[a * n + i] : 0.0;
                                double gs = ons ? D[b * n + j] : 0.0;
                                double gt = ont ? D[c * n + k] : 0.0;
                                int p = a + n * b + n * n * c;
                                double grr = Ge[0 * n3 + p], grs = Ge[1 * n3 + p];
                                double grt = Ge[2 * n3 + p], gss = Ge[3 * n3 + p];
                                double gst = Ge[4 * n3 + p], gtt = Ge[5 * n3 + p];
                                double fr = grr * gr + grs * gs + grt * gt;
                                double fs = grs * gr + gss * gs + gst * gt;
                                double ft = grt * gr + gst * gs + gtt * gt;
                                double t = gr * fr + gs * fs + gt * ft;
                                if (kappa) t = kappa[e * n3 + p] * t;
                                s += t;
                            }
                    int q = i + n * j + n * n * k;
                    if (alpha) s += alpha[e * n3 + q] * (wq[i] * wq[j] * wq[k] * J[e * n3 + q]);
                    d[e * n3 + q] = s;
                }
    }
    free(D);
    return ORA_OK;
}

/* ------------------------------------------------------------------------- */
/* O5.  Direct-stiffness summation v <- Q Q^T v (global-local numbering,
 * PAPER.md:667, Fischer 1991).  For each global id g, S_g = sum of its local
 * copies in ascending local-index order; S_g is written to every copy.       */
static const int64_t *cmp_glo;
static int cmp_by_glo(const void *pa, const void *pb)
{
    int64_t a = *(const int64_t *)pa, b = *(const int64_t *)pb;
    if (cmp_glo[a] != cmp_glo[b]) return cmp_glo[a] < cmp_glo[b] ? -1 : 1;
    return a < b ? -1 : (a > b);
}

/* order[L]: local indices sorted by (glo, local index) */
static int64_t *sorted_order(int64_t L, const int64_t *glo)
{
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (L > 0 ? L : 1));
    for (int64_t l = 0; l < L; ++l) order[l] = l;
    cmp_glo = glo;
    qsort(order, (size_t)L, sizeof(int64_t), cmp_by_glo);
    return order;
}

static void dssum_sorted(int64_t L, const int64_t *glo, const int64_t *order, double *v)
{
    int64_t a = 0;
    while (a < L) {
        int64_t b = a;
        double s = 0.0;
        while (b < L && glo[order[b]] == glo[order[a]]) { s += v[order[b]]; ++b; }
        for (int64_t t = a; t < b; ++t) v[order[t]] = s;
        a = b;
    }
}

int ora_dssum(int64_t L, const int64_t *glo, double *v)
{
    if (L < 0 || (L > 0 && (!glo || !v))) return ORA_EINVAL;
    int64_t *order = sorted_order(L, glo);
    dssum_sorted(L, glo, order, v);
    free(order);
    return ORA_OK;
}

/* Multiplicity m = Q Q^T 1. */
int ora_multiplicity(int64_t L, const int64_t *glo, double *m)
{
    if (L < 0 || (L > 0 && (!glo || !m))) return ORA_EINVAL;
    for (int64_t l = 0; l < L; ++l) m[l] = 1.0;
    return ora_dssum(L, glo, m);
}

/* ------------------------------------------------------------------------- */
/* O7.  Conjugate gradients (PCG of PAPER.md:672-673 with the identity
 * preconditioner, reading G8), Hestenes-Stiefel recurrence, SURVEY §8(c) O7:
 *   (a,b)_c = sum_L c_L a_L b_L,  c = mask / m                (reading G10)
 *   r = mask (b - Q Q^T A_L x0); rho = (r,r)_c; rho0 = rho; k = 0
 *   while k < maxit and sqrt(rho) > tol sqrt(rho0):           (reading G9)
 *     beta = (k == 0) ? 0 : rho / rho_old;  p = r + beta p
 *     w = mask Q Q^T A_L p;  alpha = rho / (w,p)_c
 *     x += alpha p;  r -= alpha w;  rho_old = rho;  rho = (r,r)_c;  k += 1
 * dirichlet[L]: 1 marks a Dirichlet node (mask 0).  x is in/out (x0 in).
 * Returns ORA_ENOCONV if maxit was reached with tol > 0 and not converged.   */
static double dot_c(int64_t L, const double *c, const double *a, const double *b)
{
    double s = 0.0;
    for (int64_t l = 0; l < L; ++l) s += c[l] * a[l] * b[l];
    return s;
}

/* Optional residual history of the next CG solves (test instrumentation, no
 * arithmetic): hist[k] = sqrt(rr_k) / sqrt(rr_0) for k = 0 .. iters, as far
 * as cap allows; NULL disables. */
static double *ora_hist = NULL;
static int ora_hist_cap = 0;
int ora_set_history(double *hist, int cap)
{
    ora_hist = (hist && cap > 0) ? hist : NULL;
    ora_hist_cap = ora_hist ? cap : 0;
    return ORA_OK;
}
static void hist_put(int k, double rr, double rr0)
{
    if (ora_hist && k < ora_hist_cap) ora_hist[k] = sqrt(rr) / sqrt(rr0);
}

/* the operator's coefficients (NULL: Poisson) */
typedef struct {
    const double *J, *kappa, *alpha;
} ora_coef;

static void apply_op(int N, int64_t E, const double *G, const ora_coef *cf, const int64_t *glo,
                     const int64_t *order, const double *mask, const double *in,
                     double *out)
{
    int64_t L = E * (N + 1) * (N + 1) * (N + 1);
    ora_ax_screened(N, E, G, cf->J, cf->kappa, cf->alpha, in, out);
    dssum_sorted(L, glo, order, out);
    for (int64_t l = 0; l < L; ++l) out[l] = mask[l] * out[l];
}

/* PCG on the screened-Coulomb operator: O7's recurrence with a
 * preconditioner M^{-1} ("PCG ... Besides the preconditioner
 * choice"; NEXT-2 of SURVEY.md §8(f)), preconditioned Hestenes-Stiefel:
 *   r = mask (b - Q Q^T A_L x0); z = M^{-1} r; rho = (r,z)_c; rr = (r,r)_c
 *   rr0 = rr; k = 0
 *   while k < maxit and sqrt(rr) > tol sqrt(rr0):            (reading G9, R4)
 *     beta = (k == 0) ? 0 : rho / rho_old;  p = z + beta p
 *     w = mask Q Q^T A_L p;  alpha = rho / (w,p)_c
 *     x += alpha p;  r -= alpha w;  z = M^{-1} r
 *     rho_old = rho;  rho = (r,z)_c;  rr = (r,r)_c;  k += 1
 * precond 0: M = I (z = r, rho = rr: exactly O7).
 * precond 1: Jacobi, M = diag of the assembled masked operator:
 *   M^{-1}_L = mask_L / (Q Q^T d)_L with d the local diagonal (ora_diag_screened)
 *   (0 at Dirichlet nodes, where r = 0 anyway).
 * The stopping rule stays on the residual norm (r,r)_c (reading R4).       */
int ora_pcg_screened(int N, int64_t E, const int64_t *glo, const uint8_t *dirichlet,
                     const double *G, const double *J, const double *kappa, const double *alpha,
                     int precond, const double *b, double *x, double tol, int maxit, int *iters,
                     double *rel_res)
{
    if (N < 1 || N > 32 || E < 0 || maxit < 0 || !(tol >= 0.0)) return ORA_EINVAL;
    if (alpha && !J) return ORA_EINVAL;
    if (precond != 0 && precond != 1) return ORA_EINVAL;
    const ora_coef cf = {J, kappa, alpha};
    int64_t L = E * (N + 1) * (N + 1) * (N + 1);
    double *mask = (double *)malloc(sizeof(double) * (L + 1));
    double *c = (double *)malloc(sizeof(double) * (L + 1));
    double *minv = (double *)malloc(sizeof(double) * (L + 1));
    double *r = (double *)malloc(sizeof(double) * (L + 1));
    double *z = (double *)malloc(sizeof(double) * (L + 1));
    double *p = (double *)malloc(sizeof(double) * (L + 1));
    double *w = (double *)malloc(sizeof(double) * (L + 1));
    int64_t *order = sorted_order(L, glo);
    for (int64_t l = 0; l < L; ++l) {
        mask[l] = dirichlet[l] ? 0.0 : 1.0;
        c[l] = 1.0;
    }
    dssum_sorted(L, glo, order, c);             /* c = multiplicity m */
    for (int64_t l = 0; l < L; ++l) c[l] = mask[l] / c[l];
    if (precond == 1) {
        ora_diag_screened(N, E, G, J, kappa, alpha, minv);   /* local diagonal d */
        dssum_sorted(L, glo, order, minv);                   /* Q Q^T d */
        for (int64_t l = 0; l < L; ++l) minv[l] = dirichlet[l] ? 0.0 : 1.0 / minv[l];
    }

    apply_op(N, E, G, &cf, glo, order, mask, x, w);  /* w = mask QQ^T A_L x0 */
    for (int64_t l = 0; l < L; ++l) r[l] = mask[l] * b[l] - w[l];
    for (int64_t l = 0; l < L; ++l) z[l] = (precond == 1) ? minv[l] * r[l] : r[l];
    for (int64_t l = 0; l < L; ++l) p[l] = 0.0;
    double rr = dot_c(L, c, r, r), rr0 = rr;
    double rho = dot_c(L, c, r, z), rho_old = 0.0;
    int k = 0;
    int status = ORA_OK;
    if (rr0 == 0.0) {
        *iters = 0;
        *rel_res = 0.0;
    } else {
        hist_put(0, rr, rr0);
        while (k < maxit && sqrt(rr) > tol * sqrt(rr0)) {
            double beta = (k == 0) ? 0.0 : rho / rho_old;
            for (int64_t l = 0; l < L; ++l) p[l] = z[l] + beta * p[l];
            apply_op(N, E, G, &cf, glo, order, mask, p, w);
            double alpha_k = rho / dot_c(L, c, w, p);
            for (int64_t l = 0; l < L; ++l) x[l] += alpha_k * p[l];
            for (int64_t l = 0; l < L; ++l) r[l] -= alpha_k * w[l];
            for (int64_t l = 0; l < L; ++l) z[l] = (precond == 1) ? minv[l] * r[l] : r[l];
            rho_old = rho;
            rho = dot_c(L, c, r, z);
            rr = dot_c(L, c, r, r);
            k += 1;
            hist_put(k, rr, rr0);
        }
        *iters = k;
        *rel_res = sqrt(rr) / sqrt(rr0);
        if (tol > 0.0 && sqrt(rr) > tol * sqrt(rr0)) status = ORA_ENOCONV;
    }
    free(mask);
    free(c);
    free(minv);
    free(r);
    free(z);
    free(p);
    free(w);
    free(order);
    return status;
}

/* NEXT-3: the single-reduction CG of Chronopoulos and Gear
 * (1989), a latency-hiding variant of the PCG of PAPER.md:672-673 (reading R7):
 * the operator is applied to the residual, A p is carried by the recurrence
 * s = w + beta s, and both inner products of an iteration, gamma = (r,u)_c and
 * delta = (w,u)_c, come from the same vectors (one reduction point):
 *   r = mask (b - Q Q^T A_L x0); u = r; w = mask Q Q^T A_L u
 *   gamma = (r,u)_c; delta = (w,u)_c; rr0 = (r,r)_c; k = 0
 *   while k < maxit and sqrt((r,r)_c) > tol sqrt(rr0):           (G9)
 *     if k == 0: beta = 0; alpha = gamma / delta
 *     else:      beta = gamma / gamma_old; alpha = gamma / (delta - beta gamma / alpha_old)
 *     p = u + beta p;  s = w + beta s;  x += alpha p;  r -= alpha s
 *     u = r;  w = mask Q Q^T A_L u
 *     gamma_old = gamma; alpha_old = alpha; gamma = (r,u)_c; delta = (w,u)_c; k += 1
 * (identity preconditioner: u = r, gamma = (r,r)_c).  Returns as ora_cg.      */
int ora_cg_cgs(int N, int64_t E, const int64_t *glo, const uint8_t *dirichlet, const double *G,
               const double *b, double *x, double tol, int maxit, int *iters, double *rel_res)
{
    if (N < 1 || N > 32 || E < 0 || maxit < 0 || !(tol >= 0.0)) return ORA_EINVAL;
    const ora_coef cf = {NULL, NULL, NULL};
    int64_t L = E * (N + 1) * (N + 1) * (N + 1);
    double *mask = (double *)malloc(sizeof(double) * (L + 1));
    double *c = (double *)malloc(sizeof(double) * (L + 1));
    double *r = (double *)malloc(sizeof(double) * (L + 1));
    double *u = (double *)malloc(sizeof(double) * (L + 1));
    double *w = (double *)malloc(sizeof(double) * (L + 1));
    double *p = (double *)malloc(sizeof(double) * (L + 1));
    double *sv = (double *)malloc(sizeof(double) * (L + 1));
    int64_t *order = sorted_order(L, glo);
    for (int64_t l = 0; l < L; ++l) {
        mask[l] = dirichlet[l] ? 0.0 : 1.0;
        c[l] = 1.0;
    }
    dssum_sorted(L, glo, order, c);
    for (int64_t l = 0; l < L; ++l) c[l] = mask[l] / c[l];

    apply_op(N, E, G, &cf, glo, order, mask, x, w);   /* w = mask QQ^T A_L x0 */
    for (int64_t l = 0; l < L; ++l) r[l] = mask[l] * b[l] - w[l];
    for (int64_t l = 0; l < L; ++l) u[l] = r[l];
    apply_op(N, E, G, &cf, glo, order, mask, u, w);   /* w = mask QQ^T A_L u */
    for (int64_t l = 0; l < L; ++l) p[l] = 0.0;
    for (int64_t l = 0; l < L; ++l) sv[l] = 0.0;
    double gamma = dot_c(L, c, r, u), delta = dot_c(L, c, w, u);
    double rr = dot_c(L, c, r, r), rr0 = rr;
    double gamma_old = 0.0, alpha_old = 0.0;
    int k = 0;
    int status = ORA_OK;
    if (rr0 == 0.0) {
        *iters = 0;
        *rel_res = 0.0;
    } else {
        hist_put(0, rr, rr0);
        while (k < maxit && sqrt(rr) > tol * sqrt(rr0)) {
            double beta, alpha;
            if (k == 0) {
                beta = 0.0;
                alpha = gamma / delta;
            } else {
                beta = gamma / gamma_old;
                alpha = gamma / (delta - beta * gamma / alpha_old);
            }
            for (int64_t l = 0; l < L; ++l) p[l] = u[l] + beta * p[l];
            for (int64_t l = 0; l < L; ++l) sv[l] = w[l] + beta * sv[l];
            for (int64_t l = 0; l < L; ++l) x[l] += alpha * p[l];
            for (int64_t l = 0; l < L; ++l) r[l] -= alpha * sv[l];
            for (int64_t l = 0; l < L; ++l) u[l] = r[l];
            apply_op(N, E, G, &cf, glo, order, mask, u, w);
            gamma_old = gamma;
            alpha_old = alpha;
            gamma = dot_c(L, c, r, u);
            delta = dot_c(L, c, w, u);
            rr = dot_c(L, c, r, r);
            k += 1;
            hist_put(k, rr, rr0);
        }
        *iters = k;
        *rel_res = sqrt(rr) / sqrt(rr0);
        if (tol > 0.0 && sqrt(rr) > tol * sqrt(rr0)) status = ORA_ENOCONV;
    }
    free(mask);
    free(c);
    free(r);
    free(u);
    free(w);
    free(p);
    free(sv);
    free(order);
    return status;
}

/* CG on the screened-Coulomb operator (NEXT-1): O7, the identity-preconditioned
 * case of ora_pcg_screened.  ora_cg is the Poisson case. */
int ora_cg_screened(int N, int64_t E, const int64_t *glo, const uint8_t *dirichlet,
                    const double *G, const double *J, const double *kappa, const double *alpha,
                    const double *b, double *x, double tol, int maxit, int *iters,
                    double *rel_res)
{
    return ora_pcg_screened(N, E, glo, dirichlet, G, J, kappa, alpha, 0, b, x, tol, maxit,
                            iters, rel_res);
}

int ora_cg(int N, int64_t E, const int64_t *glo, const uint8_t *dirichlet,
           const double *G, const double *b, double *x, double tol, int maxit,
           int *iters, double *rel_res)
{
    return ora_cg_screened(N, E, glo, dirichlet, G, NULL, NULL, NULL, b, x, tol, maxit, iters,
                           rel_res);
}
