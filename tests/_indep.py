"""Independent routes used to PIN the oracle (test code only).

Nothing here calls the oracle's arithmetic; each helper recomputes a quantity
by a different route so that a dropped term, wrong sign/index or transposed
operand in oracle/sem_oracle.c fails a comparison:

* GLL nodes from numpy's Legendre-series root finder (roots of P'_N).
* The 1-D Lagrange basis in MONOMIAL form via the Vandermonde matrix
  (not the O2 closed formula), so its derivative matrix is independent.
* Element stiffness in the PHYSICAL-gradient form
      A^e = sum_c (Grad_c)^T diag(w J) Grad_c,
      Grad_c = sum_a diag(dr_a/dx_c) D_a
  with dr/dx from numpy.linalg.inv, instead of the oracle's D^T G^ D with six
  folded factors.
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as npleg


def gll_numpy(N: int):
    """Nodes: -1, roots of P'_N (numpy), +1.  Weights 2/(N(N+1)P_N^2)."""
    cN = np.zeros(N + 1)
    cN[N] = 1.0
    inner = np.sort(npleg.legroots(npleg.legder(cN))) if N > 1 else np.array([])
    xi = np.concatenate([[-1.0], np.real(inner), [1.0]])
    PN = npleg.legval(xi, cN)
    w = 2.0 / (N * (N + 1) * PN ** 2)
    return xi, w


def lagrange_monomial(xi):
    """C[p, a]: phi_a(x) = sum_p C[p, a] x^p (inverse Vandermonde)."""
    n = len(xi)
    V = np.vander(xi, n, increasing=True)  # V[q, p] = xi_q^p
    return np.linalg.inv(V)


def deriv_vandermonde(xi):
    """Dv[q, a] = phi_a'(xi_q) from the monomial coefficients."""
    n = len(xi)
    C = lagrange_monomial(xi)
    P = np.zeros((n, n))
    for p in range(1, n):
        P[:, p] = p * xi ** (p - 1)
    return P @ C


def stiffness_1d(xi, w):
    """K1[a, b] = sum_q w_q phi_a'(xi_q) phi_b'(xi_q) (exact on GLL)."""
    Dv = deriv_vandermonde(xi)
    return Dv.T @ np.diag(w) @ Dv


def ref_grad_ops(Dv):
    n = Dv.shape[0]
    I = np.eye(n)
    Dr = np.kron(I, np.kron(I, Dv))   # acts on i (fastest)
    Ds = np.kron(I, np.kron(Dv, I))   # acts on j
    Dt = np.kron(Dv, np.kron(I, I))   # acts on k
    return Dr, Ds, Dt


def element_stiffness_physical(xyz_e, xi, w, kappa=None, alpha=None):
    """Dense n^3 x n^3 element stiffness by the physical-gradient route.
    xyz_e: [3, n^3] node coordinates.  Returns (A, J).
    kappa / alpha ([n^3], optional): the screened-Coulomb element matrix
        sum_c Grad_c^T diag(w J kappa) Grad_c + diag(w J alpha)
    (quadrature of (kappa grad u, grad v) + (alpha u, v) at the GLL nodes)."""
    n = len(xi)
    Dv = deriv_vandermonde(xi)
    Dr, Ds, Dt = ref_grad_ops(Dv)
    ops = (Dr, Ds, Dt)
    # jac[q, c, a] = d x_c / d r_a
    jac = np.zeros((n ** 3, 3, 3))
    for c in range(3):
        for a in range(3):
            jac[:, c, a] = ops[a] @ xyz_e[c]
    J = np.linalg.det(jac)
    inv = np.linalg.inv(jac)          # inv[q, a, c] = d r_a / d x_c
    w3 = np.einsum("k,j,i->kji", w, w, w).reshape(-1)
    A = np.zeros((n ** 3, n ** 3))
    wk = w3 * J if kappa is None else w3 * J * np.asarray(kappa)
    for c in range(3):
        Gc = sum(inv[:, a, c][:, None] * ops[a] for a in range(3))
        A += Gc.T @ (wk[:, None] * Gc)
    if alpha is not None:
        A += np.diag(w3 * J * np.asarray(alpha))
    return A, J


def assemble_dense(elem_mats, glo, nglobal):
    """K = sum_e Q_e^T A^e Q_e with Q_e the 0/1 scatter of element e."""
    K = np.zeros((nglobal, nglobal))
    for e, A in enumerate(elem_mats):
        g = glo[e]
        K[np.ix_(g, g)] += A
    return K


def dense_cg(K, b, tol, maxit):
    """Textbook CG on a dense SPD matrix (same stopping rule as O7)."""
    x = np.zeros_like(b)
    r = b.copy()
    rho = r @ r
    rho0 = rho
    p = np.zeros_like(b)
    k = 0
    rho_old = 0.0
    while k < maxit and np.sqrt(rho) > tol * np.sqrt(rho0):
        beta = 0.0 if k == 0 else rho / rho_old
        p = r + beta * p
        q = K @ p
        alpha = rho / (q @ p)
        x = x + alpha * p
        r = r - alpha * q
        rho_old = rho
        rho = r @ r
        k += 1
    return x, k


def dense_pcg(K, b, minv, tol, maxit):
    """Textbook preconditioned CG on a dense SPD matrix with a diagonal
    preconditioner minv (vector); stopping rule on the residual norm r.r
    (same as the oracle's reading R4)."""
    x = np.zeros_like(b)
    r = b.copy()
    z = minv * r
    rho = r @ z
    rr0 = r @ r
    rr = rr0
    p = np.zeros_like(b)
    k = 0
    rho_old = 0.0
    while k < maxit and np.sqrt(rr) > tol * np.sqrt(rr0):
        beta = 0.0 if k == 0 else rho / rho_old
        p = z + beta * p
        q = K @ p
        alpha = rho / (q @ p)
        x = x + alpha * p
        r = r - alpha * q
        z = minv * r
        rho_old = rho
        rho = r @ z
        rr = r @ r
        k += 1
    return x, k


def dense_cg_single_reduction(K, b, tol, maxit):
    """Textbook Chronopoulos-Gear CG on a dense SPD matrix (same stopping
    rule on r.r as the oracle's reading G9)."""
    x = np.zeros_like(b)
    r = b.copy()
    u = r.copy()
    w = K @ u
    gamma, delta = r @ u, w @ u
    rr0 = r @ r
    rr = rr0
    p = np.zeros_like(b)
    s = np.zeros_like(b)
    k = 0
    gamma_old = alpha_old = 0.0
    while k < maxit and np.sqrt(rr) > tol * np.sqrt(rr0):
        if k == 0:
            beta, alpha = 0.0, gamma / delta
        else:
            beta = gamma / gamma_old
            alpha = gamma / (delta - beta * gamma / alpha_old)
        p = u + beta * p
        s = w + beta * s
        x = x + alpha * p
        r = r - alpha * s
        u = r.copy()
        w = K @ u
        gamma_old, alpha_old = gamma, alpha
        gamma, delta, rr = r @ u, w @ u, r @ r
        k += 1
    return x, k
