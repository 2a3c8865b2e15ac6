"""Pins for the oracle's screened-Coulomb operator (NEXT-1):
eq:semPDE -div(kappa grad u) + alpha u = f, weak form
eq:semOperator = stiffness + mass (:593-596), lumped mass J w_abc (:605-614),
kappa weighting the flux pointwise (reading G2).

Pinned by: the Kronecker closed form with constant kappa, alpha (stiffness
scaled by kappa plus alpha J M(x)M(x)M); the dense assembled operator against the
independent physical-gradient route with variable kappa(x), alpha(x);
A 1 = alpha w J (stiffness annihilates constants, mass is diagonal); CG with
alpha > 0 and no Dirichlet nodes against dense CG / numpy.linalg.solve.
"""
import numpy as np
import pytest

from paper_1403_0968_b200 import meshgen
from tests import _indep


def _element_matrix(oracle, N, G1, J1, kappa1, alpha1):
    n3 = (N + 1) ** 3
    A = np.zeros((n3, n3))
    for q in range(n3):
        e = np.zeros(n3)
        e[q] = 1.0
        A[:, q] = oracle.ax(N, G1, e, J=J1, kappa=kappa1, alpha=alpha1)
    return A


@pytest.mark.parametrize("N", [1, 2, 3, 5])
def test_screened_kronecker_closed_form(oracle, N):
    """Affine box, constant kappa0, alpha0:
    A^e = kappa0 [(hy hz/2hx) M(x)M(x)K1 + (hx hz/2hy) M(x)K1(x)M + (hx hy/2hz) K1(x)M(x)M]
          + alpha0 (hx hy hz / 8) M(x)M(x)M."""
    hx, hy, hz = 2.0, 0.5, 1.5
    kappa0, alpha0 = 1.7, 0.6
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(1, 1, 1), lengths=(hx, hy, hz))
    G, J = oracle.geom(N, m.xyz)
    n3 = (N + 1) ** 3
    A = _element_matrix(oracle, N, G, J, np.full(n3, kappa0), np.full(n3, alpha0))
    xin, wn = _indep.gll_numpy(N)
    K1 = _indep.stiffness_1d(xin, wn)
    M = np.diag(wn)
    ref = kappa0 * ((hy * hz / (2 * hx)) * np.kron(M, np.kron(M, K1))
                    + (hx * hz / (2 * hy)) * np.kron(M, np.kron(K1, M))
                    + (hx * hy / (2 * hz)) * np.kron(K1, np.kron(M, M))) \
        + alpha0 * (hx * hy * hz / 8) * np.kron(M, np.kron(M, M))
    assert np.max(np.abs(A - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("N,elems,eps", [(2, (2, 2, 2), 0.05), (3, (2, 1, 2), 0.05),
                                         (5, (1, 1, 1), 0.1)])
def test_screened_assembled_independent_route(oracle, N, elems, eps):
    """K = sum_e Q_e^T A^e Q_e (oracle local operator) equals the dense
    physical-gradient assembly of (kappa grad u, grad v) + (alpha u, v) with a
    Vandermonde basis, for variable kappa(x), alpha(x)."""
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    kappa, alpha = meshgen.coefficients(m)
    n3 = (N + 1) ** 3
    G, J = oracle.geom(N, m.xyz)
    kap = kappa.reshape(-1, n3)
    alp = alpha.reshape(-1, n3)
    U = m.nglobal
    K_or = np.zeros((U, U))
    for e in range(m.nelem):
        A = _element_matrix(oracle, N, G[e:e + 1], J[e], kap[e], alp[e])
        g = m.glo[e]
        K_or[np.ix_(g, g)] += A
    xin, wn = _indep.gll_numpy(N)
    mats = [_indep.element_stiffness_physical(m.xyz[e], xin, wn, kappa=kap[e], alpha=alp[e])[0]
            for e in range(m.nelem)]
    K_ind = _indep.assemble_dense(mats, m.glo, U)
    scale = np.max(np.abs(K_ind))
    assert np.max(np.abs(K_or - K_ind)) <= 1e-12 * scale
    # with alpha > 0 the unmasked operator is SPD
    assert np.linalg.eigvalsh(0.5 * (K_or + K_or.T))[0] > 0


@pytest.mark.parametrize("N", [3, 6])
def test_screened_constants_and_kappa_scaling(oracle, N):
    """A 1 = alpha w_i w_j w_k J (the stiffness part annihilates constants), and
    with constant kappa = c, alpha = 0 the operator is c times the Poisson one."""
    xi, w = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(2, 2, 1), eps=0.08)
    kappa, alpha = meshgen.coefficients(m)
    G, J = oracle.geom(N, m.xyz)
    w3 = np.einsum("k,j,i->kji", w, w, w).reshape(-1)
    ones = np.ones(m.nlocal)
    got = oracle.ax(N, G, ones, J=J, kappa=kappa, alpha=alpha)
    ref = alpha * (J * w3[None]).reshape(-1)
    assert np.max(np.abs(got - ref)) <= 1e-12 * (np.max(np.abs(G)) + np.max(np.abs(ref)))
    u = meshgen.random_field(m.nlocal, 3)
    c = 2.5
    a1 = oracle.ax(N, G, u, J=J, kappa=np.full(m.nlocal, c))
    a0 = oracle.ax(N, G, u)
    assert np.max(np.abs(a1 - c * a0)) <= 1e-13 * np.max(np.abs(a1))


@pytest.mark.parametrize("N,elems", [(2, (2, 2, 2)), (4, (2, 1, 1))])
def test_screened_cg_matches_dense(oracle, N, elems):
    """alpha > 0, no Dirichlet nodes: the oracle CG (O7 recurrence on the
    screened operator) reproduces dense CG's iteration count on the assembled
    K (independent route) and numpy.linalg.solve's solution."""
    xi, w = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=0.05, dirichlet_faces=False)
    kappa, alpha = meshgen.coefficients(m, alpha0=2.0)
    n3 = (N + 1) ** 3
    G, J = oracle.geom(N, m.xyz)
    _, f = meshgen.manufactured(m)
    f = f + 1.0
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)
    x, its, rel, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-10, maxit=500,
                                J=J, kappa=kappa, alpha=alpha)
    assert st == 0
    xin, wn = _indep.gll_numpy(N)
    kap, alp = kappa.reshape(-1, n3), alpha.reshape(-1, n3)
    mats = [_indep.element_stiffness_physical(m.xyz[e], xin, wn, kappa=kap[e], alpha=alp[e])[0]
            for e in range(m.nelem)]
    K = _indep.assemble_dense(mats, m.glo, m.nglobal)
    bg = np.zeros(m.nglobal)
    bg[m.glo.reshape(-1)] = b
    xs = np.linalg.solve(K, bg)
    # the global CG in the (.,.)_c inner product is the dense CG on K
    _, its_dense = _indep.dense_cg(K, bg, 1e-10, 500)
    assert abs(its - its_dense) <= 1
    assert np.max(np.abs(x - xs[m.glo.reshape(-1)])) <= 1e-8 * np.max(np.abs(xs))
