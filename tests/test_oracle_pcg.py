"""Pins for the oracle's Jacobi-preconditioned CG (NEXT-2):
PCG of PAPER.md:672-673 ("Besides the preconditioner choice") with M = the
diagonal of the assembled masked operator.

Pinned by: the local diagonal against brute-force unit-vector probing of the
element operator and against the Kronecker closed form on an affine box; the
assembled diagonal Q Q^T d against the diagonal of the dense assembled K of the
independent physical-gradient route (Poisson and screened, variable kappa,
alpha); the PCG iteration count against a dense textbook PCG with diag(K);
agreement with numpy.linalg.solve; exact polynomial reproduction.
"""
import numpy as np
import pytest

from paper_1403_0968_b200 import meshgen
from tests import _indep


def _probe_diag(oracle, N, G, J=None, kappa=None, alpha=None):
    """(A^e)_qq by applying the oracle's Ax to unit vectors, element by element."""
    n3 = (N + 1) ** 3
    E = G.shape[0]
    d = np.zeros(E * n3)
    for e in range(E):
        sl = slice(e * n3, (e + 1) * n3)
        co = {k: (None if v is None else v.reshape(-1)[sl])
              for k, v in (("J", J), ("kappa", kappa), ("alpha", alpha))}
        for q in range(n3):
            u = np.zeros(n3)
            u[q] = 1.0
            d[e * n3 + q] = oracle.ax(N, G[e:e + 1], u, **co)[q]
    return d


@pytest.mark.parametrize("N,eps,screened", [(1, 0.0, False), (3, 0.05, False),
                                            (4, 0.05, True), (6, 0.1, True)])
def test_diag_matches_unit_vector_probe(oracle, N, eps, screened):
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(2, 1, 1), eps=eps)
    G, J = oracle.geom(N, m.xyz)
    co = {}
    if screened:
        kappa, alpha = meshgen.coefficients(m)
        co = {"J": J, "kappa": kappa, "alpha": alpha}
    d = oracle.diag(N, G, **co)
    ref = _probe_diag(oracle, N, G, **co)
    np.testing.assert_allclose(d, ref, rtol=1e-13, atol=1e-15 * np.abs(ref).max())


@pytest.mark.parametrize("N", [2, 4, 7])
def test_diag_kronecker_closed_form(oracle, N):
    """Affine box hx x hy x hz: diag(A^e)_{ijk} = (hy hz/2hx) w_k w_j K1_ii
    + (hx hz/2hy) w_k K1_jj w_i + (hx hy/2hz) K1_kk w_j w_i (K1 from the
    independent Vandermonde route)."""
    hx, hy, hz = 2.0, 0.5, 1.5
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(1, 1, 1), lengths=(hx, hy, hz))
    G, J = oracle.geom(N, m.xyz)
    xin, wn = _indep.gll_numpy(N)
    k1 = np.diag(_indep.stiffness_1d(xin, wn))
    ref = ((hy * hz / (2 * hx)) * np.einsum("k,j,i->kji", wn, wn, k1)
           + (hx * hz / (2 * hy)) * np.einsum("k,j,i->kji", wn, k1, wn)
           + (hx * hy / (2 * hz)) * np.einsum("k,j,i->kji", k1, wn, wn)).reshape(-1)
    np.testing.assert_allclose(oracle.diag(N, G), ref, rtol=1e-13)


@pytest.mark.parametrize("N,elems,eps,screened", [(2, (2, 2, 2), 0.05, False),
                                                  (3, (2, 1, 2), 0.05, True),
                                                  (5, (1, 2, 1), 0.1, True)])
def test_assembled_diag_independent_route(oracle, N, elems, eps, screened):
    """Q Q^T d equals diag(K) of the dense physical-gradient assembly."""
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    G, J = oracle.geom(N, m.xyz)
    n3 = (N + 1) ** 3
    co, kap, alp = {}, None, None
    if screened:
        kap, alp = meshgen.coefficients(m)
        co = {"J": J, "kappa": kap, "alpha": alp}
    d = oracle.dssum(m.glo, oracle.diag(N, G, **co))
    xin, wn = _indep.gll_numpy(N)
    mats = []
    for e in range(m.nelem):
        ke = None if kap is None else kap.reshape(-1, n3)[e]
        ae = None if alp is None else alp.reshape(-1, n3)[e]
        mats.append(_indep.element_stiffness_physical(m.xyz[e], xin, wn, ke, ae)[0])
    K = _indep.assemble_dense(mats, m.glo, m.nglobal)
    g = m.glo.reshape(-1)
    np.testing.assert_allclose(d, np.diag(K)[g], rtol=1e-11)


def _system(oracle, N, elems, eps, screened=False, rhs="sin"):
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    G, J = oracle.geom(N, m.xyz)
    co = {}
    if screened:
        kappa, alpha = meshgen.coefficients(m)
        co = {"J": J, "kappa": kappa, "alpha": alpha}
    us, f = meshgen.cube_poly(m) if rhs == "poly" else meshgen.manufactured(m)
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)
    return m, G, J, co, b, us


@pytest.mark.parametrize("N,elems,eps,screened", [(4, (2, 2, 2), 0.05, False),
                                                  (3, (3, 2, 2), 0.05, False),
                                                  (3, (2, 2, 2), 0.05, True)])
def test_pcg_matches_dense_pcg(oracle, N, elems, eps, screened):
    """Jacobi PCG on local storage takes exactly the iterations of a textbook
    dense PCG with minv = 1/diag(K) on the masked assembled K (independent
    route) and agrees with numpy.linalg.solve; it needs fewer iterations than
    plain CG on the deformed mesh."""
    m, G, J, co, b, _ = _system(oracle, N, elems, eps, screened)
    x, its, rel, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=1000,
                                precond="jacobi", **co)
    assert st == 0 and rel <= 1e-8
    _, its_cg, _, _ = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=1000, **co)
    assert its < its_cg
    n3 = (N + 1) ** 3
    xin, wn = _indep.gll_numpy(N)
    mats = []
    for e in range(m.nelem):
        ke = None if "kappa" not in co else co["kappa"].reshape(-1, n3)[e]
        ae = None if "alpha" not in co else co["alpha"].reshape(-1, n3)[e]
        mats.append(_indep.element_stiffness_physical(m.xyz[e], xin, wn, ke, ae)[0])
    K = _indep.assemble_dense(mats, m.glo, m.nglobal)
    g = m.glo.reshape(-1)
    interior = np.ones(m.nglobal, dtype=bool)
    interior[np.unique(g[m.dirichlet.reshape(-1) == 1])] = False
    bg = np.zeros(m.nglobal)
    bg[g] = b
    Ki = K[np.ix_(interior, interior)]
    xd, its_d = _indep.dense_pcg(Ki, bg[interior], 1.0 / np.diag(Ki), 1e-8, 1000)
    assert its == its_d
    xg = np.zeros(m.nglobal)
    xg[g] = x
    xs = np.linalg.solve(Ki, bg[interior])
    assert np.linalg.norm(xg[interior] - xs) <= 1e-6 * np.linalg.norm(xs)
    np.testing.assert_allclose(xg[interior], xd, rtol=0, atol=1e-10 * np.abs(xd).max())
    np.testing.assert_array_equal(x, xg[g])
    assert np.all(x[m.dirichlet.reshape(-1) == 1] == 0.0)


def test_pcg_polynomial_reproduction(oracle):
    """u* = x(1-x)y(1-y)z(1-z) in V_N: Jacobi PCG reproduces it at the nodes."""
    m, G, J, co, b, us = _system(oracle, 4, (2, 2, 2), 0.0, rhs="poly")
    x, its, rel, st = oracle.cg(4, m.glo, m.dirichlet, G, b, tol=1e-14, maxit=500,
                                precond="jacobi")
    assert st == 0
    assert np.max(np.abs(x - us)) <= 1e-13


def test_pcg_edge_cases(oracle):
    m, G, J, co, b, _ = _system(oracle, 3, (2, 2, 2), 0.05)
    x, its, rel, st = oracle.cg(3, m.glo, m.dirichlet, G, np.zeros_like(b), tol=1e-8,
                                maxit=10, precond="jacobi")
    assert its == 0 and rel == 0.0 and st == 0 and not x.any()
    x, its, rel, st = oracle.cg(3, m.glo, m.dirichlet, G, b, tol=1e-12, maxit=5,
                                precond="jacobi")
    assert its == 5 and st == 4
    x, its, rel, st = oracle.cg(3, m.glo, m.dirichlet, G, b, tol=0.0, maxit=7,
                                precond="jacobi")
    assert its == 7 and st == 0
