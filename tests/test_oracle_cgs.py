"""Pins for the oracle's single-reduction (Chronopoulos-Gear) CG (NEXT-3,
SURVEY.md §8(f); a latency-hiding variant of the PCG of PAPER.md:672-673,
reading R7).  Pinned by: the iteration count and iterates of a dense textbook
Chronopoulos-Gear CG on the masked assembled K of the independent route;
numpy.linalg.solve; exact polynomial reproduction; the iterates of standard
CG (the recurrences are algebraically identical: after a few iterations the
two agree to rounding); edge cases."""
import numpy as np
import pytest

from paper_1403_0968_b200 import meshgen
from tests import _indep


def _system(oracle, N, elems, eps, rhs="sin"):
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    G, J = oracle.geom(N, m.xyz)
    us, f = meshgen.cube_poly(m) if rhs == "poly" else meshgen.manufactured(m)
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)
    return m, G, J, b, us


@pytest.mark.parametrize("N,elems,eps", [(4, (2, 2, 2), 0.05), (3, (3, 2, 2), 0.05),
                                         (2, (3, 3, 2), 0.0)])
def test_cgs_matches_dense_cgs(oracle, N, elems, eps):
    m, G, J, b, _ = _system(oracle, N, elems, eps)
    x, its, rel, st = oracle.cg_single_reduction(N, m.glo, m.dirichlet, G, b, tol=1e-8,
                                                 maxit=1000)
    assert st == 0 and rel <= 1e-8
    xin, wn = _indep.gll_numpy(N)
    mats = [_indep.element_stiffness_physical(m.xyz[e], xin, wn)[0] for e in range(m.nelem)]
    K = _indep.assemble_dense(mats, m.glo, m.nglobal)
    g = m.glo.reshape(-1)
    interior = np.ones(m.nglobal, dtype=bool)
    interior[np.unique(g[m.dirichlet.reshape(-1) == 1])] = False
    bg = np.zeros(m.nglobal)
    bg[g] = b
    Ki = K[np.ix_(interior, interior)]
    xd, its_d = _indep.dense_cg_single_reduction(Ki, bg[interior], 1e-8, 1000)
    assert its == its_d
    xg = np.zeros(m.nglobal)
    xg[g] = x
    np.testing.assert_allclose(xg[interior], xd, rtol=0, atol=1e-10 * np.abs(xd).max())
    xs = np.linalg.solve(Ki, bg[interior])
    assert np.linalg.norm(xg[interior] - xs) <= 1e-6 * np.linalg.norm(xs)
    np.testing.assert_array_equal(x, xg[g])


@pytest.mark.parametrize("N,elems,eps", [(4, (2, 2, 2), 0.05), (5, (2, 2, 1), 0.1)])
def test_cgs_tracks_standard_cg(oracle, N, elems, eps):
    """Same Krylov iterates in exact arithmetic: after 10 iterations the two
    x agree far below the residual level, and the converged counts differ by
    at most one."""
    m, G, J, b, _ = _system(oracle, N, elems, eps)
    x1, _, r1, _ = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=0.0, maxit=10)
    x2, _, r2, _ = oracle.cg_single_reduction(N, m.glo, m.dirichlet, G, b, tol=0.0, maxit=10)
    assert np.linalg.norm(x1 - x2) <= 1e-10 * np.linalg.norm(x1)
    assert abs(r1 - r2) <= 1e-8 * r1
    _, i1, _, _ = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=1000)
    _, i2, _, _ = oracle.cg_single_reduction(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=1000)
    assert abs(i1 - i2) <= 1


def test_cgs_polynomial_reproduction(oracle):
    m, G, J, b, us = _system(oracle, 4, (2, 2, 2), 0.0, "poly")
    x, its, rel, st = oracle.cg_single_reduction(4, m.glo, m.dirichlet, G, b, tol=1e-14,
                                                 maxit=500)
    assert st == 0
    assert np.max(np.abs(x - us)) <= 1e-13


def test_cgs_edge_cases(oracle):
    m, G, J, b, _ = _system(oracle, 3, (2, 2, 2), 0.05)
    x, its, rel, st = oracle.cg_single_reduction(3, m.glo, m.dirichlet, G, np.zeros_like(b),
                                                 tol=1e-8, maxit=10)
    assert its == 0 and rel == 0.0 and st == 0 and not x.any()
    x, its, rel, st = oracle.cg_single_reduction(3, m.glo, m.dirichlet, G, b, tol=1e-12, maxit=5)
    assert its == 5 and st == 4
    x, its, rel, st = oracle.cg_single_reduction(3, m.glo, m.dirichlet, G, b, tol=0.0, maxit=7)
    assert its == 7 and st == 0
    x1, _, _, _ = oracle.cg_single_reduction(3, m.glo, m.dirichlet, G, b, tol=1e-10, maxit=500)
    x2, its2, _, _ = oracle.cg_single_reduction(3, m.glo, m.dirichlet, G, b, x0=x1, tol=1e-3,
                                                maxit=500)
    assert np.max(np.abs(x2 - x1)) <= 1e-9 * np.max(np.abs(x1))
