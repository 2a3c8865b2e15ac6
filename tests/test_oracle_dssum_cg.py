"""Pins for oracle O5 (DSSUM = Q Q^T) and O7 (CG).

PAPER.md:667 (global-local numbering, Fischer 1991) and :672-673 (PCG).
Pinned by: multiplicities of the box topology; DSSUM of continuous fields;
a dense 0/1 Q brute force; virtual-partition independence; exact polynomial
reproduction; a dense-matrix CG with the same stopping rule; a direct solve.
"""
import numpy as np
import pytest

from paper_1403_0968_b200 import meshgen
from tests import _indep


@pytest.mark.parametrize("N,elems", [(1, (2, 2, 2)), (3, (3, 2, 2)), (4, (2, 2, 2))])
def test_multiplicity_box_topology(oracle, N, elems):
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems)
    mult = oracle.multiplicity(m.glo)
    assert set(np.unique(mult)) <= {1.0, 2.0, 4.0, 8.0}
    ex, ey, ez = elems
    # count of unique nodes by multiplicity: vertices interior to the element grid have 8
    n8 = (ex - 1) * (ey - 1) * (ez - 1)
    u8 = len(np.unique(m.glo.reshape(-1)[mult == 8.0]))
    assert u8 == n8
    # every local copy of a node with multiplicity k appears exactly k times
    g = m.glo.reshape(-1)
    ids, counts = np.unique(g, return_counts=True)
    np.testing.assert_array_equal(mult, counts[np.searchsorted(ids, g)])
    assert len(ids) == m.nglobal


def test_dssum_matches_dense_Q(oracle):
    N = 2
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(2, 2, 1), eps=0.05)
    g = m.glo.reshape(-1)
    L, U = g.size, m.nglobal
    Q = np.zeros((L, U))
    Q[np.arange(L), g] = 1.0
    v = meshgen.random_field(L, 3)
    np.testing.assert_allclose(oracle.dssum(g, v), Q @ (Q.T @ v), rtol=0, atol=1e-15)


def test_dssum_continuous_is_multiplicity(oracle):
    N = 3
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(2, 3, 2))
    g = m.glo.reshape(-1)
    vg = meshgen.random_field(m.nglobal, 4)
    v = vg[g]
    np.testing.assert_allclose(oracle.dssum(g, v), oracle.multiplicity(g) * v, rtol=1e-15)


@pytest.mark.parametrize("parts", [(1, 1, 2), (1, 2, 2), (2, 2, 2)])
def test_dssum_virtual_partition_independence(oracle, parts):
    """Summing per-part partial DSSUMs over the shared ids equals the
    unpartitioned DSSUM (the multi-GPU exchange contract)."""
    N = 3
    elems = (2, 2, 4)
    xi, _ = oracle.gll(N)
    full = meshgen.box_mesh(N, xi, elems=elems)
    v_full = meshgen.random_field(full.nlocal, 5)
    # element (a,b,c) -> offset in the full mesh
    ex, ey, _ = elems
    key = lambda eidx: eidx[:, 0] + ex * (eidx[:, 1] + ey * eidx[:, 2])
    ref = oracle.dssum(full.glo, v_full).reshape(full.nelem, -1)
    P = parts[0] * parts[1] * parts[2]
    partials = []
    for r in range(P):
        pm = meshgen.box_mesh(N, xi, elems=elems, parts=parts, rank=r)
        vr = v_full.reshape(full.nelem, -1)[key(pm.eidx)]
        partials.append((pm, oracle.dssum(pm.glo, vr)))
    totals = np.zeros(full.nglobal)
    for pm, s in partials:
        g = pm.glo.reshape(-1)
        first = np.unique(g, return_index=True)[1]   # one copy per id per part
        np.add.at(totals, g[first], s.reshape(-1)[first])
    for pm, _ in partials:
        got = totals[pm.glo]
        np.testing.assert_allclose(got, ref[key(pm.eidx)], rtol=0, atol=1e-14)


def _cg_setup(oracle, N, elems, eps, rhs="sin"):
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    G, J = oracle.geom(N, m.xyz)
    if rhs == "sin":
        us, f = meshgen.manufactured(m)
    elif rhs == "poly":
        us, f = meshgen.cube_poly(m)
    else:
        us, f = None, meshgen.random_field(m.nlocal, 7)
        f = f.reshape(m.nelem, -1)[:, :]  # discontinuous f is fine: b is assembled
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)
    return m, G, J, b, us


@pytest.mark.parametrize("N,its_max", [(4, 40), (7, 120)])
def test_cg_polynomial_reproduction(oracle, N, its_max):
    """u* = x(1-x)y(1-y)z(1-z) lies in V_N and GLL quadrature is exact for the
    Galerkin integrals when N >= 3, so CG must reproduce u* at the nodes."""
    m, G, J, b, us = _cg_setup(oracle, N, (2, 2, 2), 0.0, "poly")
    x, its, rel, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-14, maxit=500)
    assert st == 0 and its <= its_max
    assert np.max(np.abs(x - us)) <= 1e-13


@pytest.mark.parametrize("N,elems,eps", [(4, (2, 2, 2), 0.0), (4, (2, 2, 2), 0.05),
                                         (3, (3, 2, 2), 0.05)])
def test_cg_matches_dense_cg(oracle, N, elems, eps):
    """The oracle's CG on local storage with (.,.)_c must take exactly the
    iterations of textbook CG on the dense masked assembled K (built by the
    independent route) and agree with numpy.linalg.solve."""
    m, G, J, b, _ = _cg_setup(oracle, N, elems, eps, "sin")
    x, its, rel, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=1000)
    assert st == 0
    xin, wn = _indep.gll_numpy(N)
    mats = [_indep.element_stiffness_physical(m.xyz[e], xin, wn)[0] for e in range(m.nelem)]
    K = _indep.assemble_dense(mats, m.glo, m.nglobal)
    g = m.glo.reshape(-1)
    interior = np.ones(m.nglobal, dtype=bool)
    interior[np.unique(g[m.dirichlet.reshape(-1) == 1])] = False
    bg = np.zeros(m.nglobal)
    bg[g] = b
    Ki = K[np.ix_(interior, interior)]
    xd, its_d = _indep.dense_cg(Ki, bg[interior], 1e-8, 1000)
    assert its == its_d
    xs = np.linalg.solve(Ki, bg[interior])
    xg = np.zeros(m.nglobal)
    xg[g] = x
    assert np.linalg.norm(xg[interior] - xs) <= 1e-6 * np.linalg.norm(xs)
    np.testing.assert_allclose(xg[interior], xd, rtol=0, atol=1e-10 * np.abs(xd).max())
    # solution is continuous and zero on the Dirichlet boundary
    assert np.all(x[m.dirichlet.reshape(-1) == 1] == 0.0)
    np.testing.assert_array_equal(x, xg[g])


def test_cg_spectral_accuracy(oracle):
    """Informative O8: sin solution, c1 affine error ~3.3e-5 (N=4, 2x2x2)."""
    m, G, J, b, us = _cg_setup(oracle, 4, (2, 2, 2), 0.0, "sin")
    x, its, rel, st = oracle.cg(4, m.glo, m.dirichlet, G, b, tol=1e-12, maxit=500)
    err = np.max(np.abs(x - us))
    assert 1e-6 < err < 1e-4


def test_cg_edge_cases(oracle):
    m, G, J, b, _ = _cg_setup(oracle, 3, (2, 2, 2), 0.05, "sin")
    # zero RHS: rho0 = 0 -> iters 0, x unchanged (= x0 = 0)
    x, its, rel, st = oracle.cg(3, m.glo, m.dirichlet, G, np.zeros_like(b), tol=1e-8, maxit=10)
    assert its == 0 and rel == 0.0 and st == 0 and not x.any()
    # maxit hit with tol > 0 -> status 4 (ENOCONV), iters == maxit
    x, its, rel, st = oracle.cg(3, m.glo, m.dirichlet, G, b, tol=1e-12, maxit=5)
    assert its == 5 and st == 4 and rel > 1e-12
    # tol = 0: exactly maxit iterations, status 0
    x, its, rel, st = oracle.cg(3, m.glo, m.dirichlet, G, b, tol=0.0, maxit=7)
    assert its == 7 and st == 0
    # warm start: x0 is honoured (the residual is formed from b - A x0), so a
    # restart from a converged iterate stays at the solution
    x1, its1, _, _ = oracle.cg(3, m.glo, m.dirichlet, G, b, tol=1e-10, maxit=500)
    x2, its2, _, _ = oracle.cg(3, m.glo, m.dirichlet, G, b, x0=x1, tol=1e-3, maxit=500)
    assert its2 >= 1
    assert np.max(np.abs(x2 - x1)) <= 1e-9 * np.max(np.abs(x1))
