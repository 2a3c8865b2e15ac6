"""The oracle on NON-box conforming hexahedral meshes (Omega_h
is any union of conforming hexahedra; :667 global-local numbering):
meshgen.prism_mesh -- a polygon split into quads around its centre, extruded
-- puts sides = 3, 5, 6 elements around the central vertical edge, so the
gather-scatter sees multiplicities 3, 5, 6, 10, 12 that a box never has.
Pins (no implementation compared with itself):
* multiplicities = a brute-force count of the elements whose node sets
  contain each node's coordinates, and the closed-form counts of the
  construction on the central line;
* DSSUM = the dense 0/1 Q Q^T;
* Q^T A_L Q (oracle Ax + DSSUM on scattered unit vectors) = the dense
  stiffness assembled by the independent physical-gradient / monomial route
  (tests/_indep.py), and K 1 = 0;
* CG iteration counts identical to textbook CG on the dense masked K, and the
  solution agrees with numpy.linalg.solve."""
import numpy as np
import pytest

import oracle
from paper_1403_0968_b200 import meshgen
from tests import _indep


def _mesh(N, sides, nz):
    xi, _ = oracle.gll(N)
    return meshgen.prism_mesh(N, xi, sides=sides, nz=nz)


@pytest.mark.parametrize("sides,nz", [(3, 2), (5, 1), (6, 3)])
def test_prism_multiplicities(sides, nz):
    N = 3
    m = _mesh(N, sides, nz)
    g = m.glo.reshape(-1)
    mult = oracle.multiplicity(g)
    # brute force: how many elements hold a node at each node's position
    pts = m.xyz.transpose(0, 2, 1)                       # [E, n3, 3]
    for e in range(m.nelem):
        for q in (0, 5, pts.shape[1] - 1):
            p = pts[e, q]
            cnt = sum(np.any(np.all(np.abs(pts[f] - p) < 1e-12, axis=1)) for f in range(m.nelem))
            assert mult[e * pts.shape[1] + q] == cnt
    # central vertical line: sides copies, 2 sides at the interior layer interfaces
    central = np.all(np.abs(pts[..., :2]) < 1e-12, axis=2).reshape(-1)
    ids, first = np.unique(g[central], return_index=True)
    zs = pts.reshape(-1, 3)[central][first, 2]
    m_c = mult[central][first]
    inner_iface = np.isclose(zs[:, None], np.arange(1, nz)[None, :] / nz).any(axis=1)
    assert np.all(m_c[inner_iface] == 2 * sides)
    assert np.all(m_c[~inner_iface] == sides)
    assert ids.size == nz * N + 1
    assert sides in set(mult.astype(int).tolist())


@pytest.mark.parametrize("sides", [3, 5, 6])
def test_prism_dssum_is_dense_qqt(sides):
    N = 2
    m = _mesh(N, sides, 2)
    g = m.glo.reshape(-1)
    L, U = g.size, m.nglobal
    Q = np.zeros((L, U))
    Q[np.arange(L), g] = 1.0
    v = meshgen.random_field(L, sides)
    np.testing.assert_allclose(oracle.dssum(g, v), Q @ (Q.T @ v), rtol=0, atol=1e-14)


@pytest.mark.parametrize("sides,N", [(3, 3), (5, 2), (6, 3)])
def test_prism_assembled_operator_independent_route(sides, N):
    m = _mesh(N, sides, 2)
    G, J = oracle.geom(N, m.xyz)
    assert J.min() > 0
    xin, wn = _indep.gll_numpy(N)
    mats = [_indep.element_stiffness_physical(m.xyz[e], xin, wn)[0] for e in range(m.nelem)]
    K = _indep.assemble_dense(mats, m.glo, m.nglobal)
    g = m.glo.reshape(-1)
    rng = np.random.default_rng(sides)
    for _ in range(3):
        v = rng.uniform(-1, 1, m.nglobal)
        w = oracle.dssum(g, oracle.ax(N, G, v[g]))
        Kv = K @ v
        assert np.linalg.norm(w - Kv[g]) <= 1e-12 * np.linalg.norm(Kv[g])
    assert np.abs(K @ np.ones(m.nglobal)).max() <= 1e-12 * np.abs(K).max()


@pytest.mark.parametrize("sides", [3, 5, 6])
def test_prism_cg_matches_dense_cg(sides):
    N = 3
    m = _mesh(N, sides, 2)
    G, J = oracle.geom(N, m.xyz)
    f = np.sin(np.pi * m.xyz[:, 0]) * np.cos(np.pi * m.xyz[:, 1]) * (1 + m.xyz[:, 2])
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f.reshape(-1))
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
    np.testing.assert_array_equal(x, xg[g])
