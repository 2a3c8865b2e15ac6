"""Pins for oracle O3 (geometric factors), O4 (local Ax) and O6 (assembled K).

PAPER.md:593-596 (eq:semOperator), :604 (reference map), :613 (Jacobian),
:615-625 (derivative sparsity), :627-665 (chain rule, G^ = G^T G per node).
Pinned by: closed-form affine factors; the Kronecker closed form of A^e
(with K1 from the independent Vandermonde route); A^e 1 = 0, symmetry, PSD
with a one-dimensional null space; the support pattern of A^e delta; and the
assembled stiffness against an independent physical-gradient route.
"""
import numpy as np
import pytest

from paper_1403_0968_b200 import meshgen
from tests import _indep


def _single_box(oracle, N, h=(2.0, 0.5, 1.5), eps=0.0):
    xi, _ = oracle.gll(N)
    return meshgen.box_mesh(N, xi, elems=(1, 1, 1), lengths=h, eps=eps)


@pytest.mark.parametrize("N", [1, 2, 4, 7])
def test_affine_factors_closed_form(oracle, N):
    hx, hy, hz = 2.0, 0.5, 1.5
    m = _single_box(oracle, N, (hx, hy, hz))
    G, J = oracle.geom(N, m.xyz)
    _, w = oracle.gll(N)
    w3 = np.einsum("k,j,i->kji", w, w, w).reshape(-1)
    np.testing.assert_allclose(J[0], hx * hy * hz / 8, rtol=1e-14)
    np.testing.assert_allclose(G[0, 0], w3 * hy * hz / (2 * hx), rtol=1e-13)
    np.testing.assert_allclose(G[0, 3], w3 * hx * hz / (2 * hy), rtol=1e-13)
    np.testing.assert_allclose(G[0, 5], w3 * hx * hy / (2 * hz), rtol=1e-13)
    for f in (1, 2, 4):
        assert np.max(np.abs(G[0, f])) <= 1e-14 * np.max(np.abs(G[0, 0]))


def _element_matrix(oracle, N, G1):
    n3 = (N + 1) ** 3
    A = np.zeros((n3, n3))
    for q in range(n3):
        e = np.zeros(n3)
        e[q] = 1.0
        A[:, q] = oracle.ax(N, G1, e)
    return A


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_kronecker_closed_form(oracle, N):
    """A^e = (hy hz/2hx) M(x)M(x)K1 + (hx hz/2hy) M(x)K1(x)M + (hx hy/2hz) K1(x)M(x)M
    (k (x) j (x) i order for i-fastest storage), SURVEY.md §8(c) O4."""
    hx, hy, hz = 2.0, 0.5, 1.5
    m = _single_box(oracle, N, (hx, hy, hz))
    G, _ = oracle.geom(N, m.xyz)
    A = _element_matrix(oracle, N, G)
    xi, w = _indep.gll_numpy(N)
    K1 = _indep.stiffness_1d(xi, w)
    M = np.diag(w)
    ref = (hy * hz / (2 * hx)) * np.kron(M, np.kron(M, K1)) \
        + (hx * hz / (2 * hy)) * np.kron(M, np.kron(K1, M)) \
        + (hx * hy / (2 * hz)) * np.kron(K1, np.kron(M, M))
    assert np.max(np.abs(A - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("N,eps", [(2, 0.0), (3, 0.05), (4, 0.05), (6, 0.1)])
def test_element_matrix_invariants(oracle, N, eps):
    m = _single_box(oracle, N, (1.0, 1.0, 1.0), eps=eps) if eps == 0 else None
    if m is None:
        # a deformed element: one element of a deformed 2x2x2 mesh (interior corner)
        xi, _ = oracle.gll(N)
        mm = meshgen.box_mesh(N, xi, elems=(2, 2, 2), eps=eps)
        G, _ = oracle.geom(N, mm.xyz)
        G1 = G[:1]
    else:
        G1, _ = oracle.geom(N, m.xyz)
    A = _element_matrix(oracle, N, G1)
    scale = np.max(np.abs(A))
    n3 = (N + 1) ** 3
    assert np.max(np.abs(A @ np.ones(n3))) <= 1e-13 * scale        # annihilates constants
    assert np.max(np.abs(A - A.T)) <= 1e-14 * scale                # symmetric
    ev = np.linalg.eigvalsh(0.5 * (A + A.T))
    assert ev[0] >= -1e-12 * scale                                 # PSD
    assert ev[1] > 1e-6 * scale                                    # 1-D null space


@pytest.mark.parametrize("N", [2, 4, 5])
def test_support_pattern(oracle, N):
    """PAPER.md:615-625 derivative sparsity: A^e delta_abc is supported on the
    3 lines through abc (3N+1 nodes) on an affine element and on the 3 planes
    (3n^2-3n+1 nodes) on a deformed one."""
    n = N + 1
    n3 = n ** 3
    xi, _ = oracle.gll(N)
    aff = meshgen.box_mesh(N, xi, elems=(1, 1, 1), lengths=(2.0, 0.5, 1.5))
    dfm = meshgen.box_mesh(N, xi, elems=(2, 2, 2), eps=0.1)
    Ga, _ = oracle.geom(N, aff.xyz)
    Gd, _ = oracle.geom(N, dfm.xyz)
    q = 1 + n * 1 + n * n * 1  # node (1,1,1)
    e = np.zeros(n3)
    e[q] = 1.0
    wa = oracle.ax(N, Ga, e)
    wd = oracle.ax(N, Gd[:1], e)
    assert np.count_nonzero(np.abs(wa) > 1e-14) == 3 * N + 1
    assert np.count_nonzero(np.abs(wd) > 1e-14) == 3 * n * n - 3 * n + 1


@pytest.mark.parametrize("N,elems,eps", [(2, (2, 2, 2), 0.05), (3, (2, 1, 2), 0.05),
                                         (4, (2, 2, 2), 0.05), (6, (1, 1, 1), 0.1),
                                         (8, (1, 1, 1), 0.05)])
def test_assembled_K_independent_route(oracle, N, elems, eps):
    """O6: K = sum_e Q_e^T A^e Q_e from the oracle's local Ax equals the dense
    physical-gradient assembly with a monomial (Vandermonde) basis."""
    xi, w = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    G, _ = oracle.geom(N, m.xyz)
    U = m.nglobal
    K_or = np.zeros((U, U))
    for e in range(m.nelem):
        A = _element_matrix(oracle, N, G[e:e + 1])
        g = m.glo[e]
        K_or[np.ix_(g, g)] += A
    xin, wn = _indep.gll_numpy(N)
    mats = [_indep.element_stiffness_physical(m.xyz[e], xin, wn)[0] for e in range(m.nelem)]
    K_ind = _indep.assemble_dense(mats, m.glo, U)
    scale = np.max(np.abs(K_ind))
    assert np.max(np.abs(K_or - K_ind)) <= 1e-12 * scale
    assert np.max(np.abs(K_or @ np.ones(U))) <= 1e-12 * scale
    # masked K is SPD
    interior = np.ones(U, dtype=bool)
    interior[np.unique(m.glo[m.dirichlet == 1])] = False
    Ki = K_or[np.ix_(interior, interior)]
    if Ki.size:
        assert np.linalg.eigvalsh(0.5 * (Ki + Ki.T))[0] > 0


def test_geometry_rejects_inverted_element(oracle):
    N = 2
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(1, 1, 1))
    xyz = m.xyz.copy()
    xyz[:, 0] *= -1.0   # mirror: J < 0
    with pytest.raises(oracle.OracleError):
        oracle.geom(N, xyz)


def test_mass_sums_to_volume(oracle):
    """Lumped mass J w_abc integrates 1 exactly on an
    affine box: sum over local nodes = volume."""
    N = 5
    xi, w = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(3, 2, 2), lengths=(1.5, 1.0, 0.5))
    _, J = oracle.geom(N, m.xyz)
    w3 = np.einsum("k,j,i->kji", w, w, w).reshape(-1)
    assert abs((J * w3[None]).sum() - 0.75) <= 1e-13
