"""The discretisation is independent of how the mesh is presented (element
order, element orientation, global id labels): pins of the oracle's geometry,
operator, DSSUM and CG under meshgen.relabel (random element order, random
quarter turns of each element about its k axis, a random injective global-id
relabelling with gaps).  These exercise the general global-local numbering
 beyond the lexicographic box ids."""
import numpy as np
import pytest

from paper_1403_0968_b200 import meshgen


def _pair(oracle, N, elems, eps, seed):
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    r = meshgen.relabel(m, seed)
    return m, r


def _map_by_coords(m, r):
    """local index of r -> local index of m holding the same node (same xyz)."""
    n3 = m.glo.shape[1]
    key_m = {tuple(np.round(m.xyz[e][:, q], 12)): e * n3 + q
             for e in range(m.nelem) for q in range(n3)}
    out = np.empty(r.nlocal, dtype=np.int64)
    for e in range(r.nelem):
        for q in range(n3):
            out[e * n3 + q] = key_m[tuple(np.round(r.xyz[e][:, q], 12))]
    return out


@pytest.mark.parametrize("N,elems,eps,seed", [(3, (2, 2, 2), 0.05, 1), (4, (3, 2, 1), 0.0, 2)])
def test_relabel_geometry_and_multiplicity(oracle, N, elems, eps, seed):
    m, r = _pair(oracle, N, elems, eps, seed)
    G, J = oracle.geom(N, r.xyz)
    assert np.all(J > 0)
    assert len(np.unique(r.glo)) == m.nglobal
    assert r.glo.min() >= 7 and np.any(np.diff(np.unique(r.glo)) > 1)   # non-compact ids
    mm, mr = oracle.multiplicity(m.glo), oracle.multiplicity(r.glo)
    np.testing.assert_array_equal(np.sort(mm), np.sort(mr))
    # the same global node carries the same id in every element holding it
    g = r.glo.reshape(-1)
    for gid in np.unique(g)[:200]:
        pts = r.xyz.transpose(0, 2, 1).reshape(-1, 3)[g == gid]
        assert np.ptp(pts, axis=0).max() == 0.0


@pytest.mark.parametrize("N,elems,eps,seed", [(3, (2, 2, 2), 0.05, 3), (5, (2, 1, 2), 0.1, 4)])
def test_relabel_operator_dssum_cg_invariant(oracle, N, elems, eps, seed):
    m, r = _pair(oracle, N, elems, eps, seed)
    src = _map_by_coords(m, r)
    Gm, Jm = oracle.geom(N, m.xyz)
    Gr, Jr = oracle.geom(N, r.xyz)
    # a continuous field (one value per global node): the assembled operator
    # Q Q^T A_L u agrees node by node
    u = meshgen.random_field(m.nglobal, 5)[m.glo.reshape(-1)]
    wm = oracle.dssum(m.glo, oracle.ax(N, Gm, u))
    wr = oracle.dssum(r.glo, oracle.ax(N, Gr, u[src]))
    np.testing.assert_allclose(wr, wm[src], rtol=0, atol=1e-12 * np.abs(wm).max())
    _, f = meshgen.manufactured(m)
    bm = oracle.mass_rhs(N, m.glo, m.dirichlet, Jm, f)
    br = oracle.mass_rhs(N, r.glo, r.dirichlet, Jr, f.reshape(-1)[src])
    xm, im, _, _ = oracle.cg(N, m.glo, m.dirichlet, Gm, bm, tol=1e-10, maxit=1000)
    xr, ir, _, _ = oracle.cg(N, r.glo, r.dirichlet, Gr, br, tol=1e-10, maxit=1000)
    assert abs(im - ir) <= 1
    np.testing.assert_allclose(xr, xm[src], rtol=0, atol=1e-9 * np.abs(xm).max())
