"""GPU parity on NON-box meshes (meshgen.prism_mesh):
multiplicities 3, 5, 6, 10, 12 exercise the gather-scatter branches a box
never reaches -- gs_group<3>, gs_group<6>, gs_group_generic, K2's generic
(runtime-m) group path in both K2 kernels, the Dirichlet classes of odd
multiplicity -- through Ax, DSSUM, CG, Jacobi PCG, single-reduction CG and the
multi-rank loopback exchange (layers as ranks).  Bars as tests/test_gpu_parity.py:
Ax rel-L2 <= 1e-12, DSSUM bit-identical to the oracle, identical CG counts,
x rel-L2 <= 1e-10."""
import numpy as np
import pytest

import oracle
from tests import _margin
from paper_1403_0968_b200 import meshgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1403_0968_b200 import sem
    sem.lib()
    return torch.device("cuda", 0)


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def T(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def rhs(m, J):
    f = np.sin(np.pi * m.xyz[:, 0]) * np.cos(np.pi * m.xyz[:, 1]) * (1 + m.xyz[:, 2])
    return oracle.mass_rhs(m.N, m.glo, m.dirichlet, J, f.reshape(-1))


@pytest.fixture(params=["default", "tma", "hi", "simple", "k2plain"])
def impl(request, monkeypatch):
    monkeypatch.delenv("SEM_K2", raising=False)
    monkeypatch.delenv("SEM_AX_KERNEL", raising=False)
    if request.param == "k2plain":
        monkeypatch.setenv("SEM_K2", "plain")
    elif request.param != "default":
        monkeypatch.setenv("SEM_AX_KERNEL", request.param)
    return request.param


@pytest.mark.parametrize("sides,N,nz", [(3, 3, 2), (5, 4, 2), (6, 7, 2), (3, 7, 3), (6, 10, 1),
                                        (5, 12, 2)])
def test_prism_parity(dev, impl, sides, N, nz):
    from paper_1403_0968_b200 import sem
    xi, _ = oracle.gll(N)
    m = meshgen.prism_mesh(N, xi, sides=sides, nz=nz)
    G, J = oracle.geom(N, m.xyz)
    ctx = sem.Context(m, N, device=0)
    assert ctx.nglobal == m.nglobal
    u = meshgen.random_field(m.nlocal, sides + N)
    w = ctx.ax(T(u, dev))
    wr = oracle.ax(N, G, u)
    assert relerr(w.cpu().numpy(), wr) <= 1e-12
    ctx.dssum(w)
    assert relerr(w.cpu().numpy(), oracle.dssum(m.glo, wr)) <= 1e-12
    d = ctx.dssum(T(u, dev))
    np.testing.assert_array_equal(d.cpu().numpy(), oracle.dssum(m.glo, u))
    b = rhs(m, J)
    bd = T(b, dev)
    # counts under the drift rule of tests/_margin.py (identical when the
    # oracle's stop has a margin above the measured GPU-vs-oracle drift)
    methods = [("cg", {}), ("jacobi", {"precond": "jacobi"})]
    # (SEM_AX_KERNEL=tma above N=10 selects the simple kernel: no KA variant)
    if impl != "simple" and not (impl == "tma" and N > 10):
        methods.append(("sr", {"variant": "single_reduction"}))
    for meth, kw in methods:
        x, its, rel, ok = ctx.cg(bd, tol=1e-8, maxit=3000, **kw)
        with oracle.history() as h:
            if meth == "sr":
                xr, its_r, rel_r, st = oracle.cg_single_reduction(N, m.glo, m.dirichlet, G, b,
                                                                  tol=1e-8, maxit=3000)
            else:
                xr, its_r, rel_r, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8,
                                                 maxit=3000, **kw)
        assert ok and st == 0

        def solve(k, kw=kw):
            _, it, rl, _ = ctx.cg(bd, tol=0.0, maxit=k, **kw)
            return it, rl

        dr = _margin.drift(_margin.gpu_history(solve, its_r), h.values)
        assert dr <= _margin.DRIFT_MAX[meth], (meth, dr)
        _margin.assert_count(its, its_r, _margin.margin(h.values, its_r, 1e-8), dr,
                             (meth, rel, rel_r))
        if its == its_r:
            assert relerr(x.cpu().numpy(), xr) <= 1e-10


@pytest.mark.parametrize("sides,N", [(3, 4), (6, 7)])
def test_prism_multirank_layers(dev, sides, N):
    """Two ranks, one layer each: the central line's layer-interface node has
    `sides` copies on each rank (2 sides in total)."""
    from paper_1403_0968_b200 import dist as sdist
    from paper_1403_0968_b200 import sem
    xi, _ = oracle.gll(N)
    full = meshgen.prism_mesh(N, xi, sides=sides, nz=2)
    G, J = oracle.geom(N, full.xyz)
    per = full.nelem // 2
    ranks = []
    for r in range(2):
        sl = slice(r * per, (r + 1) * per)
        ranks.append(meshgen.Mesh(N=N, xyz=np.ascontiguousarray(full.xyz[sl]),
                                  glo=np.ascontiguousarray(full.glo[sl]),
                                  dirichlet=np.ascontiguousarray(full.dirichlet[sl]),
                                  elems=full.elems, lengths=full.lengths))
    u = meshgen.random_field(full.nlocal, 4)
    b = rhs(full, J)
    n3 = (N + 1) ** 3
    ds = oracle.dssum(full.glo, u).reshape(full.nelem, n3)
    xr, its_r, _, _ = oracle.cg(N, full.glo, full.dirichlet, G, b, tol=1e-8, maxit=3000)
    xr = xr.reshape(full.nelem, n3)

    def body(lr):
        r = lr.rank
        ctx = sem.Context(ranks[r], N, device=0, loopback=lr)
        try:
            d = ctx.dssum(T(u.reshape(full.nelem, n3)[r * per:(r + 1) * per].reshape(-1), dev))
            x, its, _, ok = ctx.cg(T(b.reshape(full.nelem, n3)[r * per:(r + 1) * per].reshape(-1), dev),
                                   tol=1e-8, maxit=3000)
            return d.cpu().numpy(), x.cpu().numpy(), its, ok, ctx.nglobal
        finally:
            ctx.free()

    out = sdist.LoopbackGroup(2, device=0).run(body)
    for r, (d, x, its, ok, ng) in enumerate(out):
        assert ng == full.nglobal and ok and its == its_r
        assert relerr(d, ds[r * per:(r + 1) * per].reshape(-1)) <= 1e-12
        assert relerr(x, xr[r * per:(r + 1) * per].reshape(-1)) <= 1e-10
