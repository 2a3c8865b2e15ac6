"""GPU parity of the Jacobi-preconditioned CG (NEXT-2; PCG of
PAPER.md:672-673 "Besides the preconditioner choice"): libsem's sem_diag /
sem_pcg through the C ABI against the oracle's ora_diag_screened /
ora_pcg_screened on the same seeded inputs.  Bars as for CG: rel-L2 <= 1e-12 for
the assembled diagonal, identical iteration counts at tol 1e-8, x rel-L2 <= 1e-10
(the c3 full-size count within +-2, R3)."""
import numpy as np
import pytest

import oracle
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


@pytest.fixture(params=["tma", "hi", "simple", "tma-nograph", "tma-split"])
def impl(request, monkeypatch):
    monkeypatch.setenv("SEM_AX_KERNEL", request.param.split("-")[0])
    monkeypatch.setenv("SEM_CG_GRAPH", "0" if request.param.endswith("nograph") else "1")
    if request.param.endswith("split"):
        monkeypatch.setenv("SEM_K1_SPLIT", "0.37")
    else:
        monkeypatch.delenv("SEM_K1_SPLIT", raising=False)
    return request.param


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def T(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def make(N, elems, eps, screened=False, **kw):
    from paper_1403_0968_b200 import sem
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps, **kw)
    G, J = oracle.geom(N, m.xyz)
    co = {}
    kap = alp = None
    if screened:
        kap, alp = meshgen.coefficients(m)
        co = {"J": J, "kappa": kap, "alpha": alp}
    ctx = sem.Context(m, N, device=0, kappa=kap, alpha=alp)
    return m, G, J, co, ctx


def rhs(m, J, kind="sin"):
    if kind == "sin":
        _, f = meshgen.manufactured(m)
    else:
        f = meshgen.random_field(m.nlocal, 11)
    return oracle.mass_rhs(m.N, m.glo, m.dirichlet, J, f)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 7, 8, 10, 11, 12, 15])
@pytest.mark.parametrize("screened", [False, True])
def test_diag_parity(dev, impl, N, screened):
    """sem_diag = Q Q^T diag(A_L) vs the oracle's dssum(diag) (both layouts of
    G^: element-major for TMA/simple, slice-major for the high-order kernel)."""
    if screened and impl == "simple":
        pytest.skip("the simple kernel carries no mass term")
    m, G, J, co, ctx = make(N, (3, 2, 1), 0.05, screened)
    d = ctx.diag().cpu().numpy()
    ref = oracle.dssum(m.glo, oracle.diag(N, G, **co))
    assert relerr(d, ref) <= 1e-12, N


@pytest.mark.parametrize("N,elems,eps,kind,screened", [
    (4, (2, 2, 2), 0.05, "sin", False), (4, (2, 2, 2), 0.05, "rand", False),
    (3, (5, 4, 3), 0.05, "rand", False), (7, (8, 8, 8), 0.05, "sin", False),
    (2, (3, 3, 3), 0.0, "rand", False), (9, (2, 3, 2), 0.05, "sin", False),
    (12, (2, 2, 1), 0.05, "sin", False),
    (5, (3, 3, 2), 0.05, "sin", True), (7, (4, 4, 4), 0.05, "rand", True)])
def test_pcg_iteration_parity(dev, impl, N, elems, eps, kind, screened):
    if screened and impl == "simple":
        pytest.skip("the simple kernel carries no mass term")
    m, G, J, co, ctx = make(N, elems, eps, screened)
    b = rhs(m, J, kind)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=2000, precond="jacobi")
    xr, its_r, rel_r, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=2000,
                                     precond="jacobi", **co)
    assert ok and st == 0
    assert its == its_r, (its, its_r, rel, rel_r)
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    # final residuals drift by ~1e-3 relative over hundreds of iterations (R3)
    assert abs(rel - rel_r) <= 2e-2 * rel_r


def test_pcg_c1_twenty_iterations(dev, impl):
    m, G, J, co, ctx = make(4, (2, 2, 2), 0.05)
    b = rhs(m, J)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=0.0, maxit=20, precond="jacobi")
    xr, its_r, rel_r, st = oracle.cg(4, m.glo, m.dirichlet, G, b, tol=0.0, maxit=20,
                                     precond="jacobi")
    assert its == its_r == 20 and ok
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    assert abs(rel - rel_r) <= 1e-8 * rel_r


def test_pcg_and_cg_alternate_on_one_context(dev, impl):
    """Switching preconditioners on one context (two captured graphs) keeps
    both solves identical to their oracle runs and to a repeat."""
    m, G, J, co, ctx = make(3, (3, 2, 2), 0.05)
    b = rhs(m, J)
    _, its_c, _, _ = oracle.cg(3, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=500)
    _, its_p, _, _ = oracle.cg(3, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=500,
                               precond="jacobi")
    assert its_p < its_c
    res = []
    for pc in ("jacobi", "none", "jacobi", "none"):
        x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=500, precond=pc)
        assert ok and its == (its_p if pc == "jacobi" else its_c)
        res.append(x.clone())
    assert torch.equal(res[0], res[2]) and torch.equal(res[1], res[3])


def test_pcg_edge_cases(dev, impl):
    from paper_1403_0968_b200 import sem
    m, G, J, co, ctx = make(3, (2, 2, 2), 0.05)
    b = rhs(m, J)
    x, its, rel, ok = ctx.cg(torch.zeros(m.nlocal, dtype=torch.float64, device=dev), tol=1e-8,
                             maxit=10, precond="jacobi")
    assert its == 0 and rel == 0.0 and ok and not x.any()
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-12, maxit=5, precond="jacobi")
    xr, its_r, rel_r, st = oracle.cg(3, m.glo, m.dirichlet, G, b, tol=1e-12, maxit=5,
                                     precond="jacobi")
    assert its == its_r == 5 and not ok and st == 4
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    x0 = oracle.dssum(m.glo, meshgen.random_field(m.nlocal, 3) * 0.01) / oracle.multiplicity(m.glo)
    x0 = x0 * (1 - m.dirichlet.reshape(-1))
    x, its, rel, ok = ctx.cg(T(b, dev), x=T(x0, dev), tol=1e-9, maxit=500, precond="jacobi")
    xr, its_r, rel_r, st = oracle.cg(3, m.glo, m.dirichlet, G, b, x0=x0, tol=1e-9, maxit=500,
                                     precond="jacobi")
    assert ok and its == its_r
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    bb = T(b, dev)
    xx = torch.zeros_like(bb)
    p = sem.ctypes.c_void_p
    assert sem.lib().sem_pcg(ctx._ctx, 7, p(bb.data_ptr()), p(xx.data_ptr()), 1e-8, 10,
                             None, None) == sem.SEM_EINVAL


# (the full-size c3 Jacobi PCG solve: tests/test_gpu_c3_parity.py, drift rule)


@pytest.mark.parametrize("N", [3, 7])
def test_pcg_relabelled_mesh(dev, N):
    """Jacobi PCG on a relabelled mesh (random element order, quarter-turned
    elements, non-compact global ids): the assembled diagonal and the solve
    match the oracle."""
    from paper_1403_0968_b200 import sem
    xi, _ = oracle.gll(N)
    m = meshgen.relabel(meshgen.box_mesh(N, xi, elems=(3, 3, 2), eps=0.05), seed=11)
    G, J = oracle.geom(N, m.xyz)
    ctx = sem.Context(m, N, device=0)
    assert relerr(ctx.diag().cpu().numpy(), oracle.dssum(m.glo, oracle.diag(N, G))) <= 1e-12
    b = rhs(m, J)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=2000, precond="jacobi")
    xr, its_r, rel_r, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=2000,
                                     precond="jacobi")
    assert ok and st == 0 and its == its_r, (its, its_r)
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
