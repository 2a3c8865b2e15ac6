"""GPU parity of the single-reduction (Chronopoulos-Gear) CG (NEXT-3,
SURVEY.md §8(f); reading R7): libsem's sem_cg_sr (KA: TMA Ax + (r,w)
partials; KB: DSSUM + the recurrences on global-storage p, s, x increment)
through the C ABI against the oracle's ora_cg_cgs on the same seeded inputs.
Bars as for CG: identical iteration counts at tol 1e-8, x rel-L2 <= 1e-10
(c3 full size: +-2 iterations, R3)."""
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


@pytest.fixture(params=["tma", "hi", "tma-nograph"])
def impl(request, monkeypatch):
    monkeypatch.setenv("SEM_AX_KERNEL", request.param.split("-")[0])
    monkeypatch.setenv("SEM_CG_GRAPH", "0" if request.param.endswith("nograph") else "1")
    monkeypatch.delenv("SEM_K1_SPLIT", raising=False)
    return request.param


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def T(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def make(N, elems, eps):
    from paper_1403_0968_b200 import sem
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    G, J = oracle.geom(N, m.xyz)
    return m, G, J, sem.Context(m, N, device=0)


def rhs(m, J, kind="sin"):
    if kind == "sin":
        _, f = meshgen.manufactured(m)
    else:
        f = meshgen.random_field(m.nlocal, 11)
    return oracle.mass_rhs(m.N, m.glo, m.dirichlet, J, f)


SR = "single_reduction"


@pytest.mark.parametrize("N,elems,eps,kind", [
    (4, (2, 2, 2), 0.05, "sin"), (4, (2, 2, 2), 0.05, "rand"), (3, (5, 4, 3), 0.05, "rand"),
    (7, (8, 8, 8), 0.05, "sin"), (2, (3, 3, 3), 0.0, "rand"), (9, (2, 3, 2), 0.05, "sin"),
    (12, (2, 2, 1), 0.05, "sin"), (12, (2, 1, 2), 0.1, "sin"), (1, (4, 3, 3), 0.05, "rand")])
def test_cg_sr_iteration_parity(dev, impl, N, elems, eps, kind):
    """Counts under the drift rule of tests/_margin.py: identical when the
    oracle's stop has a margin above the measured GPU-vs-oracle residual drift
    (the recursively updated residual of this recurrence drifts a few % over a
    solve, R7), within one iteration otherwise; the drift itself
    below DRIFT_MAX (25%).  (The N=12 2x2x1 eps=0.05 case crosses with a 3%
    margin.)"""
    if impl.startswith("tma") and N > 10:
        pytest.skip("SEM_AX_KERNEL=tma above N=10 selects the simple kernel (no KA variant)")
    m, G, J, ctx = make(N, elems, eps)
    b = rhs(m, J, kind)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=2000, variant=SR)
    with oracle.history() as h:
        xr, its_r, rel_r, st = oracle.cg_single_reduction(N, m.glo, m.dirichlet, G, b, tol=1e-8,
                                                          maxit=2000)
    assert ok and st == 0
    bd = T(b, dev)

    def solve(k):
        _, it, rl, _ = ctx.cg(bd, tol=0.0, maxit=k, variant=SR)
        return it, rl

    dr = _margin.drift(_margin.gpu_history(solve, its_r), h.values)
    assert dr <= _margin.DRIFT_MAX["sr"]
    _margin.assert_count(its, its_r, _margin.margin(h.values, its_r, 1e-8), dr, (rel, rel_r))
    if its != its_r:        # one iteration apart (a narrow margin): x one step apart
        assert relerr(x.cpu().numpy(), xr) <= 1e-7
        return
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    # the final residual norms drift apart by a few % over the solve (R3)
    assert abs(rel - rel_r) <= 0.1 * rel_r


def test_cg_sr_c1_twenty_iterations(dev, impl):
    m, G, J, ctx = make(4, (2, 2, 2), 0.05)
    b = rhs(m, J)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=0.0, maxit=20, variant=SR)
    xr, its_r, rel_r, st = oracle.cg_single_reduction(4, m.glo, m.dirichlet, G, b, tol=0.0,
                                                      maxit=20)
    assert its == its_r == 20 and ok
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    assert abs(rel - rel_r) <= 1e-8 * rel_r


def test_cg_sr_edge_cases(dev, impl):
    m, G, J, ctx = make(3, (2, 2, 2), 0.05)
    b = rhs(m, J)
    x, its, rel, ok = ctx.cg(torch.zeros(m.nlocal, dtype=torch.float64, device=dev), tol=1e-8,
                             maxit=10, variant=SR)
    assert its == 0 and rel == 0.0 and ok and not x.any()
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=0, variant=SR)
    assert its == 0 and not ok and rel == 1.0
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-12, maxit=5, variant=SR)
    xr, its_r, rel_r, st = oracle.cg_single_reduction(3, m.glo, m.dirichlet, G, b, tol=1e-12,
                                                      maxit=5)
    assert its == its_r == 5 and not ok and st == 4
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    # warm start, including a DISCONTINUOUS x0 (x = x0 + increment at every copy)
    for cont in (True, False):
        x0 = meshgen.random_field(m.nlocal, 3) * 0.01
        if cont:
            x0 = oracle.dssum(m.glo, x0) / oracle.multiplicity(m.glo)
        x, its, rel, ok = ctx.cg(T(b, dev), x=T(x0, dev), tol=1e-9, maxit=500, variant=SR)
        xr, its_r, rel_r, st = oracle.cg_single_reduction(3, m.glo, m.dirichlet, G, b, x0=x0,
                                                          tol=1e-9, maxit=500)
        assert ok and its == its_r, (cont, its, its_r)
        assert relerr(x.cpu().numpy(), xr) <= 1e-10
    x1, i1, r1, _ = ctx.cg(T(b, dev), tol=1e-8, maxit=500, variant=SR)
    x2, i2, r2, _ = ctx.cg(T(b, dev), tol=1e-8, maxit=500, variant=SR)
    assert i1 == i2 and r1 == r2 and torch.equal(x1, x2)


def test_cg_sr_and_cg_alternate(dev, impl):
    """Three solvers (three captured graphs) on one context (the c1 mesh: its
    residual margins at the stop are comfortable for all three; on 3x2x2 the
    oracle's CG residual at iteration 59 is 1.009e-8, within rounding of the
    threshold, R3)."""
    m, G, J, ctx = make(4, (2, 2, 2), 0.05)
    b = rhs(m, J)
    _, its_cg, _, _ = oracle.cg(4, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=500)
    _, its_sr, _, _ = oracle.cg_single_reduction(4, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=500)
    _, its_pc, _, _ = oracle.cg(4, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=500, precond="jacobi")
    seen = {}
    for var, pc, want in ((SR, "none", its_sr), ("standard", "none", its_cg),
                          ("standard", "jacobi", its_pc), (SR, "none", its_sr),
                          ("standard", "none", its_cg)):
        x, its, _, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=500, variant=var, precond=pc)
        assert ok and its == want, (var, pc, its, want)
        if (var, pc) in seen:       # a repeat through the same captured graph is identical
            assert its == seen[(var, pc)][0] and torch.equal(x, seen[(var, pc)][1])
        seen[(var, pc)] = (its, x.clone())


def test_cg_sr_rejects_unsupported(dev, monkeypatch):
    from paper_1403_0968_b200 import sem
    xi, _ = oracle.gll(3)
    m = meshgen.box_mesh(3, xi, elems=(2, 2, 1), eps=0.05)
    kap, alp = meshgen.coefficients(m)
    ctx = sem.Context(m, 3, device=0, kappa=kap, alpha=alp)
    with pytest.raises(sem.SemError):
        ctx.cg(torch.zeros(m.nlocal, dtype=torch.float64, device=dev), variant=SR)
    monkeypatch.setenv("SEM_AX_KERNEL", "simple")
    ctx2 = sem.Context(m, 3, device=0)
    with pytest.raises(sem.SemError):
        ctx2.cg(torch.zeros(m.nlocal, dtype=torch.float64, device=dev), variant=SR)


# (the full-size c3 single-reduction solve: tests/test_gpu_c3_parity.py, drift rule)


@pytest.mark.parametrize("N", [3, 7])
def test_cg_sr_relabelled_mesh(dev, N):
    from paper_1403_0968_b200 import sem
    xi, _ = oracle.gll(N)
    m = meshgen.relabel(meshgen.box_mesh(N, xi, elems=(3, 3, 2), eps=0.05), seed=12)
    G, J = oracle.geom(N, m.xyz)
    ctx = sem.Context(m, N, device=0)
    b = rhs(m, J)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=2000, variant=SR)
    xr, its_r, rel_r, st = oracle.cg_single_reduction(N, m.glo, m.dirichlet, G, b, tol=1e-8,
                                                      maxit=2000)
    assert ok and st == 0 and its == its_r, (its, its_r)
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
