"""GPU parity of the resident CG kernel (cg_resident.cu: the whole N = 7
Poisson CG solve as one cooperative launch with x, r in TMEM and p in shared
memory; DESIGN.md §6 "Resident CG") against the plain-C oracle and against
the two-kernel schedule (SEM_CG_RESIDENT=0).

The resident kernel performs the same arithmetic as the two-kernel schedule
(same DMMA operator, same ascending-order DSSUM sums, same update
expressions, same stopping rule); only the association of
the two dot products differs (per-CTA partials).  Bars as
tests/test_gpu_parity.py: identical CG counts at tol 1e-8 (the c3-size
counts are in tests/test_gpu_c3_parity.py under the drift rule), x rel-L2 <=
1e-10 against the oracle."""
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


@pytest.fixture(autouse=True)
def _default_kernels(monkeypatch):
    for k in ("SEM_AX_KERNEL", "SEM_K1_SPLIT", "SEM_CG_GRAPH"):
        monkeypatch.delenv(k, raising=False)
    # opt-in path: the contexts are sized and set up with its tables
    monkeypatch.setenv("SEM_CG_RESIDENT", "1")


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def T(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


def box(N, elems, eps, relabel=None):
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    if relabel is not None:
        m = meshgen.relabel(m, relabel)
    G, J = oracle.geom(N, m.xyz)
    return m, G, J


def rhs(m, J, kind="sin"):
    if kind == "sin":
        _, f = meshgen.manufactured(m)
    else:
        f = meshgen.random_field(m.nlocal, 9)
    return oracle.mass_rhs(m.N, m.glo, m.dirichlet, J, f)


def solve(ctx, b, monkeypatch, resident, **kw):
    monkeypatch.setenv("SEM_CG_RESIDENT", "1" if resident else "0")
    n0 = ctx.launch_count
    out = ctx.cg(b, **kw)
    return out, ctx.launch_count - n0


@pytest.mark.parametrize("elems,eps,kind,relab", [
    ((1, 1, 1), 0.05, "sin", None),        # one element: one CTA, group 1 empty
    ((3, 2, 2), 0.05, "sin", None),        # 12 elements: 6 CTAs of 2
    ((5, 3, 1), 0.0, "rand", None),        # odd E: CTAs of 1 and 2 elements
    ((8, 8, 8), 0.05, "sin", None),
    ((8, 8, 8), 0.05, "rand", 5),          # relabelled ids and elements
    ((16, 16, 16), 0.05, "sin", 11),       # c3 size, relabelled: 28 / 27 elements per CTA
])
def test_resident_cg_parity(dev, monkeypatch, elems, eps, kind, relab):
    from paper_1403_0968_b200 import sem
    m, G, J = box(7, elems, eps, relab)
    b = rhs(m, J, kind)
    ctx = sem.Context(m, 7, device=0)
    bd = T(b, dev)
    small = m.nelem <= 512
    if small:
        xr, its_r, rel_r, st = oracle.cg(7, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=3000)
        assert st == 0
    (x, its, rel, ok), nl = solve(ctx, bd, monkeypatch, True, tol=1e-8, maxit=3000)
    ph = ctx.cg_phases()           # the resident phase clock of that solve
    assert set(ph) == set(ctx.CG_PHASES) and all(v >= 0.0 for v in ph.values())
    assert sum(ph.values()) > 0.0
    (x2, its2, rel2, ok2), nl2 = solve(ctx, bd, monkeypatch, False, tol=1e-8, maxit=3000)
    assert ok and ok2
    # one resident launch replaces ~2 launches per iteration
    assert nl <= 6 < nl2
    assert abs(its - its2) <= 1
    assert relerr(x.cpu().numpy(), x2.cpu().numpy()) <= 1e-10
    if small:
        assert its == its_r, (its, its_r, rel, rel_r)
        assert relerr(x.cpu().numpy(), xr) <= 1e-10
    ctx.free()


@pytest.mark.parametrize("k", [0, 1, 2, 7, 20])
def test_resident_fixed_count_iterates(dev, monkeypatch, k):
    """x_k after exactly k iterations (tol = 0) against the oracle's x_k."""
    from paper_1403_0968_b200 import sem
    m, G, J = box(7, (4, 3, 2), 0.05)
    b = rhs(m, J)
    ctx = sem.Context(m, 7, device=0)
    (x, its, rel, ok), _ = solve(ctx, T(b, dev), monkeypatch, True, tol=0.0, maxit=k)
    xr, its_r, rel_r, st = oracle.cg(7, m.glo, m.dirichlet, G, b, tol=0.0, maxit=k)
    assert its == its_r == k
    if k == 0:
        assert not x.any() and rel == 1.0
    else:
        assert relerr(x.cpu().numpy(), xr) <= 1e-10
        assert abs(rel - rel_r) <= 1e-8 * rel_r
    ctx.free()


def test_resident_edge_cases(dev, monkeypatch):
    from paper_1403_0968_b200 import sem
    m, G, J = box(7, (3, 3, 2), 0.05)
    b = rhs(m, J)
    ctx = sem.Context(m, 7, device=0)
    monkeypatch.setenv("SEM_CG_RESIDENT", "1")
    # zero RHS: stops before the first iteration
    x, its, rel, ok = ctx.cg(torch.zeros(m.nlocal, dtype=torch.float64, device=dev), tol=1e-8, maxit=10)
    assert its == 0 and rel == 0.0 and ok and not x.any()
    # maxit hit: not converged, the oracle's 5th iterate
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-14, maxit=5)
    xr, its_r, rel_r, st = oracle.cg(7, m.glo, m.dirichlet, G, b, tol=1e-14, maxit=5)
    assert its == its_r == 5 and not ok and st == 4
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    # warm start with a continuous x0
    x0 = meshgen.random_field(m.nlocal, 3) * 0.01
    x0 = oracle.dssum(m.glo, x0) / oracle.multiplicity(m.glo)
    x, its, rel, ok = ctx.cg(T(b, dev), x=T(x0, dev), tol=1e-9, maxit=500)
    xr, its_r, rel_r, st = oracle.cg(7, m.glo, m.dirichlet, G, b, x0=x0, tol=1e-9, maxit=500)
    assert ok and its == its_r
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    # deterministic: repeated solves are bit-identical
    x1, i1, r1, _ = ctx.cg(T(b, dev), tol=1e-8, maxit=500)
    x2, i2, r2, _ = ctx.cg(T(b, dev), tol=1e-8, maxit=500)
    assert i1 == i2 and r1 == r2 and torch.equal(x1, x2)
    ctx.free()


@pytest.mark.parametrize("sides,nz", [(3, 3), (3, 2), (5, 2), (6, 2)])
def test_resident_non_box(dev, monkeypatch, sides, nz):
    """Prism meshes: non-Dirichlet groups of multiplicity 3 and 6 (sides = 3)
    run resident (receive slots of odd counts, Dirichlet copies of odd
    multiplicity); multiplicities 10 and 12 (sides = 5, 6) exceed the
    resident limit of 8 and fall back to the two-kernel schedule."""
    from paper_1403_0968_b200 import sem
    N = 7
    xi, _ = oracle.gll(N)
    m = meshgen.prism_mesh(N, xi, sides=sides, nz=nz)
    G, J = oracle.geom(N, m.xyz)
    f = np.sin(np.pi * m.xyz[:, 0]) * np.cos(np.pi * m.xyz[:, 1]) * (1 + m.xyz[:, 2])
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f.reshape(-1))
    ctx = sem.Context(m, N, device=0)
    (x, its, rel, ok), nl = solve(ctx, T(b, dev), monkeypatch, True, tol=1e-8, maxit=3000)
    xr, its_r, rel_r, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=3000)
    glo = np.asarray(m.glo).reshape(-1)
    mult = np.bincount(glo)[glo]
    free = ~np.asarray(m.dirichlet, dtype=bool).reshape(-1)
    resident = mult[free].max() <= 8
    assert ok and st == 0 and (nl <= 6) == resident, (nl, mult[free].max())
    assert its == its_r, (its, its_r)
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    ctx.free()


def test_resident_off_by_default(dev, monkeypatch):
    """Without SEM_CG_RESIDENT=1 the context has no resident tables and sem_cg
    runs the two-kernel schedule (launches per iteration)."""
    from paper_1403_0968_b200 import sem
    monkeypatch.delenv("SEM_CG_RESIDENT")
    m, G, J = box(7, (3, 2, 2), 0.05)
    b = rhs(m, J)
    ctx = sem.Context(m, 7, device=0)
    n0 = ctx.launch_count
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=500)
    assert ok and ctx.launch_count - n0 > 2 * its
    with pytest.raises(sem.SemError):
        ctx.cg_phases()
    ctx.free()


def test_resident_capacity_boundary(dev, monkeypatch):
    """28 elements per SM is the resident capacity: E = 28 * nsm runs resident
    (a handful of launches), E = 28 * nsm + 1 falls back to the two-kernel
    schedule (launches per iteration); both agree with each other."""
    from paper_1403_0968_b200 import sem
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    cap = 28 * nsm
    res = {}
    for E, elems in ((cap, (cap // 4, 4, 1)), (cap + 4, (cap // 4 + 1, 4, 1))):
        m, G, J = box(7, elems, 0.05)
        assert m.nelem == E
        b = rhs(m, J)
        ctx = sem.Context(m, 7, device=0)
        (x, its, rel, ok), nl = solve(ctx, T(b, dev), monkeypatch, True, tol=0.0, maxit=30)
        assert its == 30
        res[E] = nl
        ctx.free()
    assert res[cap] <= 6 < res[cap + 4]
