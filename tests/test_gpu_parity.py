"""GPU parity: libsem (CUDA, sm_100a, through the C ABI) vs the plain-C oracle on
the same seeded inputs.  Bars (BASELINE.json north_star): rel-L2 <= 1e-12 for
Ax / DSSUM; identical CG iteration counts at tol 1e-8; x rel-L2 <= 1e-10
(SURVEY.md §8(c) parity bars).  Inputs come from meshgen with the ORACLE's GLL
nodes; no input or expected value comes from the CUDA path."""
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


def relerr(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.fixture(params=["tma", "hi", "simple", "tma-nograph", "tma-split", "hi-split", "dmma",
                        "dmma-split"])
def impl(request, monkeypatch):
    """All Ax kernel families -- element-staged TMA (N <= 10), vector-staged TMA
    with register-streamed G^ ("hi", N >= 6; lower N fall back to TMA), the
    simple one-block-per-element kernel (all N), the N = 7 DMMA kernel ("dmma";
    other N fall back to the defaults) -- and the CG driver with and
    without CUDA-graph chunks.  "-split": K1 as two element-range launches
    (the multi-rank boundary/interior schedule, here without an exchange)."""
    monkeypatch.setenv("SEM_AX_KERNEL", request.param.split("-")[0])
    monkeypatch.setenv("SEM_CG_GRAPH", "0" if request.param.endswith("nograph") else "1")
    if request.param.endswith("split"):
        monkeypatch.setenv("SEM_K1_SPLIT", "0.37")
    else:
        monkeypatch.delenv("SEM_K1_SPLIT", raising=False)
    return request.param


def make(N, elems, eps, **kw):
    from paper_1403_0968_b200 import sem
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps, **kw)
    G, J = oracle.geom(N, m.xyz)
    ctx = sem.Context(m, N, device=0)
    return m, G, J, ctx


def T(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


# --- Ax -------------------------------------------------------------------
@pytest.mark.parametrize("N", range(1, 16))
@pytest.mark.parametrize("eps", [0.0, 0.05])
def test_ax_parity_all_orders(dev, impl, N, eps):
    # 3x2x1 = 6 elements: several blocks for small N, a ragged last block
    # whenever EPB does not divide 6
    m, G, J, ctx = make(N, (3, 2, 1), eps)
    for seed in (0, 1, 2):
        u = meshgen.random_field(m.nlocal, seed)
        w = ctx.ax(T(u, dev)).cpu().numpy()
        assert relerr(w, oracle.ax(N, G, u)) <= 1e-12, (N, eps, seed)
    assert ctx.launch_count >= 4


@pytest.mark.parametrize("N,elems", [(7, (8, 8, 8)), (3, (13, 7, 5)), (4, (9, 5, 3)),
                                     (6, (7, 5, 3)), (2, (11, 9, 7)), (10, (3, 3, 3)),
                                     # many persistent-CTA rounds; spare lanes in every
                                     # group (EPG n^2 < GT) on the last CTA's last group
                                     (4, (21, 21, 21)), (5, (17, 17, 17)), (6, (15, 15, 13))])
def test_ax_parity_many_elements(dev, impl, N, elems):
    m, G, J, ctx = make(N, elems, 0.05)
    u = meshgen.random_field(m.nlocal, 11)
    w = ctx.ax(T(u, dev)).cpu().numpy()
    assert relerr(w, oracle.ax(N, G, u)) <= 1e-12


@pytest.mark.parametrize("N", [1, 4, 7, 15])
def test_ax_annihilates_constants_and_is_symmetric(dev, N):
    m, G, J, ctx = make(N, (2, 2, 1), 0.1)
    one = torch.ones(m.nlocal, dtype=torch.float64, device=dev)
    w = ctx.ax(one).cpu().numpy()
    scale = np.abs(ctx.ax(T(meshgen.random_field(m.nlocal, 0), dev)).cpu().numpy()).max()
    assert np.abs(w).max() <= 1e-12 * scale
    # (A u, v) == (u, A v) element-wise symmetric
    u = meshgen.random_field(m.nlocal, 1)
    v = meshgen.random_field(m.nlocal, 2)
    Au = ctx.ax(T(u, dev)).cpu().numpy()
    Av = ctx.ax(T(v, dev)).cpu().numpy()
    assert abs(Au @ v - u @ Av) <= 1e-12 * np.abs(Au @ v)
    assert u @ Au >= 0.0


def test_ax_support_pattern_on_device(dev):
    for N, eps, expect in ((4, 0.0, 3 * 4 + 1), (4, 0.1, 3 * 25 - 15 + 1)):
        m, G, J, ctx = make(N, (1, 1, 1) if eps == 0 else (2, 2, 2), eps)
        n = N + 1
        e = np.zeros(m.nlocal)
        e[1 + n + n * n] = 1.0
        w = ctx.ax(T(e, dev)).cpu().numpy()[: n ** 3]
        assert np.count_nonzero(np.abs(w) > 1e-14) == expect


# --- DSSUM / mask / mass --------------------------------------------------
@pytest.mark.parametrize("N,elems", [(1, (3, 2, 2)), (4, (2, 2, 2)), (7, (8, 8, 8)),
                                     (2, (5, 3, 4)), (15, (2, 1, 2))])
def test_dssum_parity(dev, N, elems):
    m, G, J, ctx = make(N, elems, 0.05)
    v = meshgen.random_field(m.nlocal, 4)
    t = T(v, dev)
    ctx.dssum(t)
    ref = oracle.dssum(m.glo, v)
    got = t.cpu().numpy()
    assert relerr(got, ref) <= 1e-12
    # copies summed in ascending local order, plain adds: bit-identical
    np.testing.assert_array_equal(got, ref)
    # multiplicity
    one = torch.ones(m.nlocal, dtype=torch.float64, device=dev)
    ctx.dssum(one)
    np.testing.assert_array_equal(one.cpu().numpy(), oracle.multiplicity(m.glo))


def test_mask_and_mass(dev):
    N = 5
    m, G, J, ctx = make(N, (3, 2, 2), 0.05)
    v = meshgen.random_field(m.nlocal, 6)
    t = T(v, dev)
    ctx.mask(t)
    np.testing.assert_array_equal(t.cpu().numpy(), v * (1 - m.dirichlet.reshape(-1)))
    _, f = meshgen.manufactured(m)
    b = ctx.rhs(T(f, dev)).cpu().numpy()
    bref = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)
    assert relerr(b, bref) <= 1e-13


# --- CG -------------------------------------------------------------------
def _rhs(m, J, kind="sin"):
    if kind == "sin":
        _, f = meshgen.manufactured(m)
    else:
        f = meshgen.random_field(m.nlocal, 9)
    return oracle.mass_rhs(m.N, m.glo, m.dirichlet, J, f)


def test_cg_c1_twenty_iterations(dev, impl):
    """config c1: 2x2x2, N=4, 20 CG iterations (tol = 0) -> x_20 <= 1e-10."""
    m, G, J, ctx = make(4, (2, 2, 2), 0.05)
    b = _rhs(m, J)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=0.0, maxit=20)
    xr, its_r, rel_r, st = oracle.cg(4, m.glo, m.dirichlet, G, b, tol=0.0, maxit=20)
    assert its == its_r == 20 and ok
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    assert abs(rel - rel_r) <= 1e-8 * rel_r


@pytest.mark.parametrize("N,elems,eps,kind", [
    (4, (2, 2, 2), 0.0, "sin"), (4, (2, 2, 2), 0.05, "sin"), (4, (2, 2, 2), 0.05, "rand"),
    (7, (8, 8, 8), 0.05, "sin"), (3, (5, 4, 3), 0.05, "rand"), (2, (3, 3, 3), 0.0, "rand"),
    (9, (2, 3, 2), 0.05, "sin")])
def test_cg_iteration_parity(dev, impl, N, elems, eps, kind):
    m, G, J, ctx = make(N, elems, eps)
    b = _rhs(m, J, kind)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=2000)
    xr, its_r, rel_r, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=2000)
    assert ok and st == 0
    assert its == its_r, (its, its_r, rel, rel_r)
    assert relerr(x.cpu().numpy(), xr) <= 1e-10


def test_cg_edge_cases(dev, impl):
    m, G, J, ctx = make(3, (2, 2, 2), 0.05)
    b = _rhs(m, J)
    # zero RHS
    x, its, rel, ok = ctx.cg(torch.zeros(m.nlocal, dtype=torch.float64, device=dev), tol=1e-8,
                             maxit=10)
    assert its == 0 and rel == 0.0 and ok and not x.any()
    # maxit = 0
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=0)
    assert its == 0 and not ok and rel == 1.0
    # maxit hit -> not converged, iters == maxit, x == oracle's 5th iterate
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-12, maxit=5)
    xr, its_r, rel_r, st = oracle.cg(3, m.glo, m.dirichlet, G, b, tol=1e-12, maxit=5)
    assert its == its_r == 5 and not ok and st == 4
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    # warm start x0 != 0
    x0 = meshgen.random_field(m.nlocal, 3) * 0.01
    x0 = oracle.dssum(m.glo, x0) / oracle.multiplicity(m.glo)   # continuous
    x, its, rel, ok = ctx.cg(T(b, dev), x=T(x0, dev), tol=1e-9, maxit=500)
    xr, its_r, rel_r, st = oracle.cg(3, m.glo, m.dirichlet, G, b, x0=x0, tol=1e-9, maxit=500)
    assert ok and its == its_r
    assert relerr(x.cpu().numpy(), xr) <= 1e-10
    # repeated solves on one context give identical results (deterministic)
    x1, i1, r1, _ = ctx.cg(T(b, dev), tol=1e-8, maxit=500)
    x2, i2, r2, _ = ctx.cg(T(b, dev), tol=1e-8, maxit=500)
    assert i1 == i2 and r1 == r2 and torch.equal(x1, x2)


def test_cg_polynomial_reproduction_on_device(dev):
    m, G, J, ctx = make(4, (2, 2, 2), 0.0)
    us, f = meshgen.cube_poly(m)
    b = oracle.mass_rhs(4, m.glo, m.dirichlet, J, f)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-14, maxit=500)
    assert ok and np.abs(x.cpu().numpy() - us).max() <= 1e-13


def test_bad_arguments_raise(dev):
    from paper_1403_0968_b200 import sem
    m, G, J, ctx = make(2, (1, 1, 1), 0.0)
    with pytest.raises(ValueError):
        ctx.ax(torch.zeros(5, dtype=torch.float64, device=dev))
    with pytest.raises(TypeError):
        ctx.ax(torch.zeros(m.nlocal, dtype=torch.float32, device=dev))
    with pytest.raises(TypeError):
        ctx.ax(torch.zeros(m.nlocal, dtype=torch.float64))
    u = torch.zeros(m.nlocal, dtype=torch.float64, device=dev)
    ptr = sem.ctypes.c_void_p(u.data_ptr())
    assert sem.lib().sem_ax(ctx._ctx, ptr, ptr) == sem.SEM_EINVAL   # u, w alias


@pytest.mark.parametrize("N", [2, 7, 13])
def test_8_byte_offset_vectors_rejected(dev, N):
    """include/sem.h: vectors must be 16-byte aligned (bulk copies, 128-bit
    accesses); an 8-byte-offset view is refused with SEM_EINVAL before any
    launch, and the context stays usable."""
    from paper_1403_0968_b200 import sem
    m, G, J, ctx = make(N, (2, 1, 1), 0.05)
    big = torch.zeros(2 * m.nlocal + 2, dtype=torch.float64, device=dev)
    u, w = big[1:m.nlocal + 1], big[m.nlocal + 2:]
    assert u.data_ptr() % 16 == 8
    for fn in (lambda: ctx.ax(u, w), lambda: ctx.dssum(u), lambda: ctx.cg(u, w, tol=1e-8)):
        with pytest.raises(sem.SemError) as ei:
            fn()
        assert ei.value.code == sem.SEM_EINVAL
    uu = meshgen.random_field(m.nlocal, 3)
    assert relerr(ctx.ax(T(uu, dev)).cpu().numpy(), oracle.ax(N, G, uu)) <= 1e-12


# --- full-size configuration c3 (4096 el, N=7, eps=0.05), as bench.py runs it ---
@pytest.fixture(scope="module")
def c3(dev):
    from paper_1403_0968_b200 import sem
    N = 7
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(16, 16, 16), eps=0.05)
    G, J = oracle.geom(N, m.xyz)
    ctx = sem.Context(m, N, device=0)
    return m, G, J, ctx


def test_c3_ax_and_dssum_full_size(dev, c3):
    m, G, J, ctx = c3
    u = meshgen.random_field(m.nlocal, 21)
    w = ctx.ax(T(u, dev))
    wr = oracle.ax(7, G, u)
    assert relerr(w.cpu().numpy(), wr) <= 1e-12
    ctx.dssum(w)
    assert relerr(w.cpu().numpy(), oracle.dssum(m.glo, wr)) <= 1e-12


# (the full-size c3 CG solve: tests/test_gpu_c3_parity.py, drift rule)


# --- the same discretisation presented differently (meshgen.relabel): random
# element order, quarter-turned elements, non-compact global ids ---
@pytest.mark.parametrize("N,elems", [(3, (4, 3, 3)), (7, (4, 4, 3)), (12, (2, 2, 2))])
def test_relabelled_mesh_parity(dev, impl, N, elems):
    from paper_1403_0968_b200 import sem
    xi, _ = oracle.gll(N)
    m = meshgen.relabel(meshgen.box_mesh(N, xi, elems=elems, eps=0.05), seed=N)
    G, J = oracle.geom(N, m.xyz)
    ctx = sem.Context(m, N, device=0)
    u = meshgen.random_field(m.nlocal, 1)
    w = ctx.ax(T(u, dev))
    wr = oracle.ax(N, G, u)
    assert relerr(w.cpu().numpy(), wr) <= 1e-12
    ctx.dssum(w)
    assert relerr(w.cpu().numpy(), oracle.dssum(m.glo, wr)) <= 1e-12
    _, f = meshgen.manufactured(m)
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)
    x, its, rel, ok = ctx.cg(T(b, dev), tol=1e-8, maxit=3000)
    xr, its_r, rel_r, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=3000)
    assert ok and st == 0 and its == its_r, (its, its_r)
    assert relerr(x.cpu().numpy(), xr) <= 1e-10


@pytest.mark.parametrize("extra", [0, 4])
def test_dmma_plain_w_selection_boundary(dev, monkeypatch, extra):
    """The N = 7 plain Ax picks two warps per element (three groups per SM) for
    meshes of at most 4 x SMs elements and four warps above (ax_dmma.cuh
    launch_dmma_plain): both sides of the boundary against the oracle."""
    monkeypatch.delenv("SEM_DMMA_W", raising=False)
    monkeypatch.delenv("SEM_AX_KERNEL", raising=False)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    E = 4 * nsm + extra
    m, G, J, ctx = make(7, (E // 4, 4, 1), 0.05)
    assert m.nelem == E
    u = meshgen.random_field(m.nlocal, 5)
    w = ctx.ax(T(u, dev))
    assert relerr(w.cpu().numpy(), oracle.ax(7, G, u)) <= 1e-12
    ctx.free()
