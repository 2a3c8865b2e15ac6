"""Multi-rank device path on ONE GPU (PAPER.md:667
global-local numbering): P = 2, 4, 8 ranks as P contexts of this process, one
host thread and one stream each, joined by libsem's in-process loopback
transport (include/sem.h sem_loopback_unique_id).  What runs is the library's
multi-rank code -- exchange plan, pack / combine kernels, rank-ordered sums,
the boundary/interior K1 split with the exchange on the side stream, the
multi-rank CG prologues and the rank folds (cg_red / sr_fold) -- with
device-to-device copies where NCCL would move the bytes.

Bars:
* partitioned DSSUM bit-identical to the rank-ordered sum of the oracle's
  per-rank partial sums (O5 "virtual partition independence": each rank sums
  its own copies in ascending local order, ranks are added in ascending rank
  order -- SURVEY.md G16), and rel-L2 <= 1e-12 against the unpartitioned
  oracle;
* Ax per rank rel-L2 <= 1e-12 against the oracle (elements are independent);
* CG / Jacobi PCG / single-reduction CG: the same iteration count as the
  oracle on the full mesh and as the one-rank GPU solve, x rel-L2 <= 1e-10,
  every rank reporting the same count, residual and nglobal.
Inputs: meshgen boxes partitioned as 1x1x2 / 1x2x2 / 2x2x2 blocks (c5's
partition), the oracle's GLL nodes; no expected value comes from the CUDA path.

The peer-memory transport (SEM_COMM=p2p) runs the same checks in a fresh
process: tests/test_gpu_p2p.py.
"""
import numpy as np
import pytest

import oracle
from paper_1403_0968_b200 import meshgen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(autouse=True)
def host_transport(monkeypatch):
    monkeypatch.delenv("SEM_COMM", raising=False)


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


def _key(eidx, elems):
    ex, ey, _ = elems
    return eidx[:, 0] + ex * (eidx[:, 1] + ey * eidx[:, 2])


def partition(N, elems, P, eps=0.05, boundary_first=True):
    """Full mesh (element order a fastest) and the P rank meshes, with each
    rank's element positions in the full mesh."""
    xi, _ = oracle.gll(N)
    full = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    parts = meshgen.default_parts(P)
    ranks = [meshgen.box_mesh(N, xi, elems=elems, eps=eps, parts=parts, rank=r,
                              boundary_first=boundary_first) for r in range(P)]
    pos = [_key(m.eidx, elems) for m in ranks]
    for m, p in zip(ranks, pos):       # same discretisation, element by element
        assert np.array_equal(m.glo, full.glo[p])
        assert np.array_equal(m.xyz, full.xyz[p])
    return full, ranks, pos


def rank_ordered_dssum(ranks, vs):
    """Expected partitioned Q Q^T: per-rank oracle partial sums (ascending
    local order), added across ranks in ascending rank order."""
    top = max(int(m.glo.max()) for m in ranks) + 1
    acc = np.zeros(top)
    seen = np.zeros(top, dtype=bool)
    for m, v in zip(ranks, vs):
        g = m.glo.reshape(-1)
        part = oracle.dssum(g, v)
        ids, first = np.unique(g, return_index=True)
        vals = part[first]
        acc[ids] = np.where(seen[ids], acc[ids] + vals, vals)
        seen[ids] = True
    return [acc[m.glo.reshape(-1)] for m in ranks]


def run_ranks(P, fn):
    from paper_1403_0968_b200 import dist as sdist
    return sdist.LoopbackGroup(P, device=0).run(fn)


def T(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)


CASES = [  # (N, global elements, P): TMA (N=3, 4), DMMA (N=7), high-order (N=11)
    (3, (4, 4, 4), 2), (3, (4, 4, 4), 8),
    (4, (2, 4, 4), 2), (4, (4, 4, 4), 4), (4, (4, 4, 4), 8),
    (7, (2, 2, 4), 2), (7, (4, 4, 4), 4), (7, (4, 4, 4), 8),
    (11, (2, 2, 4), 2), (11, (2, 4, 4), 4),
]


@pytest.mark.parametrize("N,elems,P", CASES)
@pytest.mark.parametrize("bfirst", [True, False])
def test_multirank_ax_dssum(dev, N, elems, P, bfirst):
    from paper_1403_0968_b200 import sem
    full, ranks, pos = partition(N, elems, P, boundary_first=bfirst)
    n3 = (N + 1) ** 3
    vfull = meshgen.random_field(full.nlocal, 5).reshape(full.nelem, n3)
    vs = [vfull[p].reshape(-1) for p in pos]
    G_full, _ = oracle.geom(N, full.xyz)
    ax_full = oracle.ax(N, G_full, vfull.reshape(-1)).reshape(full.nelem, n3)
    ds_full = oracle.dssum(full.glo.reshape(-1), vfull.reshape(-1)).reshape(full.nelem, n3)
    expect = rank_ordered_dssum(ranks, vs)

    def body(lr):
        m = ranks[lr.rank]
        ctx = sem.Context(m, N, device=0, loopback=lr)
        try:
            u = T(vs[lr.rank], dev)
            w = ctx.ax(u)
            d = ctx.dssum(u.clone())
            d2 = ctx.dssum(d.clone())          # a second exchange on the same buffers
            return (w.cpu().numpy(), d.cpu().numpy(), d2.cpu().numpy(), ctx.nglobal,
                    ctx.launch_count)
        finally:
            ctx.free()

    out = run_ranks(P, body)
    ng_full = int(np.unique(full.glo).size)
    for r, (w, d, d2, ng, nl) in enumerate(out):
        assert ng == ng_full
        assert relerr(w, ax_full[pos[r]].reshape(-1)) <= 1e-12
        np.testing.assert_array_equal(d, expect[r])
        assert relerr(d, ds_full[pos[r]].reshape(-1)) <= 1e-12
        # Q Q^T of an assembled field multiplies it by the global multiplicity
        mult = oracle.multiplicity(full.glo.reshape(-1)).reshape(full.nelem, n3)[pos[r]].reshape(-1)
        assert relerr(d2, mult * d) <= 1e-12
        assert nl > 0
    # every rank holds bit-identical values at the nodes it shares
    vals = {}
    for r, (_, d, _, _, _) in enumerate(out):
        for gid, v in zip(ranks[r].glo.reshape(-1), d):
            if gid in vals:
                assert vals[gid] == v
            vals[gid] = v


def _solve_all(dev, N, ranks, bs, method, tol, maxit):
    from paper_1403_0968_b200 import sem

    def body(lr):
        ctx = sem.Context(ranks[lr.rank], N, device=0, loopback=lr)
        try:
            b = T(bs[lr.rank], dev)
            kw = {}
            if method == "jacobi":
                kw["precond"] = "jacobi"
            elif method == "sr":
                kw["variant"] = "single_reduction"
            ctx.profile(True)                 # per-launch records: K1 launch count
            x, its, rel, ok = ctx.cg(b, tol=tol, maxit=maxit, **kw)
            k1 = ctx.profile_read()["k1"][1]
            ctx.profile(False)
            return x.cpu().numpy(), its, rel, ok, k1
        finally:
            ctx.free()

    return run_ranks(len(ranks), body)


def k1_split_expected(m):
    """The library splits K1 into a boundary and an interior launch when the
    elements holding interface copies, [0, nbnd), are not all of them; with
    meshgen's boundary-first order nbnd = nboundary (rounded up to even for
    odd n^3, the range launches' alignment)."""
    nb = int(m.nboundary)
    if ((m.N + 1) ** 3) & 1:
        nb += nb & 1
    return 0 < nb < m.nelem


def _oracle_solve(N, full, G, b, method, tol, maxit):
    if method == "sr":
        return oracle.cg_single_reduction(N, full.glo, full.dirichlet, G, b, tol=tol, maxit=maxit)
    return oracle.cg(N, full.glo, full.dirichlet, G, b, tol=tol, maxit=maxit,
                     precond="jacobi" if method == "jacobi" else "none")


CG_CASES = [
    (3, (4, 4, 4), 2), (3, (4, 4, 4), 8),
    (4, (4, 4, 4), 4), (4, (4, 4, 4), 8),
    (7, (2, 2, 4), 2), (7, (4, 4, 4), 8),
    (11, (2, 2, 4), 2),
]


@pytest.mark.parametrize("N,elems,P", CG_CASES)
@pytest.mark.parametrize("method", ["cg", "jacobi", "sr"])
def test_multirank_cg(dev, N, elems, P, method):
    from paper_1403_0968_b200 import sem
    full, ranks, pos = partition(N, elems, P)
    n3 = (N + 1) ** 3
    G, J = oracle.geom(N, full.xyz)
    _, f = meshgen.manufactured(full)
    b = oracle.mass_rhs(N, full.glo, full.dirichlet, J, f).reshape(full.nelem, n3)
    bs = [b[p].reshape(-1) for p in pos]
    tol, maxit = 1e-8, 2000
    xr, its_r, rel_r, st = _oracle_solve(N, full, G, b.reshape(-1), method, tol, maxit)
    assert st == 0
    xr = xr.reshape(full.nelem, n3)
    out = _solve_all(dev, N, ranks, bs, method, tol, maxit)
    # the one-rank GPU solve of the same system
    one = _solve_all(dev, N, [full], [b.reshape(-1)], method, tol, maxit)[0]
    nsplit = 0
    for r, (x, its, rel, ok, k1) in enumerate(out):
        assert ok
        assert its == its_r == one[1], (r, its, its_r, one[1])
        assert rel == out[0][2]
        assert relerr(x, xr[pos[r]].reshape(-1)) <= 1e-10
        if method != "sr":                   # the SR variant's KA is not split
            split = k1_split_expected(ranks[r])
            nsplit += split
            assert k1 == its * (2 if split else 1), (r, k1, its, split)
    if method != "sr" and P <= 4:
        assert nsplit > 0                    # the overlapped schedule really ran


@pytest.mark.parametrize("P", [2, 8])
def test_multirank_cg_fixed_iterations(dev, P):
    """c1-style fixed-count solve (tol = 0, 20 iterations) on a partitioned
    c1 mesh: x_20 against the oracle's, every rank."""
    N, elems = 4, (2, 2, 2)
    full, ranks, pos = partition(N, elems, P)
    n3 = (N + 1) ** 3
    G, J = oracle.geom(N, full.xyz)
    _, f = meshgen.manufactured(full)
    b = oracle.mass_rhs(N, full.glo, full.dirichlet, J, f).reshape(full.nelem, n3)
    xr, its_r, _, _ = oracle.cg(N, full.glo, full.dirichlet, G, b.reshape(-1), tol=0.0, maxit=20)
    out = _solve_all(dev, N, ranks, [b[p].reshape(-1) for p in pos], "cg", 0.0, 20)
    xr = xr.reshape(full.nelem, n3)
    for r, (x, its, _, _, _) in enumerate(out):
        assert its == its_r == 20
        assert relerr(x, xr[pos[r]].reshape(-1)) <= 1e-10


def test_loopback_peer_failure_times_out(dev, monkeypatch):
    """A rank that never joins the collective makes its peer fail with
    SEM_ENCCL after the timeout instead of hanging (failure detection)."""
    from paper_1403_0968_b200 import dist as sdist
    from paper_1403_0968_b200 import sem
    monkeypatch.setenv("SEM_LOOPBACK_TIMEOUT_MS", "2000")
    full, ranks, pos = partition(4, (2, 2, 2), 2)
    grp = sdist.LoopbackGroup(2, device=0)
    res = {}

    def body(lr):
        ctx = sem.Context(ranks[lr.rank], 4, device=0, loopback=lr)
        try:
            if lr.rank == 0:
                u = T(meshgen.random_field(ctx.nlocal, 1), dev)
                try:
                    ctx.dssum(u)
                    res["rc"] = 0
                except sem.SemError as e:
                    res["rc"] = e.code
            return None
        finally:
            if lr.rank == 0:
                ctx.free()
            else:
                res["peer"] = ctx       # rank 1 skips the collective (freed below)

    grp.run(body)
    res.pop("peer").free()
    assert res["rc"] == sem.SEM_ENCCL
