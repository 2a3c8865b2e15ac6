"""The two K1 schedules at N >= 8: the split K1 (k1u_kernel's
x / p update with the scalar prologue, then the tensor-core operator with the
(p, A p) partials accumulated in phase A) -- the default at N >= 11, forced
here at N = 8..10 -- and the fused CUDA-core K1 (forced at N >= 11 with
SEM_K1_AX=fused), each against the oracle: CG and Jacobi PCG with identical
iteration counts, x within 1e-10, on small deformed meshes and on a
relabelled one (quarter-turned elements, non-compact ids).  Also the split
with the CUDA-core operator (the TMA / high-order Ax kernels with the DOT
flag; the default at N = 9, forced at other orders without SEM_DMMAG)."""
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
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("N,mode", [(8, "split"), (9, "split"), (10, "split"), (11, "fused"),
                                    (12, "split"), (13, "fused"), (15, "split"), (15, "fused"),
                                    (3, "cudacore-split"), (6, "cudacore-split"), (8, "cudacore-split"),
                                    (9, "cudacore-default"), (9, "cudacore-fused"),
                                    (11, "cudacore-split")])
@pytest.mark.parametrize("relabel", [False, True])
def test_k1_schedules(dev, monkeypatch, N, mode, relabel):
    from paper_1403_0968_b200 import sem
    if mode.startswith("cudacore"):
        monkeypatch.setenv("SEM_DMMAG", "0")
        sub = mode.split("-")[1]
        if sub == "default":
            monkeypatch.delenv("SEM_K1_AX", raising=False)
        else:
            monkeypatch.setenv("SEM_K1_AX", sub)
    else:
        monkeypatch.setenv("SEM_DMMAG", "1")
        monkeypatch.setenv("SEM_K1_AX", mode)
    monkeypatch.delenv("SEM_AX_KERNEL", raising=False)
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(2, 2, 1) if N >= 12 else (3, 2, 2), eps=0.05)
    if relabel:
        m = meshgen.relabel(m, seed=N)
    G, J = oracle.geom(N, m.xyz)
    ctx = sem.Context(m, N, device=0)
    _, f = meshgen.manufactured(m)
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)
    bd = torch.from_numpy(b).to(dev)
    for precond in ("none", "jacobi"):
        x, its, rel, ok = ctx.cg(bd, tol=1e-8, maxit=3000, precond=precond)
        with oracle.history() as h:
            xr, its_r, rel_r, st = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=3000,
                                             precond=precond)
        assert ok and st == 0

        def solve(k, precond=precond):
            _, it, rl, _ = ctx.cg(bd, tol=0.0, maxit=k, precond=precond)
            return it, rl

        meth = "jacobi" if precond == "jacobi" else "cg"
        dr = _margin.drift(_margin.gpu_history(solve, its_r), h.values)
        assert dr <= _margin.DRIFT_MAX[meth], (precond, dr)
        _margin.assert_count(its, its_r, _margin.margin(h.values, its_r, 1e-8), dr,
                             (precond, rel, rel_r))
        if its == its_r:
            assert relerr(x.cpu().numpy(), xr) <= 1e-10
    # fixed count: x_20 (no stopping decision involved)
    x, its, _, _ = ctx.cg(bd, tol=0.0, maxit=20)
    xr, _, _, _ = oracle.cg(N, m.glo, m.dirichlet, G, b, tol=0.0, maxit=20)
    assert its == 20 and relerr(x.cpu().numpy(), xr) <= 1e-10
