"""Config c4 at full size (BASELINE.json configs[3]: ~16.8 M local DOF,
e = round(256/n) elements per side, the order sweep of tools/order_sweep.py)
in the launch configuration the sweep times (the default kernel for each N:
tensor-core kernels at N = 7 and 10..15, CUDA-core TMA kernels otherwise):
Ax on the whole mesh, checked against the oracle on a random sample of
elements (the oracle's operator is element-local, so G^ is formed for the
sampled elements only).  Bar: rel-L2 <= 1e-12 on the sample."""
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


@pytest.mark.parametrize("N", [3, 6, 7, 8, 10, 11, 12, 13, 15])
def test_c4_full_size_ax_sampled(dev, N, monkeypatch):
    from paper_1403_0968_b200 import sem
    monkeypatch.delenv("SEM_AX_KERNEL", raising=False)
    monkeypatch.delenv("SEM_DMMAG", raising=False)
    n = N + 1
    e = round(256 / n)
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=(e, e, e), eps=0.05)
    ctx = sem.Context(m, N, device=0)
    u = meshgen.random_field(m.nlocal, N)
    w = ctx.ax(torch.from_numpy(u).to(dev)).cpu().numpy().reshape(m.nelem, -1)
    rng = np.random.default_rng(100 + N)
    idx = np.sort(np.concatenate([[0, m.nelem - 1], rng.choice(m.nelem, 62, replace=False)]))
    G, _ = oracle.geom(N, m.xyz[idx])
    ref = oracle.ax(N, G, u.reshape(m.nelem, -1)[idx]).reshape(len(idx), -1)
    err = np.linalg.norm(w[idx] - ref) / np.linalg.norm(ref)
    assert err <= 1e-12, (N, err)
    ctx.free()
