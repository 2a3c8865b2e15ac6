"""GPU parity of the finite-difference wave-equation step (NEXT-4, SURVEY.md
§8(f); lst:fdCode PAPER.md:418-449): libsem's fd2d_step / fd2d_run through the
C ABI (include/fd.h) against the oracle's ora_fd_step on the same seeded
inputs and the same weights.

* fd2d_step / fd2d_run (the default, any weights -- the central stencils of
  fd_weights included): the kernel evaluates the listing's operations in the
  same order without FMA contraction -> BIT-EXACT equality.
* fd2d_run_ex(FD_REGROUPED), symmetric weights only: the pair-regrouped FMA
  kernel (reading R6c) -> within the rounding bound
  (4r + 8) eps (2|u1| + |u2| + dt^2 sum|omega| 2 max|u1|), eps = 2^-53."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1403_0968_b200 import fd
    fd.lib()
    return torch.device("cuda", 0)


def fields(h, w, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1, 1, (h, w)), rng.uniform(-1, 1, (h, w))


def T(a, dev):
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def asym(om):
    """The same weights with omega_{+r} nudged (not symmetric)."""
    om = om.copy()
    om[-1] *= 1.0 + 2.0 ** -20
    return om


def sym_bound(u1, u2, om, dt):
    r = om.size // 2
    scale = 2 * np.abs(u1) + np.abs(u2) + dt * dt * np.abs(om).sum() * 2 * np.abs(u1).max()
    return (4 * r + 8) * 2.0 ** -53 * scale


SHAPES = [(64, 256), (100, 300), (37, 513), (129, 17), (15, 15), (70, 1024)]


@pytest.mark.parametrize("r", range(1, 8))
@pytest.mark.parametrize("h,w", SHAPES)
@pytest.mark.parametrize("weights", ["central", "asym"])
def test_fd_step_bit_exact(dev, r, h, w, weights):
    from paper_1403_0968_b200 import fd
    if min(h, w) < 2 * r + 1:
        pytest.skip("grid smaller than the stencil")
    u1, u2 = fields(h, w, r * 1000 + h + w)
    om = oracle.fd_weights(r, 2.0 / w)
    if weights == "asym":
        om = asym(om)
    dt = 0.3 * 2.0 / w
    ref = oracle.fd_step(u1, u2, om, dt)
    u3 = torch.empty((h, w), dtype=torch.float64, device=dev)
    fd.step(T(u1, dev), T(u2, dev), u3, om, dt)
    np.testing.assert_array_equal(u3.cpu().numpy(), ref)


@pytest.mark.parametrize("r", range(1, 8))
@pytest.mark.parametrize("h,w", SHAPES)
def test_fd_regrouped_within_rounding(dev, r, h, w):
    from paper_1403_0968_b200 import fd
    if min(h, w) < 2 * r + 1:
        pytest.skip("grid smaller than the stencil")
    u1, u2 = fields(h, w, r * 7 + h + w)
    om = oracle.fd_weights(r, 2.0 / w)
    dt = 0.3 * 2.0 / w
    ref = oracle.fd_step(u1, u2, om, dt)
    u3 = torch.empty((h, w), dtype=torch.float64, device=dev)
    new, _ = fd.run(T(u1, dev), T(u2, dev), u3, om, dt, 1, regrouped=True)
    assert new is u3
    err = np.abs(u3.cpu().numpy() - ref)
    assert np.all(err <= sym_bound(u1, u2, om, dt)), err.max()


def test_fd_regrouped_rejects_asymmetric_weights(dev):
    from paper_1403_0968_b200 import fd, sem
    h, w, r = 32, 64, 3
    u1, u2 = fields(h, w, 1)
    g = [T(u1, dev), T(u2, dev), torch.empty((h, w), dtype=torch.float64, device=dev)]
    with pytest.raises(sem.SemError) as ei:
        fd.run(*g, asym(oracle.fd_weights(r, 2.0 / w)), 0.01, 1, regrouped=True)
    assert ei.value.code == sem.SEM_EINVAL


@pytest.mark.parametrize("r", [1, 3, 7])
def test_fd_run_rotation_bit_exact(dev, r):
    """Several steps with the (u1, u2, u3) <- (u3, u1, u2) rotation (R6b)."""
    from paper_1403_0968_b200 import fd
    h, w, steps = 96, 320, 5
    u1, u2 = fields(h, w, 7 + r)
    om = asym(oracle.fd_weights(r, 2.0 / w))
    dt = 0.25 * 2.0 / w
    a, b = u1.copy(), u2.copy()
    for _ in range(steps):
        a, b = oracle.fd_step(a, b, om, dt), a
    g1, g2 = T(u1, dev), T(u2, dev)
    g3 = torch.empty_like(g1)
    new, prev = fd.run(g1, g2, g3, om, dt, steps)
    np.testing.assert_array_equal(new.cpu().numpy(), a)
    np.testing.assert_array_equal(prev.cpu().numpy(), b)
    # zero steps: nothing moves
    new0, prev0 = fd.run(g1, g2, g3, om, dt, 0)
    assert new0 is g1 and prev0 is g2


def test_fd_full_size_r7(dev):
    """The benchmark grid (8192 x 8192, stencil size 15): the default kernel
    bench.py --workload fd times bit-exact with the central weights, the
    regrouped variant within the rounding bound everywhere."""
    from paper_1403_0968_b200 import fd
    h = w = 8192
    r = 7
    u1, u2 = fields(h, w, 99)
    om = oracle.fd_weights(r, 2.0 / w)
    dt = 0.2 * 2.0 / w
    ref = oracle.fd_step(u1, u2, om, dt)
    g1, g2 = T(u1, dev), T(u2, dev)
    u3 = torch.empty((h, w), dtype=torch.float64, device=dev)
    fd.step(g1, g2, u3, om, dt)
    np.testing.assert_array_equal(u3.cpu().numpy(), ref)
    fd.run(g1, g2, u3, om, dt, 1, regrouped=True)
    assert np.all(np.abs(u3.cpu().numpy() - ref) <= sym_bound(u1, u2, om, dt))


def test_fd_library_weights_drive_the_kernel(dev):
    """The library's own (Fornberg) weights, used end to end: bit-exact with
    the oracle's step on the same weights, and within rounding of the oracle's
    closed-form weights."""
    from paper_1403_0968_b200 import fd
    h, w, r = 64, 512, 5
    u1, u2 = fields(h, w, 5)
    om_lib = fd.weights(r, 2.0 / w)
    om_ora = oracle.fd_weights(r, 2.0 / w)
    dt = 0.3 * 2.0 / w
    u3 = torch.empty((h, w), dtype=torch.float64, device=dev)
    fd.step(T(u1, dev), T(u2, dev), u3, om_lib, dt)
    np.testing.assert_array_equal(u3.cpu().numpy(), oracle.fd_step(u1, u2, om_lib, dt))
    ref = oracle.fd_step(u1, u2, om_ora, dt)
    np.testing.assert_allclose(u3.cpu().numpy(), ref, rtol=0, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("r", [1, 3, 7])
@pytest.mark.parametrize("h,w", [(17, 17), (32, 32), (48, 64)])
def test_fd_run_default_weights_bit_exact(dev, r, h, w):
    """10 steps with the library's central weights on SPEC.md's shapes: the
    default path is bit-exact with the oracle (no regrouping
    unless asked for)."""
    from paper_1403_0968_b200 import fd
    if min(h, w) < 2 * r + 1:
        pytest.skip("grid smaller than the stencil")
    steps = 10
    u1, u2 = fields(h, w, 3 + r + h)
    om = fd.weights(r, 2.0 / w)
    dt = 0.25 * 2.0 / w
    a, b = u1.copy(), u2.copy()
    for _ in range(steps):
        a, b = oracle.fd_step(a, b, om, dt), a
    g1, g2 = T(u1, dev), T(u2, dev)
    new, prev = fd.run(g1, g2, torch.empty_like(g1), om, dt, steps)
    np.testing.assert_array_equal(new.cpu().numpy(), a)
    np.testing.assert_array_equal(prev.cpu().numpy(), b)


@pytest.mark.parametrize("r", [2, 7])
def test_fd_run_regrouped(dev, r):
    from paper_1403_0968_b200 import fd
    h, w, steps = 64, 512, 4
    u1, u2 = fields(h, w, 3 + r)
    om = oracle.fd_weights(r, 2.0 / w)
    dt = 0.25 * 2.0 / w
    a, b = u1.copy(), u2.copy()
    for _ in range(steps):
        a, b = oracle.fd_step(a, b, om, dt), a
    g1, g2 = T(u1, dev), T(u2, dev)
    new, prev = fd.run(g1, g2, torch.empty_like(g1), om, dt, steps, regrouped=True)
    # the literal update amplifies (|-2 - dt^2 s| > 1): bound relative to the size
    np.testing.assert_allclose(new.cpu().numpy(), a, rtol=0, atol=1e-12 * np.abs(a).max())
    np.testing.assert_allclose(prev.cpu().numpy(), b, rtol=0, atol=1e-12 * np.abs(b).max())


def test_fd_concurrent_streams_different_weights(dev):
    """Two streams with different radii and weights interleaved: each result
    bit-exact (omega travels with the launch, no shared __constant__ state)."""
    from paper_1403_0968_b200 import fd
    h, w = 96, 512
    outs = []
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    jobs = []
    for q, r in enumerate((2, 6)):
        u1, u2 = fields(h, w, 40 + q)
        om = asym(oracle.fd_weights(r, 2.0 / w))
        g = [T(u1, dev), T(u2, dev), torch.empty((h, w), dtype=torch.float64, device=dev)]
        jobs.append((u1, u2, om, g))
    torch.cuda.synchronize()
    for _ in range(20):
        for (u1, u2, om, g), st in zip(jobs, streams):
            fd.step(g[0], g[1], g[2], om, 0.01, stream=st)
    torch.cuda.synchronize()
    for u1, u2, om, g in jobs:
        np.testing.assert_array_equal(g[2].cpu().numpy(), oracle.fd_step(u1, u2, om, 0.01))
