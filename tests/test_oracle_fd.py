"""Pins for the oracle's finite-difference wave-equation step (NEXT-4,
SURVEY.md §8(f), alg:fdPseudocode, lst:fdCode).

Pinned by: the weights against an independent numpy solve of the moment
(Taylor) conditions and exactness on polynomials of degree <= 2r+1 (reading
R6); the step against a dense periodic-shift route, a Fourier-mode closed form,
the constant-field value, and a hand-computed delta example (SPEC.md:261's
16x16, r=1, dt=0.1 case)."""
import numpy as np
import pytest


def _moment_weights(r, dx):
    """Solve sum_k omega_k (k dx)^p = 2 [p == 2], p = 0..2r (numpy)."""
    ks = np.arange(-r, r + 1, dtype=np.float64) * dx
    A = np.vander(ks, 2 * r + 1, increasing=True).T        # A[p, k] = (k dx)^p
    rhs = np.zeros(2 * r + 1)
    rhs[2] = 2.0
    return np.linalg.solve(A, rhs)


@pytest.mark.parametrize("r", range(1, 8))
@pytest.mark.parametrize("dx", [1.0, 0.01])
def test_weights_moment_conditions(oracle, r, dx):
    w = oracle.fd_weights(r, dx)
    ref = _moment_weights(r, dx)
    np.testing.assert_allclose(w, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())
    assert abs(w.sum()) <= 1e-12 * np.abs(w).max()
    np.testing.assert_array_equal(w, w[::-1])


@pytest.mark.parametrize("r", range(1, 8))
def test_weights_exact_on_polynomials(oracle, r):
    dx = 0.1
    w = oracle.fd_weights(r, dx)
    x0 = 0.3
    ks = np.arange(-r, r + 1) * dx
    for p in range(0, 2 * r + 2):
        approx = np.dot(w, (x0 + ks) ** p)
        exact = p * (p - 1) * x0 ** (p - 2) if p >= 2 else 0.0
        assert abs(approx - exact) <= 1e-6 * max(1.0, abs(exact)), (r, p)
    # and not for degree 2r+2 (the order is exactly 2r)
    p = 2 * r + 2
    assert abs(np.dot(w, (x0 + ks) ** p) - p * (p - 1) * x0 ** (p - 2)) > 1e-12


def test_closed_weights_r1_r2(oracle):
    np.testing.assert_array_equal(oracle.fd_weights(1, 1.0), [1.0, -2.0, 1.0])
    np.testing.assert_allclose(oracle.fd_weights(2, 1.0) * 12, [-1, 16, -30, 16, -1], rtol=1e-15)


def _dense_step(u1, u2, w, dt):
    """lap via periodic shifts (np.roll), summed over k."""
    r = w.size // 2
    lap = np.zeros_like(u1)
    for k in range(-r, r + 1):
        lap += w[r + k] * np.roll(u1, -k, axis=1) + w[r + k] * np.roll(u1, -k, axis=0)
    return -2 * u1 + u2 - dt * dt * lap


@pytest.mark.parametrize("r,h,w", [(1, 16, 16), (3, 17, 29), (7, 40, 15), (5, 11, 64)])
def test_step_dense_route(oracle, r, h, w):
    rng = np.random.default_rng(r)
    u1 = rng.uniform(-1, 1, (h, w))
    u2 = rng.uniform(-1, 1, (h, w))
    wt = oracle.fd_weights(r, 2.0 / w)
    got = oracle.fd_step(u1, u2, wt, 1e-3)
    np.testing.assert_allclose(got, _dense_step(u1, u2, wt, 1e-3), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("r", [1, 4, 7])
def test_step_fourier_mode(oracle, r):
    h, w, mx, my = 24, 36, 5, 3
    dx, dt = 2.0 / w, 0.002
    wt = oracle.fd_weights(r, dx)
    j, i = np.meshgrid(np.arange(h), np.arange(w), indexing="ij")
    u1 = np.cos(2 * np.pi * (mx * i / w + my * j / h))
    u2 = np.sin(2 * np.pi * (i / w)) * 0.5
    ks = np.arange(-r, r + 1)
    sx = np.dot(wt, np.cos(2 * np.pi * mx * ks / w))
    sy = np.dot(wt, np.cos(2 * np.pi * my * ks / h))
    ref = (-2.0 - dt * dt * (sx + sy)) * u1 + u2
    np.testing.assert_allclose(oracle.fd_step(u1, u2, wt, dt), ref, rtol=0, atol=1e-12)


def test_step_constant_field(oracle):
    wt = oracle.fd_weights(4, 0.05)
    c = 0.75
    u = np.full((20, 20), c)
    got = oracle.fd_step(u, u, wt, 0.01)
    np.testing.assert_allclose(got, -c, rtol=0, atol=1e-12)


def test_step_delta_example(oracle):
    """16x16, r=1, omega = {1,-2,1}, dt = 0.1, u1 = u2 = delta at (8,8):
    center lap = -4 -> u3 = -2 + 1 + 0.04 = -0.96; the 4 neighbours lap = 1 ->
    u3 = -0.01; every other node 0 (worked by hand from lst:fdCode)."""
    u = np.zeros((16, 16))
    u[8, 8] = 1.0
    got = oracle.fd_step(u, u, np.array([1.0, -2.0, 1.0]), 0.1)
    ref = np.zeros((16, 16))
    ref[8, 8] = -0.96
    for (a, b) in ((7, 8), (9, 8), (8, 7), (8, 9)):
        ref[a, b] = -0.01
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-15)
    assert np.count_nonzero(got) == 5


def test_step_rejects_bad_sizes(oracle):
    with pytest.raises(oracle.OracleError):
        oracle.fd_step(np.zeros((4, 4)), np.zeros((4, 4)), oracle.fd_weights(3, 1.0), 0.1)
