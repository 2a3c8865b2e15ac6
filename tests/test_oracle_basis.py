"""Pins for oracle O1 (GLL nodes/weights) and O2 (differentiation matrix).

PAPER.md:599 (GLL basis), :608/:614 (weights), :618-625 (phi').  Pinned by
closed forms (tests/golden/gll_closed_forms.json), quadrature exactness,
an independent numpy root finder, exactness of D on P_N, D 1 = 0, the
summation-by-parts identity and the closed-form 1-D stiffness matrices.
"""
import json
import math
import os

import numpy as np
import pytest

from tests import _indep

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "gll_closed_forms.json")))


def _ev(s):
    return eval(s, {"sqrt": math.sqrt})


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5])
def test_gll_closed_forms(oracle, N):
    xi, w = oracle.gll(N)
    np.testing.assert_allclose(xi, [_ev(s) for s in GOLD["nodes"][str(N)]], rtol=0, atol=2e-16)
    np.testing.assert_allclose(w, [_ev(s) for s in GOLD["weights"][str(N)]], rtol=0, atol=4e-16)


@pytest.mark.parametrize("N", range(1, 16))
def test_gll_sum_symmetry_and_numpy_route(oracle, N):
    xi, w = oracle.gll(N)
    assert abs(w.sum() - 2.0) <= 1e-15 * N
    np.testing.assert_array_equal(xi, -xi[::-1])
    np.testing.assert_array_equal(w, w[::-1])
    assert np.all(np.diff(xi) > 0)
    xr, wr = _indep.gll_numpy(N)
    np.testing.assert_allclose(xi, xr, rtol=0, atol=1e-14)
    np.testing.assert_allclose(w, wr, rtol=0, atol=1e-14)


@pytest.mark.parametrize("N", range(1, 16))
def test_gll_quadrature_exact_to_degree_2N_minus_1(oracle, N):
    xi, w = oracle.gll(N)
    for p in range(0, 2 * N):
        exact = 0.0 if p % 2 else 2.0 / (p + 1)
        assert abs(w @ xi ** p - exact) <= 1e-14, (N, p)
    # and NOT exact at degree 2N (Lobatto rule has degree 2N-1)
    p = 2 * N
    assert abs(w @ xi ** p - 2.0 / (p + 1)) > 1e-11


@pytest.mark.parametrize("N", range(1, 16))
def test_D_exact_on_polynomials(oracle, N):
    xi, _ = oracle.gll(N)
    D = oracle.deriv(N, xi)
    assert np.max(np.abs(D @ np.ones(N + 1))) <= 1e-14 * N * N   # D 1 = 0 (negative-sum diagonal)
    for p in range(1, N + 1):
        err = np.max(np.abs(D @ xi ** p - p * xi ** (p - 1)))
        assert err <= 2e-12, (N, p, err)


@pytest.mark.parametrize("N", range(1, 16))
def test_D_matches_vandermonde_route(oracle, N):
    if N > 10:
        pytest.skip("Vandermonde too ill-conditioned above N=10")
    xi, _ = oracle.gll(N)
    D = oracle.deriv(N, xi)
    Dv = _indep.deriv_vandermonde(xi)
    np.testing.assert_allclose(D, Dv, rtol=0, atol=1e-9 * np.abs(Dv).max())


@pytest.mark.parametrize("N", range(1, 16))
def test_summation_by_parts(oracle, N):
    xi, w = oracle.gll(N)
    D = oracle.deriv(N, xi)
    W = np.diag(w)
    S = W @ D + D.T @ W
    B = np.zeros((N + 1, N + 1))
    B[0, 0], B[N, N] = -1.0, 1.0
    assert np.max(np.abs(S - B)) <= 1e-14 * (N + 1) ** 2


@pytest.mark.parametrize("N", [1, 2])
def test_K1_closed_forms(oracle, N):
    xi, w = oracle.gll(N)
    D = oracle.deriv(N, xi)
    K1 = D.T @ np.diag(w) @ D
    ref = np.array([[_ev(s) for s in row] for row in GOLD["K1"][str(N)]])
    np.testing.assert_allclose(K1, ref, rtol=0, atol=1e-15)


def test_D_diagonal_textbook_values(oracle):
    """Endpoint diagonal entries -N(N+1)/4 and +N(N+1)/4, interior 0 (odd/even
    symmetry), which the negative-sum rule must reproduce to rounding."""
    for N in range(1, 12):
        D = oracle.deriv(N)
        assert abs(D[0, 0] + N * (N + 1) / 4) <= 1e-12 * N * N
        assert abs(D[N, N] - N * (N + 1) / 4) <= 1e-12 * N * N
        for i in range(1, N):
            assert abs(D[i, i]) <= 1e-12 * N * N


def test_oracle_rejects_bad_order(oracle):
    with pytest.raises(oracle.OracleError):
        oracle.gll(0)
