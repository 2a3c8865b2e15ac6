"""The oracle's operator may run its element loop on several host threads
(bench.py's all-core CPU baseline).  Elements are independent, so the
threaded oracle must return BIT-IDENTICAL results -- for Ax (plain and
screened) and for whole CG / PCG / single-reduction solves, whose dot
products, DSSUM and recurrences stay sequential."""
import os

import numpy as np
import pytest

import oracle
from paper_1403_0968_b200 import meshgen


@pytest.fixture
def threads():
    n = max(2, len(os.sched_getaffinity(0)))
    yield n
    oracle.set_threads(1)


def _mesh(N, elems, eps=0.05):
    xi, _ = oracle.gll(N)
    m = meshgen.box_mesh(N, xi, elems=elems, eps=eps)
    G, J = oracle.geom(N, m.xyz)
    return m, G, J


@pytest.mark.parametrize("N", [3, 7])
def test_threaded_ax_bit_identical(threads, N):
    m, G, J = _mesh(N, (3, 2, 4))
    u = meshgen.random_field(m.nlocal, 3)
    kappa, alpha = meshgen.coefficients(m)
    oracle.set_threads(1)
    w1 = oracle.ax(N, G, u)
    s1 = oracle.ax(N, G, u, J=J, kappa=kappa, alpha=alpha)
    oracle.set_threads(threads)
    assert oracle.get_threads() == threads
    np.testing.assert_array_equal(oracle.ax(N, G, u), w1)
    np.testing.assert_array_equal(oracle.ax(N, G, u, J=J, kappa=kappa, alpha=alpha), s1)


@pytest.mark.parametrize("method", ["cg", "jacobi", "sr"])
def test_threaded_solves_bit_identical(threads, method):
    N = 4
    m, G, J = _mesh(N, (3, 3, 2))
    _, f = meshgen.manufactured(m)
    b = oracle.mass_rhs(N, m.glo, m.dirichlet, J, f)

    def solve():
        if method == "sr":
            return oracle.cg_single_reduction(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=500)
        return oracle.cg(N, m.glo, m.dirichlet, G, b, tol=1e-8, maxit=500,
                         precond="jacobi" if method == "jacobi" else "none")

    oracle.set_threads(1)
    x1, it1, r1, _ = solve()
    oracle.set_threads(threads)
    x2, it2, r2, _ = solve()
    assert it1 == it2 and r1 == r2
    np.testing.assert_array_equal(x1, x2)


def test_set_threads_rejects_zero():
    with pytest.raises(oracle.OracleError):
        oracle.set_threads(0)
