"""ctypes wrapper around the plain-C oracle (oracle/sem_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this module.  It shares no
code with the CUDA library (paper_1403_0968_b200/csrc) and never imports it.

Each wrapper names the SURVEY.md §8(c) step (O1..O7) and the PAPER.md passage
it follows; see the C source for the definitions.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sem_oracle.c")
_SRC_FD = os.path.join(_HERE, "fd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# Plain build: -O2, no -ffast-math, no FMA contraction (FP64 rounding order is
# exactly the order written in the C source).
# -fopenmp: the element loop of the operator may use several host threads
# (set_threads; CPU baseline timing only, results bit-identical).
GCC_CMD = ["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-ffp-contract=off",
           "-fno-fast-math", "-fopenmp", _SRC, _SRC_FD, "-o", _LIB, "-lm"]

_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(_SRC_FD)):
        subprocess.check_call(GCC_CMD)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.ora_gll.argtypes = [ctypes.c_int, P, P]
        L.ora_deriv.argtypes = [ctypes.c_int, P, P]
        L.ora_geom.argtypes = [ctypes.c_int, i64, P, P, P]
        L.ora_ax.argtypes = [ctypes.c_int, i64, P, P, P]
        L.ora_dssum.argtypes = [i64, P, P]
        L.ora_multiplicity.argtypes = [i64, P, P]
        L.ora_cg.argtypes = [ctypes.c_int, i64, P, P, P, P, P, ctypes.c_double,
                             ctypes.c_int, P, P]
        L.ora_ax_screened.argtypes = [ctypes.c_int, i64, P, P, P, P, P, P]
        L.ora_cg_screened.argtypes = [ctypes.c_int, i64, P, P, P, P, P, P, P, P,
                                      ctypes.c_double, ctypes.c_int, P, P]
        L.ora_cg_cgs.argtypes = [ctypes.c_int, i64, P, P, P, P, P, ctypes.c_double, ctypes.c_int,
                                 P, P]
        L.ora_fd_weights.argtypes = [ctypes.c_int, ctypes.c_double, P]
        L.ora_fd_step.argtypes = [i64, i64, ctypes.c_int, P, ctypes.c_double, P, P, P]
        L.ora_diag_screened.argtypes = [ctypes.c_int, i64, P, P, P, P, P]
        L.ora_pcg_screened.argtypes = [ctypes.c_int, i64, P, P, P, P, P, P, ctypes.c_int, P, P,
                                       ctypes.c_double, ctypes.c_int, P, P]
        L.ora_set_threads.argtypes = [ctypes.c_int]
        L.ora_set_history.argtypes = [P, ctypes.c_int]
        L.ora_get_threads.argtypes = []
        for f in (L.ora_set_history, L.ora_set_threads, L.ora_get_threads, L.ora_gll, L.ora_deriv, L.ora_geom, L.ora_ax, L.ora_dssum,
                  L.ora_multiplicity, L.ora_cg, L.ora_ax_screened, L.ora_cg_screened,
                  L.ora_diag_screened, L.ora_pcg_screened, L.ora_fd_weights, L.ora_fd_step, L.ora_cg_cgs):
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _opt(a, size):
    """Optional per-node coefficient array -> contiguous float64 (or None)."""
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    assert a.size == size
    return a


def _po(a):
    return None if a is None else _p(a)


class OracleError(RuntimeError):
    pass


def _check(rc, what):
    if rc != 0:
        raise OracleError(f"{what} failed with status {rc}")


def set_threads(n: int) -> None:
    """Host threads of the operator's element loop (1 = the plain sequential
    oracle).  Dot products, DSSUM and the CG recurrence stay sequential, so
    every result is bit-identical for any n."""
    if lib().ora_set_threads(int(n)) != 0:
        raise OracleError(f"ora_set_threads({n})")


class history:
    """Context manager: record the relative residual sqrt(rr_k / rr_0),
    k = 0 .. iters, of the CG solves run inside it (instrumentation only).
    ``h.values`` holds the last solve's history."""

    def __init__(self, cap: int = 100000):
        self.buf = np.full(cap, np.nan)
        self.values = None

    def __enter__(self):
        lib().ora_set_history(self.buf.ctypes.data, self.buf.size)
        return self

    def __exit__(self, *exc):
        lib().ora_set_history(None, 0)
        v = self.buf
        n = int(np.argmax(np.isnan(v))) if np.isnan(v).any() else v.size
        self.values = v[:n].copy()
        return False


def get_threads() -> int:
    return int(lib().ora_get_threads())


def gll(N: int):
    """O1: GLL nodes xi and weights w."""
    xi = np.zeros(N + 1)
    w = np.zeros(N + 1)
    _check(lib().ora_gll(N, _p(xi), _p(w)), "ora_gll")
    return xi, w


def deriv(N: int, xi=None):
    """O2: D_im = phi'_m(xi_i), row-major [i, m]."""
    if xi is None:
        xi, _ = gll(N)
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    D = np.zeros((N + 1, N + 1))
    _check(lib().ora_deriv(N, _p(xi), _p(D)), "ora_deriv")
    return D


def geom(N: int, xyz: np.ndarray):
    """O3: geometric factors G [E,6,n^3] (rr,rs,rt,ss,st,tt; w J folded) and
    pointwise Jacobian J [E,n^3]."""
    n3 = (N + 1) ** 3
    xyz = np.ascontiguousarray(xyz, dtype=np.float64).reshape(-1, 3, n3)
    E = xyz.shape[0]
    G = np.zeros((E, 6, n3))
    J = np.zeros((E, n3))
    _check(lib().ora_geom(N, E, _p(xyz), _p(G), _p(J)), "ora_geom")
    return G, J


def ax(N: int, G: np.ndarray, u: np.ndarray, J=None, kappa=None, alpha=None) -> np.ndarray:
    """O4: local unassembled unmasked w = A_L u (eq:semOperator).
    With kappa / alpha (per local node; NEXT-1, eq:semPDE :580-586) the
    screened-Coulomb operator D^T (kappa G^) D + alpha W J (J needed with alpha)."""
    n3 = (N + 1) ** 3
    G = np.ascontiguousarray(G, dtype=np.float64)
    E = G.size // (6 * n3)
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    assert u.size == E * n3
    w = np.zeros(E * n3)
    if J is None and kappa is None and alpha is None:
        _check(lib().ora_ax(N, E, _p(G), _p(u), _p(w)), "ora_ax")
        return w
    J, kappa, alpha = (_opt(a, E * n3) for a in (J, kappa, alpha))
    _check(lib().ora_ax_screened(N, E, _p(G), _po(J), _po(kappa), _po(alpha), _p(u), _p(w)),
           "ora_ax_screened")
    return w


def dssum(glo: np.ndarray, v: np.ndarray) -> np.ndarray:
    """O5: Q Q^T v, copies summed in ascending local order."""
    glo = np.ascontiguousarray(glo, dtype=np.int64).reshape(-1)
    out = np.array(v, dtype=np.float64).reshape(-1).copy()
    assert out.size == glo.size
    _check(lib().ora_dssum(glo.size, _p(glo), _p(out)), "ora_dssum")
    return out


def multiplicity(glo: np.ndarray) -> np.ndarray:
    glo = np.ascontiguousarray(glo, dtype=np.int64).reshape(-1)
    m = np.zeros(glo.size)
    _check(lib().ora_multiplicity(glo.size, _p(glo), _p(m)), "ora_multiplicity")
    return m


PRECOND = {"none": 0, "jacobi": 1}


def diag(N: int, G: np.ndarray, J=None, kappa=None, alpha=None) -> np.ndarray:
    """NEXT-2: local diagonal d_L = diag(A^e) of the (screened) operator, the
    input of the Jacobi preconditioner (PCG); unassembled."""
    n3 = (N + 1) ** 3
    G = np.ascontiguousarray(G, dtype=np.float64)
    E = G.size // (6 * n3)
    J, kappa, alpha = (_opt(a, E * n3) for a in (J, kappa, alpha))
    d = np.zeros(E * n3)
    _check(lib().ora_diag_screened(N, E, _p(G), _po(J), _po(kappa), _po(alpha), _p(d)),
           "ora_diag_screened")
    return d


def cg(N: int, glo, dirichlet, G, b, x0=None, tol=1e-8, maxit=1000, J=None, kappa=None,
       alpha=None, precond: str = "none"):
    """O7: CG (PCG of PAPER.md:672-673, identity preconditioner).
    Returns (x, iters, rel_res, status) with status 0 = converged, 4 = maxit.
    kappa / alpha (+ J): the screened-Coulomb operator of ax() (NEXT-1).
    precond="jacobi": the Jacobi-preconditioned recurrence (NEXT-2,
    ora_pcg_screened); the stopping rule stays on (r,r)_c."""
    n3 = (N + 1) ** 3
    glo = np.ascontiguousarray(glo, dtype=np.int64).reshape(-1)
    dirichlet = np.ascontiguousarray(dirichlet, dtype=np.uint8).reshape(-1)
    G = np.ascontiguousarray(G, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    E = glo.size // n3
    x = np.zeros(E * n3) if x0 is None else np.array(x0, dtype=np.float64).reshape(-1).copy()
    iters = ctypes.c_int(0)
    rel = ctypes.c_double(0.0)
    pc = PRECOND[precond]
    if J is None and kappa is None and alpha is None and pc == 0:
        rc = lib().ora_cg(N, E, _p(glo), _p(dirichlet), _p(G), _p(b), _p(x), float(tol),
                          int(maxit), ctypes.byref(iters), ctypes.byref(rel))
    else:
        J, kappa, alpha = (_opt(a, E * n3) for a in (J, kappa, alpha))
        rc = lib().ora_pcg_screened(N, E, _p(glo), _p(dirichlet), _p(G), _po(J), _po(kappa),
                                    _po(alpha), pc, _p(b), _p(x), float(tol), int(maxit),
                                    ctypes.byref(iters), ctypes.byref(rel))
    if rc not in (0, 4):
        raise OracleError(f"ora_cg failed with status {rc}")
    return x, iters.value, rel.value, rc


def cg_single_reduction(N: int, glo, dirichlet, G, b, x0=None, tol=1e-8, maxit=1000):
    """NEXT-3: Chronopoulos-Gear single-reduction CG (reading R7), Poisson
    operator, identity preconditioner.  Returns (x, iters, rel_res, status)."""
    n3 = (N + 1) ** 3
    glo = np.ascontiguousarray(glo, dtype=np.int64).reshape(-1)
    dirichlet = np.ascontiguousarray(dirichlet, dtype=np.uint8).reshape(-1)
    G = np.ascontiguousarray(G, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
    E = glo.size // n3
    x = np.zeros(E * n3) if x0 is None else np.array(x0, dtype=np.float64).reshape(-1).copy()
    iters = ctypes.c_int(0)
    rel = ctypes.c_double(0.0)
    rc = lib().ora_cg_cgs(N, E, _p(glo), _p(dirichlet), _p(G), _p(b), _p(x), float(tol), int(maxit),
                          ctypes.byref(iters), ctypes.byref(rel))
    if rc not in (0, 4):
        raise OracleError(f"ora_cg_cgs failed with status {rc}")
    return x, iters.value, rel.value, rc


def mass_rhs(N: int, glo, dirichlet, J, f):
    """b = mask Q Q^T (W J f): lumped mass (diagonal J w_abc)
    applied to nodal f, assembled and masked (reading G7)."""
    n = N + 1
    _, w = gll(N)
    w3 = np.einsum("k,j,i->kji", w, w, w).reshape(-1)
    J = np.asarray(J).reshape(-1, n ** 3)
    bl = (J * w3[None, :]).reshape(-1) * np.asarray(f).reshape(-1)
    b = dssum(glo, bl)
    return b * (1.0 - np.asarray(dirichlet, dtype=np.float64).reshape(-1))


# --- NEXT-4: the finite-difference wave-equation example ---
def fd_weights(r: int, dx: float) -> np.ndarray:
    """omega_{-r..r}: central second-derivative weights of order 2r / dx^2
    (reading R6; the paper gives none)."""
    w = np.zeros(2 * r + 1)
    _check(lib().ora_fd_weights(int(r), float(dx), _p(w)), "ora_fd_weights")
    return w


def fd_step(u1: np.ndarray, u2: np.ndarray, weights: np.ndarray, dt: float) -> np.ndarray:
    """u3 of lst:fdCode on the periodic h x w grid of u1."""
    u1 = np.ascontiguousarray(u1, dtype=np.float64)
    u2 = np.ascontiguousarray(u2, dtype=np.float64)
    weights = np.ascontiguousarray(weights, dtype=np.float64)
    h, w = u1.shape
    assert u2.shape == u1.shape and weights.size % 2 == 1
    r = weights.size // 2
    u3 = np.zeros_like(u1)
    _check(lib().ora_fd_step(w, h, r, _p(weights), float(dt), _p(u1), _p(u2), _p(u3)),
           "ora_fd_step")
    return u3
