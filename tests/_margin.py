"""Iteration-count parity under a measured drift (reading R3).

Two correct FP64 implementations of the same CG recurrence (GPU: FMA
contraction, blocked dot products; oracle: sequential sums, no FMA) produce
relative-residual histories rel_k = sqrt(rr_k / rr_0) that drift apart by a
relative amount delta_k which grows slowly over a solve.  The oracle stops at
`its` for tolerance tol with the relative margin

    margin = min( min_{j < its} rel_j / tol - 1 ,  1 - rel_its / tol ).

If max_{k <= its} delta_k < margin, the GPU's stopping decision is provably
the oracle's (every earlier GPU residual stays above tol, the one at `its`
falls below).  So: counts must be IDENTICAL when margin > drift, and may
differ by at most one iteration otherwise; and the drift itself must stay
under a stated bound, a guard against an implementation error (which shows
as an O(1) divergence): DRIFT_MAX = 25% on any mesh (rounding amplification
grows with the conditioning: up to 13% measured for the single-reduction
recurrence on small N = 9, 12 boxes, 11% for CG on the 6-sided prism mesh
with its thin kite elements), C3_DRIFT_MAX = 5% on the c3 benchmark mesh
(measured: CG 1.3%, Jacobi PCG 1e-8, single-reduction 1.5%).  The GPU history is measured by fixed-count
solves (tol = 0, maxit = k); the oracle's by oracle.history()."""
import math

import numpy as np

DRIFT_MAX = {"cg": 0.25, "jacobi": 0.25, "sr": 0.25}
C3_DRIFT_MAX = {"cg": 0.05, "jacobi": 0.05, "sr": 0.05}


def margin(hist, its, tol):
    """Relative margin of the oracle's stop at `its` for tolerance `tol`."""
    hist = np.asarray(hist)
    below = hist[its]
    above = hist[:its].min() if its > 0 else math.inf
    return min(above / tol - 1.0, 1.0 - below / tol)


def gpu_history(solve, kmax):
    """rel_k of the GPU solver for k = 0 .. kmax; solve(k) -> (its, rel)."""
    h = [1.0]
    for k in range(1, kmax + 1):
        it, rel = solve(k)
        assert it == k
        h.append(rel)
    return np.asarray(h)


def drift(h_gpu, h_ora, kmax=None):
    n = min(len(h_gpu), len(h_ora)) if kmax is None else kmax + 1
    return float(np.max(np.abs(np.asarray(h_gpu[:n]) / np.asarray(h_ora[:n]) - 1.0)))


def assert_count(its, its_r, marg, dr, info=()):
    """Identical counts when the oracle's margin exceeds the measured drift."""
    if marg > dr:
        assert its == its_r, ("margin", marg, "drift", dr, its, its_r, *info)
    else:
        assert abs(its - its_r) <= 1, ("margin", marg, "drift", dr, its, its_r, *info)


def wide_margin_tols(h_ora, h_gpu, count=3, start_frac=0.25, factor=2.0):
    """Tolerances at which the oracle's stop has a margin >= factor x the
    measured drift up to that iteration: for iteration k the admissible tol
    lies in (rel_k, min_{j<k} rel_j); take the geometric mean where that
    interval is wide enough.  Returns [(tol, k, margin)], spread over the
    solve (from start_frac of it on)."""
    h = np.asarray(h_ora)
    run_min = np.minimum.accumulate(h)
    cands = []
    for k in range(max(1, int(start_frac * (len(h) - 1))), min(len(h), len(h_gpu))):
        lo, hi = h[k], run_min[k - 1]
        t = math.sqrt(lo * hi)
        marg = min(hi / t - 1.0, 1.0 - lo / t)
        if marg > factor * drift(h_gpu, h, k):
            cands.append((t, k, marg))
    if not cands:
        return []
    idx = np.linspace(0, len(cands) - 1, min(count, len(cands))).round().astype(int)
    return [cands[i] for i in sorted(set(idx))]
