"""Thin Python binding of libsem (include/sem.h) -- argument marshalling only.

Every step of the hot path runs in the CUDA kernels of libsem.so; this module
only turns torch tensors into pointers, owns the device workspace (PyTorch
caching allocator) and raises on a non-zero status.  There is no CPU fallback:
if libsem.so is missing or no GPU is present, the calls fail loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsem.so")

SEM_OK, SEM_EINVAL, SEM_ECUDA, SEM_ENCCL, SEM_ENOCONV, SEM_ESTATE = range(6)
SEM_NMAX = 15

ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_size_t, ctypes.c_void_p)


class SemMesh(ctypes.Structure):
    _fields_ = [
        ("nelem", ctypes.c_int32),
        ("xyz", ctypes.c_void_p),
        ("glo", ctypes.c_void_p),
        ("dirichlet", ctypes.c_void_p),
        ("nboundary", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("nranks", ctypes.c_int32),
        ("nccl_id", ctypes.c_void_p),
        ("allgather", ALLGATHER_FN),
        ("allgather_user", ctypes.c_void_p),
        ("device", ctypes.c_int32),
        ("kappa", ctypes.c_void_p),
        ("alpha", ctypes.c_void_p),
    ]


EXPORTS = ["sem_version", "sem_gll", "sem_workspace_bytes", "sem_setup", "sem_sizes",
           "sem_ax", "sem_dssum", "sem_mask", "sem_mass", "sem_cg", "sem_launch_count",
           "sem_free", "sem_strerror", "sem_last_error", "sem_nccl_id_bytes",
           "sem_nccl_get_unique_id", "sem_loopback_unique_id", "sem_profile", "sem_profile_read", "sem_kernel_replay", "sem_exchange_plan", "sem_status", "sem_cg_phases",
           "sem_pcg", "sem_diag", "sem_cg_sr", "fd_weights", "fd2d_step", "fd2d_run", "fd2d_run_ex"]

# preconditioners of sem_pcg (include/sem.h enum sem_precond)
PRECOND = {"none": 0, "jacobi": 1}

_lib = None


class SemError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def lib():
    """Load libsem.so (built by __graft_entry__.build()); fail loudly if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise SemError(SEM_ESTATE, f"{LIB_PATH} missing: run __graft_entry__.build() "
                                   "(the CUDA extension is required; there is no fallback)")
    L = ctypes.CDLL(LIB_PATH)
    P, i64 = ctypes.c_void_p, ctypes.c_int64
    L.sem_version.restype = ctypes.c_char_p
    L.sem_gll.argtypes = [ctypes.c_int, P, P]
    L.sem_workspace_bytes.argtypes = [ctypes.POINTER(SemMesh), ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_size_t)]
    L.sem_setup.argtypes = [ctypes.POINTER(SemMesh), ctypes.c_int, P, ctypes.c_size_t, P,
                            ctypes.POINTER(P)]
    L.sem_sizes.argtypes = [P, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.sem_ax.argtypes = [P, P, P]
    L.sem_dssum.argtypes = [P, P]
    L.sem_mask.argtypes = [P, P]
    L.sem_mass.argtypes = [P, P, P]
    L.sem_cg.argtypes = [P, P, P, ctypes.c_double, ctypes.c_int,
                         ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
    L.sem_pcg.argtypes = [P, ctypes.c_int, P, P, ctypes.c_double, ctypes.c_int,
                          ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
    L.sem_diag.argtypes = [P, P]
    L.sem_cg_sr.argtypes = [P, P, P, ctypes.c_double, ctypes.c_int,
                            ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
    L.sem_status.argtypes = [P]
    L.sem_status.restype = ctypes.c_int
    L.sem_launch_count.argtypes = [P]
    L.sem_launch_count.restype = i64
    L.sem_free.argtypes = [P]
    L.sem_free.restype = None
    L.sem_strerror.argtypes = [ctypes.c_int]
    L.sem_strerror.restype = ctypes.c_char_p
    L.sem_last_error.argtypes = [P]
    L.sem_last_error.restype = ctypes.c_char_p
    L.sem_nccl_id_bytes.restype = ctypes.c_int
    L.sem_profile.argtypes = [P, ctypes.c_int]
    L.sem_profile_read.argtypes = [P, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                   ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double)]
    L.sem_nccl_get_unique_id.argtypes = [P]
    L.sem_loopback_unique_id.argtypes = [P]
    L.sem_kernel_replay.argtypes = [P, ctypes.c_int, ctypes.c_int]
    L.sem_cg_phases.argtypes = [P, ctypes.POINTER(ctypes.c_double)]
    L.sem_exchange_plan.argtypes = [ctypes.POINTER(SemMesh), ctypes.c_int, P, P, i64,
                                    ctypes.POINTER(i64), ctypes.POINTER(i64)]
    for f in ("sem_gll", "sem_workspace_bytes", "sem_setup", "sem_sizes", "sem_ax", "sem_dssum",
              "sem_mask", "sem_mass", "sem_cg", "sem_nccl_get_unique_id", "sem_loopback_unique_id", "sem_profile",
              "sem_profile_read", "sem_kernel_replay", "sem_exchange_plan", "sem_pcg", "sem_diag", "sem_cg_sr",
              "sem_cg_phases"):
        getattr(L, f).restype = ctypes.c_int
    _lib = L
    return L


def _check(rc, ctx=None):
    if rc != SEM_OK:
        msg = lib().sem_last_error(ctx).decode(errors="replace")
        raise SemError(rc, msg or lib().sem_strerror(rc).decode())


def gll(N: int):
    """The library's own GLL nodes/weights; host-only."""
    xi = np.zeros(N + 1)
    w = np.zeros(N + 1)
    _check(lib().sem_gll(int(N), xi.ctypes.data, w.ctypes.data))
    return xi, w


def _dptr(t, n, name):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
        raise TypeError(f"{name} must be a CUDA float64 tensor")
    if not t.is_contiguous() or t.numel() != n:
        raise ValueError(f"{name} must be contiguous with {n} elements, got {tuple(t.shape)}")
    return ctypes.c_void_p(t.data_ptr())


class Context:
    """sem_setup() on one rank.  ``mesh`` is a meshgen.Mesh (or any object with
    xyz [E,3,n^3] f64, glo [E,n^3] i64, dirichlet [E,n^3] u8 and optional
    nboundary).  ``group``: torch.distributed process group for nranks > 1.
    ``kappa`` / ``alpha``: per-local-node screened-Coulomb coefficients
    (host arrays, [E*n^3]; None = Poisson), see include/sem.h.
    ``loopback``: a ``dist.LoopbackRank`` -- this context is one rank of an
    in-process multi-rank world on one GPU (test transport, include/sem.h
    sem_loopback_unique_id); the device work goes on the CALLING thread's
    current torch stream."""

    def __init__(self, mesh, N: int | None = None, device: int | None = None, group=None,
                 kappa=None, alpha=None, loopback=None):
        import torch
        L = lib()
        self.N = int(mesh.N if N is None else N)
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self._xyz = np.ascontiguousarray(mesh.xyz, dtype=np.float64)
        self._glo = np.ascontiguousarray(mesh.glo, dtype=np.int64)
        self._dir = np.ascontiguousarray(mesh.dirichlet, dtype=np.uint8)
        E = int(self._glo.shape[0])
        m = SemMesh()
        m.nelem = E
        m.xyz = self._xyz.ctypes.data
        m.glo = self._glo.ctypes.data
        m.dirichlet = self._dir.ctypes.data
        m.nboundary = int(getattr(mesh, "nboundary", 0) or 0)
        m.device = self.device
        self._kappa = None if kappa is None else np.ascontiguousarray(kappa, dtype=np.float64).reshape(-1)
        self._alpha = None if alpha is None else np.ascontiguousarray(alpha, dtype=np.float64).reshape(-1)
        for name, a in (("kappa", self._kappa), ("alpha", self._alpha)):
            if a is not None and a.size != self._glo.size:
                raise ValueError(f"{name} must hold {self._glo.size} values, got {a.size}")
        m.kappa = None if self._kappa is None else self._kappa.ctypes.data
        m.alpha = None if self._alpha is None else self._alpha.ctypes.data
        self._group = group
        self._keep = []
        if loopback is not None:
            m.rank, m.nranks = int(loopback.rank), int(loopback.nranks)
            self._keep.append(loopback.id)
            m.nccl_id = ctypes.cast(loopback.id, ctypes.c_void_p)
            cb = loopback.allgather_fn()
            self._keep.append(cb)
            m.allgather = cb
        elif group is not None and torch.distributed.get_world_size(group) > 1:
            from . import dist as _dist
            m.rank = torch.distributed.get_rank(group)
            m.nranks = torch.distributed.get_world_size(group)
            nid = _dist.broadcast_nccl_id(group)
            self._keep.append(nid)
            m.nccl_id = ctypes.cast(nid, ctypes.c_void_p)
            cb = _dist.make_allgather(group)
            self._keep.append(cb)
            m.allgather = cb
        else:
            m.rank, m.nranks = 0, 1
            m.allgather = ALLGATHER_FN()
        self._mesh = m
        nbytes = ctypes.c_size_t(0)
        _check(L.sem_workspace_bytes(ctypes.byref(m), self.N, ctypes.byref(nbytes)))
        with torch.cuda.device(self.device):
            self.workspace = torch.empty(int(nbytes.value), dtype=torch.uint8, device="cuda")
            self.stream = torch.cuda.current_stream()
        ctx = ctypes.c_void_p()
        _check(L.sem_setup(ctypes.byref(m), self.N, ctypes.c_void_p(self.workspace.data_ptr()),
                           nbytes.value, ctypes.c_void_p(self.stream.cuda_stream),
                           ctypes.byref(ctx)))
        self._ctx = ctx
        nl, ng = ctypes.c_int64(0), ctypes.c_int64(0)
        _check(L.sem_sizes(ctx, ctypes.byref(nl), ctypes.byref(ng)), ctx)
        self.nlocal, self.nglobal = int(nl.value), int(ng.value)
        self.nelem = E

    # -- entry points -------------------------------------------------------
    def ax(self, u, w=None):
        import torch
        if w is None:
            w = torch.empty_like(u)
        _check(lib().sem_ax(self._ctx, _dptr(u, self.nlocal, "u"), _dptr(w, self.nlocal, "w")),
               self._ctx)
        return w

    def dssum(self, w):
        _check(lib().sem_dssum(self._ctx, _dptr(w, self.nlocal, "w")), self._ctx)
        return w

    def mask(self, w):
        _check(lib().sem_mask(self._ctx, _dptr(w, self.nlocal, "w")), self._ctx)
        return w

    def mass(self, f, b=None):
        import torch
        if b is None:
            b = torch.empty_like(f)
        _check(lib().sem_mass(self._ctx, _dptr(f, self.nlocal, "f"), _dptr(b, self.nlocal, "b")),
               self._ctx)
        return b

    def cg(self, b, x=None, tol: float = 1e-8, maxit: int = 1000, raise_noconv: bool = False,
           precond: str = "none", variant: str = "standard"):
        """Returns (x, iters, rel_res, converged).  precond="jacobi": sem_pcg
        with the Jacobi preconditioner (NEXT-2).  variant="single_reduction":
        sem_cg_sr, the Chronopoulos-Gear recurrence (NEXT-3)."""
        import torch
        if x is None:
            x = torch.zeros_like(b)
        it = ctypes.c_int(0)
        rr = ctypes.c_double(0.0)
        if variant == "single_reduction":
            if precond != "none":
                raise ValueError("the single-reduction variant has no preconditioner")
            rc = lib().sem_cg_sr(self._ctx, _dptr(b, self.nlocal, "b"), _dptr(x, self.nlocal, "x"),
                                 float(tol), int(maxit), ctypes.byref(it), ctypes.byref(rr))
        elif variant != "standard":
            raise ValueError(f"unknown CG variant {variant!r}")
        elif precond == "none":
            rc = lib().sem_cg(self._ctx, _dptr(b, self.nlocal, "b"), _dptr(x, self.nlocal, "x"),
                              float(tol), int(maxit), ctypes.byref(it), ctypes.byref(rr))
        else:
            rc = lib().sem_pcg(self._ctx, PRECOND[precond], _dptr(b, self.nlocal, "b"),
                               _dptr(x, self.nlocal, "x"), float(tol), int(maxit),
                               ctypes.byref(it), ctypes.byref(rr))
        if rc == SEM_ENOCONV and not raise_noconv:
            return x, it.value, rr.value, False
        _check(rc, self._ctx)
        return x, it.value, rr.value, True

    def diag(self, d=None):
        """d = Q Q^T diag(A_L): assembled operator diagonal in local storage."""
        import torch
        if d is None:
            d = torch.empty(self.nlocal, dtype=torch.float64, device=f"cuda:{self.device}")
        _check(lib().sem_diag(self._ctx, _dptr(d, self.nlocal, "d")), self._ctx)
        return d

    def rhs(self, f):
        """b = mask Q Q^T (B_L f): assembled, masked right-hand side."""
        b = self.mass(f)
        self.dssum(b)
        self.mask(b)
        return b

    PROF_CLASSES = ("ax", "k1", "k2", "dssum", "other", "rcg")

    def profile(self, enable: bool = True):
        _check(lib().sem_profile(self._ctx, 1 if enable else 0), self._ctx)

    def profile_read(self):
        """{class: (device ms, launches, algorithmic bytes)} since profile(True)."""
        out = {}
        for i, nm in enumerate(self.PROF_CLASSES):
            ms, n, by = ctypes.c_double(0), ctypes.c_int64(0), ctypes.c_double(0)
            _check(lib().sem_profile_read(self._ctx, i, ctypes.byref(ms), ctypes.byref(n),
                                          ctypes.byref(by)), self._ctx)
            out[nm] = (ms.value, n.value, by.value)
        return out

    CG_PHASES = ("update_operator", "barrier_pap", "dssum_r_update", "barrier_rr")

    def cg_phases(self):
        """{phase: us per iteration} of CTA 0 in the last sem_cg, which must
        have run as the resident kernel (include/sem.h sem_cg_phases)."""
        us = (ctypes.c_double * 4)()
        _check(lib().sem_cg_phases(self._ctx, us), self._ctx)
        return dict(zip(self.CG_PHASES, list(us)))

    KERNELS = {"ax": 0, "k1": 1, "k2": 2, "ax+dssum": 3}

    def kernel_replay(self, which: str, reps: int):
        """Enqueue `reps` back-to-back launches of one CG kernel as one graph on
        the context stream (benchmark helper; internal CG state left undefined)."""
        _check(lib().sem_kernel_replay(self._ctx, self.KERNELS[which], int(reps)), self._ctx)

    def status(self):
        """Raise the context's sticky error (sem_status), if any."""
        _check(lib().sem_status(self._ctx), self._ctx)

    @property
    def launch_count(self) -> int:
        return int(lib().sem_launch_count(self._ctx))

    def free(self):
        if getattr(self, "_ctx", None):
            lib().sem_free(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
