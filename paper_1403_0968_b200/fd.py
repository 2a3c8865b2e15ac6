"""ctypes binding of include/fd.h (argument marshalling only): the
finite-difference wave-equation step of arXiv 1403.0968, lst:fdCode
(SURVEY.md §8(f) NEXT-4).  Every step runs in libsem.so's
sm_100a kernel; there is no CPU fallback."""
from __future__ import annotations

import ctypes

import numpy as np

from . import sem

_fd = None


def lib():
    global _fd
    if _fd is None:
        L = sem.lib()
        P, i64 = ctypes.c_void_p, ctypes.c_int64
        L.fd_weights.argtypes = [ctypes.c_int, ctypes.c_double, P]
        L.fd2d_step.argtypes = [P, P, P, i64, i64, ctypes.c_int, P, ctypes.c_double, P]
        L.fd2d_run.argtypes = [P, P, P, i64, i64, ctypes.c_int, P, ctypes.c_double, ctypes.c_int,
                               P, ctypes.POINTER(ctypes.c_int)]
        L.fd2d_run_ex.argtypes = [P, P, P, i64, i64, ctypes.c_int, P, ctypes.c_double,
                                  ctypes.c_int, ctypes.c_int, P, ctypes.POINTER(ctypes.c_int)]
        for f in (L.fd_weights, L.fd2d_step, L.fd2d_run, L.fd2d_run_ex):
            f.restype = ctypes.c_int
        _fd = L
    return _fd


def _check(rc):
    if rc != sem.SEM_OK:
        msg = sem.lib().sem_last_error(None).decode(errors="replace")
        raise sem.SemError(rc, msg)


def weights(r: int, dx: float) -> np.ndarray:
    """omega_{-r..r} (reading R6: central second-derivative weights of order 2r)."""
    w = np.zeros(2 * r + 1)
    _check(lib().fd_weights(int(r), float(dx), w.ctypes.data_as(ctypes.c_void_p)))
    return w


def _grid(t, name):
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda:
        raise TypeError(f"{name} must be a float64 CUDA tensor")
    if t.dim() != 2 or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous [h, w] tensor")
    return ctypes.c_void_p(t.data_ptr())


def step(u1, u2, u3, omega, dt: float, stream=None):
    """u3 <- -2 u1 + u2 - dt^2 lap(u1) on the periodic [h, w] grid (one launch)."""
    import torch
    h, w = u1.shape
    if u2.shape != u1.shape or u3.shape != u1.shape:
        raise ValueError("u1, u2, u3 must have the same shape")
    om = np.ascontiguousarray(omega, dtype=np.float64)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    _check(lib().fd2d_step(_grid(u1, "u1"), _grid(u2, "u2"), _grid(u3, "u3"), w, h, om.size // 2,
                           om.ctypes.data_as(ctypes.c_void_p), float(dt), ctypes.c_void_p(s)))
    return u3


FD_REGROUPED = 1


def run(u1, u2, u3, omega, dt: float, steps: int, stream=None, regrouped: bool = False):
    """`steps` steps with (u1, u2, u3) <- (u3, u1, u2) after each (reading R6b).
    regrouped=True: fd2d_run_ex with FD_REGROUPED (pair-regrouped FMA form,
    reading R6c; symmetric weights only); default: the listing's order,
    bit-identical to the oracle.  Returns (newest, previous) tensors."""
    import torch
    h, w = u1.shape
    om = np.ascontiguousarray(omega, dtype=np.float64)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    latest = ctypes.c_int(-1)
    _check(lib().fd2d_run_ex(_grid(u1, "u1"), _grid(u2, "u2"), _grid(u3, "u3"), w, h,
                             om.size // 2, om.ctypes.data_as(ctypes.c_void_p), float(dt),
                             int(steps), FD_REGROUPED if regrouped else 0, ctypes.c_void_p(s),
                             ctypes.byref(latest)))
    bufs = (u1, u2, u3)
    return bufs[latest.value], bufs[(latest.value + 1) % 3]
