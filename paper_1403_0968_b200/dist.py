"""torch.distributed plumbing for multi-rank libsem contexts (marshalling only).

* the NCCL unique id is created by rank 0 (``sem_nccl_get_unique_id``) and
  broadcast to the other ranks;
* the setup-time host all-gather the library calls back into
  (``sem_allgather_fn``) is implemented with torch.distributed -- CPU tensors on a
  gloo group, CUDA tensors on an NCCL group.
The per-iteration data path (interface exchange, dot products) runs on the
library's own NCCL communicator, not through here.
"""
from __future__ import annotations

import ctypes

import numpy as np


def _backend(group):
    import torch.distributed as dist
    return dist.get_backend(group)


def broadcast_nccl_id(group):
    import torch
    import torch.distributed as dist

    from . import sem
    L = sem.lib()
    nb = L.sem_nccl_id_bytes()
    buf = (ctypes.c_uint8 * nb)()
    if dist.get_rank(group) == 0:
        rc = L.sem_nccl_get_unique_id(ctypes.cast(buf, ctypes.c_void_p))
        if rc != 0:
            raise sem.SemError(rc, "ncclGetUniqueId failed")
    t = torch.tensor(np.frombuffer(bytes(buf), dtype=np.uint8).copy())
    if _backend(group) == "nccl":
        t = t.cuda()
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast(t, src=src, group=group)
    out = (ctypes.c_uint8 * nb).from_buffer_copy(t.cpu().numpy().tobytes())
    return out


def make_allgather(group):
    """A ``sem_allgather_fn`` backed by torch.distributed on ``group``."""
    import torch
    import torch.distributed as dist

    from .sem import ALLGATHER_FN
    world = dist.get_world_size(group)
    on_gpu = _backend(group) == "nccl"

    def _cb(user, send, nbytes, recv):
        try:
            src = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(send)).copy()
            t = torch.from_numpy(src)
            out = torch.empty(world * nbytes, dtype=torch.uint8)
            if on_gpu:
                t, out = t.cuda(), out.cuda()
            dist.all_gather_into_tensor(out, t, group=group)
            host = out.cpu().numpy()
            ctypes.memmove(recv, host.ctypes.data, world * nbytes)
            return 0
        except Exception:  # never raise across the C ABI
            return 1

    return ALLGATHER_FN(_cb)


def exchange_plan(mesh, N: int, group):
    """Host-only ``sem_exchange_plan``: (counts per rank, shared ids, nglobal)."""
    import torch.distributed as dist

    from . import sem
    L = sem.lib()
    glo = np.ascontiguousarray(mesh.glo, dtype=np.int64)
    dirichlet = np.ascontiguousarray(mesh.dirichlet, dtype=np.uint8)
    xyz = np.ascontiguousarray(mesh.xyz, dtype=np.float64)
    m = sem.SemMesh()
    m.nelem = glo.shape[0]
    m.xyz = xyz.ctypes.data
    m.glo = glo.ctypes.data
    m.dirichlet = dirichlet.ctypes.data
    m.rank = dist.get_rank(group)
    m.nranks = dist.get_world_size(group)
    cb = make_allgather(group)
    m.allgather = cb
    counts = np.zeros(m.nranks, dtype=np.int64)
    cap = glo.size
    ids = np.zeros(cap, dtype=np.int64)
    nslot = ctypes.c_int64(0)
    ng = ctypes.c_int64(0)
    rc = L.sem_exchange_plan(ctypes.byref(m), int(N), counts.ctypes.data, ids.ctypes.data, cap,
                             ctypes.byref(nslot), ctypes.byref(ng))
    sem._check(rc)
    return counts, ids[: nslot.value].copy(), int(ng.value)
