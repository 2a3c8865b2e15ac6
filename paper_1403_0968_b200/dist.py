"""torch.distributed plumbing for multi-rank libsem contexts (marshalling only).

* the NCCL unique id is created by rank 0 (``sem_nccl_get_unique_id``) and
  broadcast to the other ranks;
* the setup-time host all-gather the library calls back into
  (``sem_allgather_fn``) is implemented with torch.distributed -- CPU tensors on a
  gloo group, CUDA tensors on an NCCL group.
The per-iteration data path (interface exchange, dot products) runs on the
library's own NCCL communicator, not through here.

``LoopbackGroup`` is the test harness for that data path on ONE GPU (NCCL
refuses two ranks on one device): P ranks as P host threads of this process,
each with its own torch stream and libsem context, joined by the library's
in-process loopback transport (include/sem.h sem_loopback_unique_id).  The
setup-time all-gather is a threading rendezvous.
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


class LoopbackRank:
    """Rank ``rank`` of a ``LoopbackGroup`` (pass as ``sem.Context(loopback=...)``)."""

    def __init__(self, group, rank):
        self.group, self.rank, self.nranks, self.id = group, rank, group.nranks, group.id

    def allgather_fn(self):
        return self.group._allgather_fn(self.rank)

    def barrier(self):
        """Host rendezvous of all ranks of the group (e.g. after a warm-up,
        before the first device-side collective of the peer-memory
        transport)."""
        self.group._barrier.wait()


class LoopbackGroup:
    """P in-process ranks on one device (test transport).  ``run(fn)`` calls
    ``fn(rank: LoopbackRank)`` on P threads at once, each inside its own
    ``torch.cuda.stream``, and returns the P results in rank order (the first
    exception is re-raised after every thread has ended)."""

    def __init__(self, nranks: int, device: int = 0):
        import threading

        from . import sem
        self.nranks = int(nranks)
        self.device = int(device)
        nb = sem.lib().sem_nccl_id_bytes()
        self.id = (ctypes.c_uint8 * nb)()
        rc = sem.lib().sem_loopback_unique_id(ctypes.cast(self.id, ctypes.c_void_p))
        if rc != 0:
            raise sem.SemError(rc, "sem_loopback_unique_id failed")
        self._barrier = threading.Barrier(self.nranks, timeout=300)
        self._slots = [None] * self.nranks

    def _allgather_fn(self, rank):
        from .sem import ALLGATHER_FN

        def _cb(user, send, nbytes, recv):
            try:
                self._slots[rank] = ctypes.string_at(send, nbytes)
                self._barrier.wait()
                blob = b"".join(self._slots)
                ctypes.memmove(recv, blob, len(blob))
                self._barrier.wait()
                return 0
            except Exception:  # never raise across the C ABI
                self._barrier.abort()
                return 1

        return ALLGATHER_FN(_cb)

    def rank(self, r: int) -> LoopbackRank:
        return LoopbackRank(self, r)

    def run(self, fn):
        import threading

        import torch
        out = [None] * self.nranks
        errs = [None] * self.nranks

        def _body(r):
            try:
                torch.cuda.set_device(self.device)
                with torch.cuda.stream(torch.cuda.Stream(self.device)):
                    out[r] = fn(self.rank(r))
                    torch.cuda.current_stream().synchronize()
            except BaseException as e:  # noqa: BLE001 -- re-raised below
                errs[r] = e
                self._barrier.abort()

        th = [threading.Thread(target=_body, args=(r,), daemon=True) for r in range(self.nranks)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        # the root cause first: peers of a failed rank see a broken barrier
        first = [e for e in errs if e is not None and not isinstance(e, threading.BrokenBarrierError)]
        first += [e for e in errs if e is not None]
        if first:
            raise first[0]
        return out
