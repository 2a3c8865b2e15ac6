"""Multi-rank host logic on CPU (gloo, world_size 2 and 4): the interface
exchange plan libsem builds in sem_setup (via the host-only C-ABI call
sem_exchange_plan and the torch.distributed all-gather callback), and the
partition-independent DSSUM it implies: per-rank partial
sums in ascending local order, exchanged along the plan, added in ascending
rank order == the unpartitioned Q Q^T of the oracle, bit-identical on every
rank that holds a shared node.  The GPU data path (pack/NCCL/combine kernels)
uses exactly this plan and this order."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

N = 3
ELEMS = (2, 4, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, parts, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1403_0968_b200 import dist as sdist
        from paper_1403_0968_b200 import meshgen
        xi, _ = oracle.gll(N)
        m = meshgen.box_mesh(N, xi, elems=ELEMS, eps=0.05, parts=parts, rank=rank,
                             boundary_first=True)
        counts, ids, nglobal = sdist.exchange_plan(m, N, dist.group.WORLD)
        # --- emulate the device path with the plan (numpy + gloo) ---
        full = meshgen.box_mesh(N, xi, elems=ELEMS, eps=0.05)
        ex, ey, _ = ELEMS
        key = lambda e: e[:, 0] + ex * (e[:, 1] + ey * e[:, 2])
        v_full = meshgen.random_field(full.nlocal, 17).reshape(full.nelem, -1)
        v = v_full[key(m.eidx)].reshape(-1)
        g = m.glo.reshape(-1)
        local = oracle.dssum(g, v)                   # own copies, ascending local order
        first = {}
        for l in range(g.size):
            first.setdefault(int(g[l]), l)
        # pack per peer in plan order, exchange (padded all_gather)
        import torch
        off = np.concatenate([[0], np.cumsum(counts)])
        send = np.array([local[first[int(i)]] for i in ids]) if ids.size else np.zeros(0)
        mx = torch.tensor([send.size])
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        pad = np.zeros(int(mx.item()))
        pad[: send.size] = send
        allv = [torch.zeros(int(mx.item()), dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allv, torch.from_numpy(pad))
        allc = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allc, torch.from_numpy(counts))
        # what peer p sent to me sits at p's offset for me
        contrib = {}   # gid -> {rank: partial}
        for p in range(world):
            if p == rank:
                continue
            pc = allc[p].numpy()
            poff = np.concatenate([[0], np.cumsum(pc)])
            seg = allv[p].numpy()[poff[rank]:poff[rank + 1]]
            mine = ids[off[p]:off[p + 1]]
            assert seg.size == mine.size
            for gid, val in zip(mine, seg):
                contrib.setdefault(int(gid), {})[p] = val
        out = local.copy()
        for gid, d in contrib.items():
            d[rank] = local[first[gid]]
            tot = None
            for p in sorted(d):
                tot = d[p] if tot is None else tot + d[p]
            out[g == gid] = tot
        ref = oracle.dssum(full.glo, v_full.reshape(-1)).reshape(full.nelem, -1)[key(m.eidx)]
        err = np.abs(out - ref.reshape(-1)).max() / np.abs(ref).max()
        q.put((rank, counts.tolist(), ids.tolist(), nglobal, m.glo.tolist(),
               {int(k): float(out[first[k]]) for k in contrib}, float(err), full.nglobal))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,parts", [(2, (1, 1, 2)), (4, (1, 2, 2))])
def test_exchange_plan_and_partitioned_dssum(world, parts):
    from paper_1403_0968_b200 import _build
    _build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, parts, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    surf = {}
    for r, (_, counts, ids, nglobal, glo, shared_vals, err, nfull) in res.items():
        assert nglobal == nfull                       # distinct ids over all ranks
        assert err <= 1e-14                           # == unpartitioned Q Q^T
        surf[r] = set(np.asarray(glo).reshape(-1).tolist())
    for r in range(world):
        _, counts, ids, _, _, vals, _, _ = res[r]
        off = np.concatenate([[0], np.cumsum(counts)])
        for p in range(world):
            seg = ids[off[p]:off[p + 1]]
            assert seg == sorted(seg)                 # ascending within a peer
            truth = sorted(surf[r] & surf[p]) if p != r else []
            assert seg == truth                       # exactly the shared ids
            # the peer lists the same ids for me, in the same order
            _, pc, pids, _, _, _, _, _ = res[p]
            poff = np.concatenate([[0], np.cumsum(pc)])
            assert pids[poff[r]:poff[r + 1]] == seg
        # bit-identical shared values on every rank holding the node
        for p in range(world):
            for gid, val in vals.items():
                if gid in res[p][5]:
                    assert res[p][5][gid] == val
