"""Host logic of the distributed GMRES (SURVEY §8(e) x §8(f) rank 2), no GPU: the ghost-exchange
plan libiga computes (iga_krylov_plan, host-only C++) is checked for every rank of several layouts
-- mirrored send/receive pairs, ghost layers covering every column an owned row references (the
Alg. 3 pattern of the oracle) -- and exchanged between real processes over torch.distributed gloo
(world_size 2 and 4) in the plan's order: every ghost cell must receive the global row id it stands
for, also when one peer sits on both sides of a two-rank periodic axis."""
import itertools
import os
import socket

import numpy as np
import pytest

import oracle
import workloads

iga = pytest.importorskip("paper_1305_4452_b200")

LAYOUTS = [(3, 12, [2, 2]), (3, 12, [2, 1]), (3, 12, [3, 2]), (1, 16, [2, 2]), (2, 12, [2, 2]),
           (7, 12, [2, 2]), (4, 6, [2, 1, 2]), (5, 8, [2, 2, 2]), (6, 8, [1, 2])]


def _plans(w, procs):
    nr = int(np.prod(procs))
    return [iga.krylov_plan(w, {"rank": r, "nranks": nr, "procs": procs}) for r in range(nr)]


def _ext_global(w, p, cell):
    """global node of an extended-box cell (None outside an open axis)"""
    node = 0
    for a in range(w.dim):
        g = p["own_lo"][a] - p["ghost"][a] + cell[a]
        if w.periodic[a]:
            g %= w.nfun[a]
        elif g < 0 or g >= w.nfun[a]:
            return None
        node = node * w.nfun[a] + g
    return node


def _box_ids(w, p, m):
    rows = []
    for b in itertools.product(*[range(m["box_n"][a]) for a in range(w.dim)]):
        cell = [m["box_lo"][a] + b[a] for a in range(w.dim)]
        node = _ext_global(w, p, cell)
        rows.extend(node * w.dof + i for i in range(w.dof))
    return np.array(rows, dtype=np.int64)


@pytest.mark.parametrize("cid,n,procs", LAYOUTS)
def test_krylov_plan_consistent(cid, n, procs):
    w = workloads.make(cid, n=n)
    plans = _plans(w, procs)
    osp = oracle.Space.from_workload(w)
    for r, p in enumerate(plans):
        # mirrored pairs: my send with offset o to q = q's receive with offset -o from me, same cells
        for m in p["send"]:
            q = plans[m["peer"]]
            mo = [-x for x in m["offset"]]
            match = [x for x in q["recv"] if x["peer"] == r and x["offset"] == mo]
            assert len(match) == 1, (r, m)
            assert match[0]["rows"] == m["rows"]
            np.testing.assert_array_equal(_box_ids(w, p, m), _box_ids(w, q, match[0]))
        # the ghost layers hold every node an owned row references (Alg. 3 pattern)
        ghost = set()
        for m in p["recv"]:
            ghost.update((_box_ids(w, p, m) // w.dof).tolist())
        owned = set()
        for g in itertools.product(*[range(p["own_lo"][a], p["own_hi"][a]) for a in range(w.dim)]):
            node = 0
            for a in range(w.dim):
                node = node * w.nfun[a] + g[a]
            owned.add(node)
        rows = np.array(sorted(o * w.dof for o in owned), dtype=np.int64)
        rp, cols = osp.pattern_rows(rows)
        referenced = set((np.asarray(cols) // w.dof).tolist())
        assert referenced <= owned | ghost, (r, sorted(referenced - owned - ghost)[:5])
        assert not (ghost & owned)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cid, n, procs, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        w = workloads.make(cid, n=n)
        p = iga.krylov_plan(w, {"rank": rank, "nranks": world, "procs": procs})
        reqs, bufs = [], []
        for m in p["send"]:                       # the plan's order: sends ascending offset
            reqs.append(dist.isend(torch.from_numpy(_box_ids(w, p, m)), dst=m["peer"]))
        for m in p["recv"]:                       # receives descending offset (pairs repeated peers)
            t = torch.empty(m["rows"], dtype=torch.int64)
            reqs.append(dist.irecv(t, src=m["peer"]))
            bufs.append((m, t))
        for rq in reqs:
            rq.wait()
        ok = all(np.array_equal(t.numpy(), _box_ids(w, p, m)) for m, t in bufs)
        # the global dot product of the all-reduce: owned rows add up to the whole space
        cnt = torch.tensor([int(np.prod([p["own_hi"][a] - p["own_lo"][a] for a in range(w.dim)])) * w.dof])
        dist.all_reduce(cnt)
        ok = ok and int(cnt.item()) == w.ndof
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, len(bufs)))
    except Exception as e:          # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("cid,n,procs", [(3, 12, [2, 1]), (3, 12, [2, 2]), (5, 8, [1, 2, 2])])
def test_gloo_ghost_exchange(cid, n, procs):
    import torch.multiprocessing as mp
    world = int(np.prod(procs))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cid, n, procs, q)) for r in range(world)]
    for pr in ps:
        pr.start()
    res = [q.get(timeout=180) for _ in ps]
    for pr in ps:
        pr.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
    assert sum(k for _, _, k in res if isinstance(k, int)) > 0
