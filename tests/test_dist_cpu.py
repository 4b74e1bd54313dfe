"""Multi-rank host logic, no GPU: the box decomposition and exchange plan that
libiga computes (iga_dist_plan, host-only C++), checked for every rank of several layouts, and
exchanged between real processes over torch.distributed gloo (world_size 2 and 4): every
message's rows, as global row ids, must arrive where the receiver expects them.
"""
import itertools
import os
import socket

import numpy as np
import pytest

import workloads

iga = pytest.importorskip("paper_1305_4452_b200")

LAYOUTS = [
    (1, 16, [2, 1]), (1, 16, [2, 2]), (2, 12, [3, 2]), (3, 12, [2, 2]), (3, 12, [4, 1]),
    (4, 6, [2, 2, 1]), (4, 6, [2, 2, 2]), (5, 8, [2, 2, 2]), (5, 9, [1, 3, 2]), (7, 12, [2, 2]),
]


def _plans(w, procs):
    n = int(np.prod(procs))
    return [iga.dist_plan(w, {"rank": r, "nranks": n, "procs": procs}) for r in range(n)]


def _box_rows(w, p, msg, send):
    """global row ids of a message box, in message order (node-major, dof innermost)"""
    lo = msg["box_lo"]
    rng = [range(msg["box_n"][a]) for a in range(w.dim)]
    rows = []
    for b in itertools.product(*rng):
        node = 0
        for a in range(w.dim):
            g = (p["own_lo"][a] + lo[a] + b[a]) % w.nfun[a]
            node = node * w.nfun[a] + g
        rows.extend(node * w.dof + i for i in range(w.dof))
    return np.array(rows, dtype=np.int64)


def _touched(w, p):
    """nodes touched by the rank's elements (support of every element in its element box)"""
    sets = []
    for a in range(w.dim):
        deg = w.degree[a]
        s = set()
        for e in range(p["el_lo"][a], p["el_hi"][a]):
            for k in range(deg + 1):
                s.add((e + k) % w.nfun[a])          # uniform knots: element e touches functions e..e+p
        sets.append(s)
    return sets


@pytest.mark.parametrize("cid,n,procs", LAYOUTS)
def test_plan_consistent(cid, n, procs):
    w = workloads.make(cid, n=n)
    plans = _plans(w, procs)
    # owned boxes tile the function grid exactly once; element boxes tile the element grid
    own = np.zeros(w.nfun[:w.dim], dtype=np.int32)
    nel = [len(w.knots[a]) - 2 * w.degree[a] - 1 for a in range(w.dim)]
    els = np.zeros(nel, dtype=np.int32)
    for p in plans:
        own[tuple(slice(p["own_lo"][a], p["own_hi"][a]) for a in range(w.dim))] += 1
        els[tuple(slice(p["el_lo"][a], p["el_hi"][a]) for a in range(w.dim))] += 1
    assert (own == 1).all()
    assert (els == 1).all()
    for r, p in enumerate(plans):
        # touched box = owned + halo above it, and it covers every function the rank's elements touch
        for a, s in enumerate(_touched(w, p)):
            ext = {(p["own_lo"][a] + l) % w.nfun[a] for l in range(p["ext_n"][a])}
            assert s == ext, (r, a)
        # each send has the mirror receive on its peer: same sub-box, same rows, same values,
        # same global row ids (sender's halo box == receiver's owned box)
        for m in p["send"]:
            q = plans[m["peer"]]
            match = [x for x in q["recv"] if x["peer"] == r and x["subbox"] == m["subbox"]]
            assert len(match) == 1, (r, m)
            x = match[0]
            assert (x["rows"], x["values"]) == (m["rows"], m["values"])
            np.testing.assert_array_equal(_box_rows(w, p, m, True), _box_rows(w, q, x, False))
        assert len(p["recv"]) == sum(1 for q2, pp in enumerate(plans) for m in pp["send"] if m["peer"] == r)


def test_plan_rejects_too_fine():
    w = workloads.make(1, n=4)                 # 4 elements, p = 2: 4 ranks on an axis leaves 1 element each
    with pytest.raises(iga.IgaError):
        iga.dist_plan(w, {"rank": 0, "nranks": 4, "procs": [4, 1]})
    with pytest.raises(iga.IgaError):
        iga.dist_plan(w, {"rank": 0, "nranks": 3, "procs": [2, 2]})


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
        p = iga.dist_plan(w, {"rank": rank, "nranks": world, "procs": procs})
        # the ghost/halo transport pattern of dist.cu, with row ids as payload: up messages go to
        # the owner, which checks them against its receive box
        reqs, bufs = [], []
        for m in p["send"]:
            t = torch.from_numpy(_box_rows(w, p, m, True))
            reqs.append(dist.isend(t, dst=m["peer"]))
        for m in p["recv"]:
            t = torch.empty(m["rows"], dtype=torch.int64)
            reqs.append(dist.irecv(t, src=m["peer"]))
            bufs.append((m, t))
        for rq in reqs:
            rq.wait()
        ok = all(np.array_equal(t.numpy(), _box_rows(w, p, m, False)) for m, t in bufs)
        # owned rows of all ranks add up to the whole space
        cnt = torch.tensor([int(np.prod([p["own_hi"][a] - p["own_lo"][a] for a in range(w.dim)])) * w.dof])
        dist.all_reduce(cnt)
        ok = ok and int(cnt.item()) == w.ndof
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, ok, len(bufs)))
    except Exception as e:          # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e)))


@pytest.mark.parametrize("cid,n,procs", [(3, 12, [2, 1]), (5, 8, [2, 2, 1]), (4, 6, [1, 2, 2])])
def test_gloo_exchange(cid, n, procs):
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
