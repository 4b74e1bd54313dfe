"""The NCCL transport of the box decomposition (IGA_XPORT_NCCL: one process per GPU):
ghost-U and halo-row exchanges with NCCL send/recv, the halo residual, and the distributed GMRES
(ghost exchange per SpMV, all-reduced Gram-Schmidt dots).  Two processes on two GPUs each compare
their owned rows with the in-process IGA_XPORT_LOCAL group result (itself checked against the
oracle in test_gpu_dist.py), including procs = 2 on a PERIODIC axis, where the two neighbour
offsets of a rank go to the same peer (the send/receive order must pair them up).

Skipped when fewer than two CUDA devices are visible (this build's GPU pool gives one GPU per
call; the LOCAL transport runs the same packing / sub-box / K5 code on one GPU)."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys, json, itertools
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["IGA_ROOT"]); sys.path.insert(0, os.path.join(os.environ["IGA_ROOT"], "tests"))
import paper_1305_4452_b200 as iga, workloads
from parity_util import rowmax_rel_err, vec_rel_err
cid, n, procs = int(sys.argv[1]), int(sys.argv[2]), [int(x) for x in sys.argv[3].split(",")]
rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
w = workloads.make(cid, n=n)
obj = [iga.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
sp = iga.Space.from_workload(w, device=rank, dist={"rank": rank, "nranks": ws, "procs": procs,
                                                   "transport": iga.XPORT_NCCL, "nccl_id": obj[0]})
def owned(sp):
    rows = []
    for g in itertools.product(*[range(sp.owned_lo[a], sp.owned_hi[a]) for a in range(w.dim)]):
        node = 0
        for a in range(w.dim):
            node = node * w.nfun[a] + g[a]
        rows.extend(node * w.dof + i for i in range(w.dof))
    return np.array(rows, np.int64)
R = owned(sp)
ph = iga.make_phys(w.phys, w.params)
rp, ci = sp.csr_pattern()
vals, F = sp.form_jacobian(ph, w.a, w.b, torch.from_numpy(w.U[R]).to(dev), torch.from_numpy(w.Udot[R]).to(dev),
                           want_F=True)
sp.check()
# the same decomposition in-process on this GPU (LOCAL transport), rank `rank`'s rows
loc = [iga.Space.from_workload(w, device=rank, dist={"rank": r, "nranks": ws, "procs": procs,
                                                     "transport": iga.XPORT_LOCAL}) for r in range(ws)]
rows = [owned(s) for s in loc]
lv, lF = iga.form_jacobian_group(loc, ph, w.a, w.b, [torch.from_numpy(w.U[r]).to(dev) for r in rows],
                                 [torch.from_numpy(w.Udot[r]).to(dev) for r in rows], want_F=True)
lrp, lci = loc[rank].csr_pattern()
ok = bool(torch.equal(rp, lrp) and torch.equal(ci, lci))
err = rowmax_rel_err(lrp.cpu().numpy(), lv[rank].cpu().numpy(), vals.cpu().numpy())
ferr = vec_rel_err(lF[rank].cpu().numpy(), F.cpu().numpy())
# distributed GMRES on the NCCL ranks vs the in-process group
b = -F
x, it, rr = sp.gmres(rp, ci, vals, b, restart=10, maxit=10, rtol=0.0)
lx = iga.gmres_group(loc, [s.csr_pattern()[0] for s in loc], [s.csr_pattern()[1] for s in loc], lv,
                     [-f for f in lF], restart=10, maxit=10)[0]
xerr = float((x - lx[rank]).abs().max() / lx[rank].abs().max().clamp_min(1e-300))
print(json.dumps({"rank": rank, "pattern": ok, "err": err, "ferr": ferr, "xerr": xerr}), flush=True)
dist.destroy_process_group()
'''


@pytest.mark.parametrize("cid,n,procs", [(3, 12, "2,1"), (5, 6, "2,1,1"), (4, 5, "1,2,1"), (7, 10, "1,2")])
def test_nccl_two_ranks_match_local_group(cid, n, procs, tmp_path):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices (NCCL transport)")
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    env = dict(os.environ, IGA_ROOT=ROOT)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(29600 + cid), str(script), str(cid),
                        str(n), procs], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    import json
    outs = [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(outs) == 2
    for o in outs:
        assert o["pattern"], o
        assert o["err"] <= 1e-11 and o["ferr"] <= 1e-11, o
        assert o["xerr"] <= 1e-8, o
