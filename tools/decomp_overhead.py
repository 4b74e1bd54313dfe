"""Cost of the box decomposition itself, measured in-process on ONE GPU (IGA_XPORT_LOCAL: the
ranks run one after another, exchanges are device copies): single-rank Jacobian time vs the sum
of the per-rank work of an N-rank decomposition of the same mesh (halo-slab sub-box launches,
ghost / halo packing, K5 adds).  Not a scaling measurement -- no rank waits on another.
usage: python tools/decomp_overhead.py CONFIG PROCS...   e.g. 5 2 2 2"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_4452_b200 as iga  # noqa: E402
import workloads  # noqa: E402

cid, procs = int(sys.argv[1]), [int(x) for x in sys.argv[2:]]
w = workloads.make(cid)
dev = torch.device("cuda", 0)
ph = iga.make_phys(w.phys, w.params)


def timeit(fn, n=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.mean(ts)


sp = iga.Space.from_workload(w)
U, Ud = torch.from_numpy(w.U).to(dev), torch.from_numpy(w.Udot).to(dev)
vals = torch.empty(sp.nnz, dtype=torch.float64, device=dev)
F = torch.empty(sp.nrows, dtype=torch.float64, device=dev)
t1 = timeit(lambda: sp.form_jacobian(ph, w.a, w.b, U, Ud, vals=vals, F=F))
del vals, F, sp
torch.cuda.empty_cache()
nr = int(np.prod(procs))
spaces = [iga.Space.from_workload(w, dist={"rank": r, "nranks": nr, "procs": procs, "transport": iga.XPORT_LOCAL})
          for r in range(nr)]
rows = []
for s_ in spaces:
    idx = np.zeros(1, dtype=np.int64)
    for a in range(w.dim):
        g = np.arange(s_.owned_lo[a], s_.owned_hi[a], dtype=np.int64)
        idx = (idx[:, None] * w.nfun[a] + g[None, :]).reshape(-1)
    rows.append((idx[:, None] * w.dof + np.arange(w.dof)[None, :]).reshape(-1))
Us = [torch.from_numpy(w.U[r]).to(dev) for r in rows]
Uds = [torch.from_numpy(w.Udot[r]).to(dev) for r in rows]
vs = [torch.empty(s_.nnz, dtype=torch.float64, device=dev) for s_ in spaces]
Fs = [torch.empty(s_.nrows, dtype=torch.float64, device=dev) for s_ in spaces]
tN = timeit(lambda: iga.form_jacobian_group(spaces, ph, w.a, w.b, Us, Uds, vals=vs, Fs=Fs))
print(json.dumps({"workload": w.name, "procs": procs, "single_rank_ms": t1, "all_ranks_in_process_ms": tN,
                  "overhead": tN / t1 - 1.0}))
