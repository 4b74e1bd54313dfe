"""Small end-to-end exercise of every kernel family for compute-sanitizer (memcheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_4452_b200 as iga  # noqa: E402
import workloads  # noqa: E402

dev = torch.device("cuda", 0)
for cid, n in ((1, 5), (2, 6), (3, 9), (4, 3), (5, 5)):
    w = workloads.make(cid, n=n)
    for opt in (None, "split", "general"):
        sp = iga.Space.from_workload(w)
        if opt:
            sp.set_option(opt, 1)
        rp, ci = sp.csr_pattern()
        ph = iga.make_phys(w.phys, w.params)
        U = torch.from_numpy(w.U).to(dev)
        Ud = torch.from_numpy(w.Udot).to(dev)
        vals, F = sp.form_jacobian(ph, w.a, w.b, U, Ud, want_F=True)
        sp.form_residual(ph, U, Ud)
        sp.check()
    sp = iga.Space.from_workload(w)
    sp.basis_eval(3)
    sp.check()
    procs = [2, 2] if w.dim == 2 else [2, 1, 2]
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
    iga.form_jacobian_group(spaces, iga.make_phys(w.phys, w.params), w.a, w.b, Us, Uds, want_F=True)
    iga.form_residual_group(spaces, iga.make_phys(w.phys, w.params), Us, Uds)
    for s_ in spaces:
        s_.check()
    torch.cuda.synchronize()
    print("ok", cid, flush=True)
