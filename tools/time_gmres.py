"""Time iga_gmres (GMRES(30) + block-Jacobi ILU(0), 30 iterations = the paper's per-Newton-step
budget) on a config's libiga Jacobian, and the SpMV alone (k_spmv via maxit=0 is not
separable, so the solve is timed whole and per iteration)."""
import argparse
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1305_4452_b200 as iga   # noqa: E402
import workloads   # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--maxit", type=int, default=30)
ap.add_argument("--block", type=int, default=32)
ap.add_argument("--precond", type=int, default=2)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
w = workloads.make(a.config)
sp = iga.Space.from_workload(w)
dev = torch.device("cuda", 0)
rp, ci = sp.csr_pattern()
ph = iga.make_phys(w.phys, w.params)
vals, F = sp.form_jacobian(ph, w.a, w.b, torch.from_numpy(w.U).to(dev), torch.from_numpy(w.Udot).to(dev), want_F=True)
sp.check()
b = -F
n, nnz = b.numel(), vals.numel()
res = {}
for maxit in (0, 1, a.maxit):
    ts = []
    for r in range(a.reps + 1):
        x = torch.zeros_like(b)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, it, rr = sp.gmres(rp, ci, vals, b, x=x, restart=30, maxit=maxit, rtol=0.0, precond=a.precond,
                             block_rows=a.block)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    res[maxit] = (float(np.median(ts)), it, rr, sp.last_launch_count())
t0, t1, tk = res[0][0], res[1][0], res[a.maxit][0]
per_it = (tk - t1) / max(1, a.maxit - 1)
# algorithmic bytes of one iteration j (average over j = 0..m-1), one Gram-Schmidt pass:
# SpMV nnz*12 + (n+1)*8 (row_ptr) + n*8 (x) + n*8 (y); multi-dot (j+2) n*8; multi-axpy (j+3) n*8;
# preconditioner vectors r, z, diag 3n*8 (its in-block L/U slots are not counted)
m = a.maxit
avg_j = (m - 1) / 2
bytes_it = nnz * 12 + 3 * n * 8 + ((avg_j + 2) + (avg_j + 3)) * n * 8 + 3 * n * 8
out = {"config": a.config, "n": n, "nnz": nnz, "block_rows": a.block, "precond": a.precond,
       "ms_setup_and_residual(maxit=0)": t0, "ms_maxit1": t1, f"ms_maxit{m}": tk, "ms_per_iteration": per_it,
       "relres": res[m][2], "relres_1": res[1][2], "launches": res[m][3],
       "alg_bytes_per_iteration": bytes_it, "GBps_per_iteration": bytes_it / (per_it * 1e-3) / 1e9}
print(json.dumps(out))
