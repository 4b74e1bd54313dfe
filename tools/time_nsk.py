"""Time the NSK Jacobian + residual (split path) at 256^2 (SURVEY §8(f) rank 4 measurement)."""
import json, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1305_4452_b200 as iga  # noqa: E402
import workloads  # noqa: E402
w = workloads.make(6)
dev = torch.device("cuda", 0)
sp = iga.Space.from_workload(w)
U, Ud = torch.from_numpy(w.U).to(dev), torch.from_numpy(w.Udot).to(dev)
ph = iga.make_phys(w.phys, w.params)
vals = torch.empty(sp.nnz, dtype=torch.float64, device=dev)
F = torch.empty(sp.nrows, dtype=torch.float64, device=dev)
for _ in range(3):
    sp.form_jacobian(ph, w.a, w.b, U, Ud, vals=vals, F=F)
sp.check()
ms = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sp.form_jacobian(ph, w.a, w.b, U, Ud, vals=vals, F=F)
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
sp.profile(True); sp.profile_reset()
sp.form_jacobian(ph, w.a, w.b, U, Ud, vals=vals, F=F)
prof = sp.profile_read()
t = statistics.mean(ms)
print(json.dumps({"workload": w.name, "ms_per_step": t, "qpts_per_s": sp.nqp / (t * 1e-3), "nnz": sp.nnz,
                  "kernels": {k: v[1] / v[0] for k, v in prof.items()}}))
