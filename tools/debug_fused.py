import numpy as np, torch, sys
sys.path.insert(0, '.')
import workloads, paper_1305_4452_b200 as iga
def run(w, split):
    sp = iga.Space.from_workload(w)
    if split: sp.set_option("split", 1)
    dev = torch.device("cuda", 0)
    rp, ci = sp.csr_pattern()
    v, F = sp.form_jacobian(iga.make_phys(w.phys, w.params), w.a, w.b, torch.from_numpy(w.U).to(dev), torch.from_numpy(w.Udot).to(dev), want_F=True)
    torch.cuda.synchronize()
    return rp.cpu().numpy(), ci.cpu().numpy(), v.cpu().numpy(), F.cpu().numpy()
for cid, n in [(2, 3), (2, 4), (2, 9), (1, 5), (3, 6)]:
    w = workloads.make(cid, n=n)
    rp, ci, v0, F0 = run(w, True)
    _, _, v1, F1 = run(w, False)
    bad = np.nonzero(np.abs(v0 - v1) > 1e-10 * np.abs(v0).max())[0]
    nf = w.nfun[1]
    print("cfg", cid, "n", n, "nbad", len(bad), "Ferr", np.abs(F0 - F1).max())
    for k in bad[:12]:
        r = np.searchsorted(rp, k, side='right') - 1
        c = ci[k]
        print("  row", divmod(r, nf), "col", divmod(int(c), nf), v0[k], v1[k])
