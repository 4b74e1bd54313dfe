"""GPU parity of the multi-rank path on one GPU: all ranks of a box
decomposition live in this process (IGA_XPORT_LOCAL), their kernels run one after another on one
stream and the ghost-U / halo-row exchanges are device copies -- the same packing, sub-box CSR
layout and K5 adds that the NCCL transport moves between GPUs.  Every rank's owned rows are
compared with the oracle's rows (pattern bit-exact, values within the row-max tolerance).
"""
import itertools

import numpy as np
import pytest

import oracle
import workloads
from parity_util import ROW_TOL, rowmax_rel_err, vec_rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1305_4452_b200 as iga
    return iga


def _owned_rows(w, sp):
    rng = [range(sp.owned_lo[a], sp.owned_hi[a]) for a in range(w.dim)]
    rows = []
    for g in itertools.product(*rng):
        node = 0
        for a in range(w.dim):
            node = node * w.nfun[a] + g[a]
        rows.extend(node * w.dof + i for i in range(w.dof))
    return np.array(rows, dtype=np.int64)


LAYOUTS = [
    (1, 16, [2, 2]), (2, 12, [2, 3]), (3, 12, [2, 1]), (3, 16, [2, 2]), (3, 33, [3, 2]),
    (4, 6, [2, 2, 1]), (4, 5, [1, 2, 2]), (5, 8, [2, 2, 2]), (5, 7, [2, 1, 3]), (6, 8, [2, 2]),
    (7, 12, [2, 2]), (7, 10, [1, 3]),
]


@pytest.mark.parametrize("cid,n,procs", LAYOUTS)
def test_group_parity(cid, n, procs):
    iga = _gpu()
    w = workloads.make(cid, n=n)
    nr = int(np.prod(procs))
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(11 + cid)
    Ud_full = rng.uniform(-0.1, 0.1, w.U.size) if w.phys in (1, 3, 4) else w.Udot
    spaces = [iga.Space.from_workload(w, dist={"rank": r, "nranks": nr, "procs": procs,
                                               "transport": iga.XPORT_LOCAL}) for r in range(nr)]
    rows = [_owned_rows(w, sp) for sp in spaces]
    assert sorted(np.concatenate(rows).tolist()) == list(range(w.ndof))
    Us = [torch.from_numpy(w.U[r]).to(dev) for r in rows]
    Uds = [torch.from_numpy(Ud_full[r]).to(dev) for r in rows]
    ph = iga.make_phys(w.phys, w.params)
    vals, Fs = iga.form_jacobian_group(spaces, ph, w.a, w.b, Us, Uds, want_F=True)
    Frs = iga.form_residual_group(spaces, ph, Us, Uds)
    for sp in spaces:
        sp.check()
    osp = oracle.Space.from_workload(w)
    K, T, Fo = osp.assemble_dense(w.phys, w.params, w.a, w.b, w.U, Ud_full)
    orp, oci, ov = oracle.dense_to_csr(K, T)
    for r, sp in enumerate(spaces):
        rp, ci = sp.csr_pattern()
        rp, ci = rp.cpu().numpy(), ci.cpu().numpy()
        R = rows[r]
        idx = np.concatenate([np.arange(orp[g], orp[g + 1]) for g in R])
        srp = np.zeros(len(R) + 1, np.int64)
        srp[1:] = np.cumsum(orp[R + 1] - orp[R])
        assert np.array_equal(rp, srp), f"rank {r}: row_ptr"
        assert np.array_equal(ci, oci[idx]), f"rank {r}: col_idx"
        assert rowmax_rel_err(srp, ov[idx], vals[r].cpu().numpy()) <= ROW_TOL, f"rank {r}: values"
        assert vec_rel_err(Fo, np.concatenate([Fs[k].cpu().numpy() for k in range(nr)])[np.argsort(np.concatenate(rows))]) <= ROW_TOL
        assert vec_rel_err(Fo, np.concatenate([Frs[k].cpu().numpy() for k in range(nr)])[np.argsort(np.concatenate(rows))]) <= ROW_TOL


@pytest.mark.parametrize("cid,procs", [(3, [2, 2]), (5, [2, 2, 2]), (4, [2, 2, 2])])
def test_group_matches_single_rank_full_size_probe(cid, procs):
    """A larger mesh (the bench's fused kernels at a few tiles per rank): the union of the
    ranks' owned rows equals the single-rank assembly."""
    iga = _gpu()
    n = {3: 96, 4: 16, 5: 16}[cid]
    w = workloads.make(cid, n=n)
    nr = int(np.prod(procs))
    dev = torch.device("cuda", 0)
    sp1 = iga.Space.from_workload(w)
    ph = iga.make_phys(w.phys, w.params)
    v1, F1 = sp1.form_jacobian(ph, w.a, w.b, torch.from_numpy(w.U).to(dev), torch.from_numpy(w.Udot).to(dev),
                               want_F=True)
    rp1, _ = sp1.csr_pattern()
    rp1 = rp1.cpu().numpy()
    v1 = v1.cpu().numpy()
    spaces = [iga.Space.from_workload(w, dist={"rank": r, "nranks": nr, "procs": procs,
                                               "transport": iga.XPORT_LOCAL}) for r in range(nr)]
    rows = [_owned_rows(w, sp) for sp in spaces]
    Us = [torch.from_numpy(w.U[r]).to(dev) for r in rows]
    Uds = [torch.from_numpy(w.Udot[r]).to(dev) for r in rows]
    vals, Fs = iga.form_jacobian_group(spaces, ph, w.a, w.b, Us, Uds, want_F=True)
    for r, sp in enumerate(spaces):
        sp.check()
        R = rows[r]
        idx = np.concatenate([np.arange(rp1[g], rp1[g + 1]) for g in R])
        srp = np.zeros(len(R) + 1, np.int64)
        srp[1:] = np.cumsum(rp1[R + 1] - rp1[R])
        assert rowmax_rel_err(srp, v1[idx], vals[r].cpu().numpy()) <= ROW_TOL
    Fall = np.zeros(w.ndof)
    for r in range(nr):
        Fall[rows[r]] = Fs[r].cpu().numpy()
    assert vec_rel_err(F1.cpu().numpy(), Fall) <= ROW_TOL
