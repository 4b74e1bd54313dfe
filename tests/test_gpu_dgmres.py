"""GPU parity of the distributed GMRES (iga_gmres_group: in-process ranks of a box decomposition
on one GPU, the same ghost-layer exchange, dot all-reduce and per-rank block-Jacobi ILU(0) that the
NCCL transport runs across GPUs) against the solver oracle on the permuted global system: the
ranks' owned rows concatenated in local order, block-Jacobi blocks = 32-row runs inside each
rank's segment (the paper's one block per process, cut as on one rank).  Matrix and right-hand
side are the oracle's; tolerance as tests/test_gpu_krylov.py (1e-8 after 30 iterations)."""
import itertools

import numpy as np
import pytest

import oracle
import workloads
from oracle import krylov

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


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.device("cuda", 0))


@pytest.mark.parametrize("cid,n,procs,precond", [(3, 12, [2, 2], 2), (3, 16, [2, 1], 2), (3, 12, [3, 2], 2),
                                                 (2, 12, [2, 2], 2), (6, 8, [2, 2], 2), (7, 12, [2, 2], 2),
                                                 (5, 6, [2, 1, 1], 1), (4, 5, [1, 2, 1], 1)])
def test_group_gmres_matches_oracle(cid, n, procs, precond):
    iga = _gpu()
    w = workloads.make(cid, n=n)
    nr = int(np.prod(procs))
    rng = np.random.default_rng(300 + cid)
    Ud = rng.uniform(-0.1, 0.1, w.U.size) if w.phys in (1, 3, 4) else w.Udot
    osp = oracle.Space.from_workload(w)
    K, T, F = osp.assemble_dense(w.phys, w.params, w.a, w.b, w.U, Ud)
    if cid == 4:                                   # Neo-Hooke: rigid modes, shift to a definite system
        K = K + np.eye(K.shape[0]) * np.abs(K).max()
    orp, oci, ov = oracle.dense_to_csr(K, T)
    spaces = [iga.Space.from_workload(w, dist={"rank": r, "nranks": nr, "procs": procs,
                                               "transport": iga.XPORT_LOCAL}) for r in range(nr)]
    rows = [_owned_rows(w, sp) for sp in spaces]
    rps, cis, vals, bs = [], [], [], []
    for R in rows:
        idx = np.concatenate([np.arange(orp[g], orp[g + 1]) for g in R])
        srp = np.zeros(len(R) + 1, np.int64)
        srp[1:] = np.cumsum(orp[R + 1] - orp[R])
        rps.append(_dev(srp)); cis.append(_dev(np.asarray(oci)[idx].astype(np.int32)))
        vals.append(_dev(np.asarray(ov)[idx])); bs.append(_dev(-np.asarray(F)[R]))
    xs, it, rr = iga.gmres_group(spaces, rps, cis, vals, bs, restart=30, maxit=30, precond=precond)
    # oracle on the permuted system
    P = np.concatenate(rows)
    Kp = K[np.ix_(P, P)]
    Tp = np.asarray(T)[np.ix_(P, P)] if T is not None else None
    prp, pci, pv = oracle.dense_to_csr(Kp, Tp if Tp is not None else (Kp != 0))
    starts, off = [], 0
    for R in rows:
        starts.extend(range(off, off + len(R), 32))
        off += len(R)
    xo, ito, rro = krylov.gmres(np.asarray(prp, np.int64), np.asarray(pci, np.int32), np.asarray(pv), -np.asarray(F)[P],
                                restart=30, maxit=30, rtol=0.0, precond=precond, block_rows=starts)
    assert it == ito == 30
    xg = np.concatenate([x.cpu().numpy() for x in xs])
    assert np.max(np.abs(xg - xo)) <= 1e-8 * np.max(np.abs(xo)), (np.max(np.abs(xg - xo)), np.max(np.abs(xo)))
    assert abs(rr - rro) <= 1e-7 * rro + 1e-13


def test_single_rank_group_equals_gmres():
    iga = _gpu()
    w = workloads.make(3, n=16)
    sp = iga.Space.from_workload(w)
    rp, ci = sp.csr_pattern()
    ph = iga.make_phys(w.phys, w.params)
    vals, F = sp.form_jacobian(ph, w.a, w.b, _dev(w.U), _dev(w.Udot), want_F=True)
    b = -F
    x1, it1, r1 = sp.gmres(rp, ci, vals, b, maxit=30, rtol=0.0)
    xs, it2, r2 = iga.gmres_group([sp], [rp], [ci], [vals], [b], maxit=30)
    assert it1 == it2 == 30
    assert float((x1 - xs[0]).abs().max()) <= 1e-9 * float(x1.abs().max())


@pytest.mark.parametrize("cid,n,procs", [(3, 12, [2, 2]), (6, 8, [2, 1])])
def test_group_alpha_step_matches_oracle(cid, n, procs):
    """One generalized-alpha step (2 Newton x 30 GMRES) of in-process ranks: distributed assembly +
    distributed solve, against the oracle stepper whose linear solve is the oracle GMRES on the
    permuted system with the ranks' block partition."""
    from oracle import stepper
    iga = _gpu()
    w = workloads.make(cid, n=n)
    nr = int(np.prod(procs))
    dt = w.b * 9.0 / 4.0
    osp = oracle.Space.from_workload(w)
    spaces = [iga.Space.from_workload(w, dist={"rank": r, "nranks": nr, "procs": procs,
                                               "transport": iga.XPORT_LOCAL}) for r in range(nr)]
    rows = [_owned_rows(w, sp) for sp in spaces]
    P = np.concatenate(rows)
    starts, off = [], 0
    for R in rows:
        starts.extend(range(off, off + len(R), 32))
        off += len(R)

    def assemble(Ua, Uda, a, b):
        K, T, F = osp.assemble_dense(w.phys, w.params, a, b, Ua, Uda)
        return (K, T), np.asarray(F)

    def solve(J, Rv):
        K, T = J
        prp, pci, pv = oracle.dense_to_csr(K[np.ix_(P, P)], np.asarray(T)[np.ix_(P, P)])
        xp, _, _ = krylov.gmres(np.asarray(prp, np.int64), np.asarray(pci, np.int32), np.asarray(pv), Rv[P],
                                restart=30, maxit=30, rtol=0.0, precond=2, block_rows=starts)
        x = np.zeros_like(Rv)
        x[P] = xp
        return x

    U0 = np.array(w.U, dtype=np.float64)
    Ud0 = np.array(w.Udot, dtype=np.float64)
    Uo, Udo, norms = stepper.alpha_step(assemble, solve, U0, Ud0, 0.5, dt, 2)
    rps, cis, vals, Us, Uds = [], [], [], [], []
    for r, sp in enumerate(spaces):
        rp, ci = sp.csr_pattern()
        rps.append(rp); cis.append(ci)
        vals.append(torch.empty(ci.numel(), dtype=torch.float64, device=rp.device))
        Us.append(_dev(U0[rows[r]])); Uds.append(_dev(Ud0[rows[r]]))
    ph = iga.make_phys(w.phys, w.params)
    st = iga.alpha_step_group(spaces, ph, Us, Uds, rps, cis, vals, 0.5, dt)
    for sp in spaces:
        sp.check()
    np.testing.assert_allclose(st["res_norm"], norms, rtol=1e-8)
    Ug = np.zeros_like(U0)
    Udg = np.zeros_like(Ud0)
    for r in range(nr):
        Ug[rows[r]] = Us[r].cpu().numpy()
        Udg[rows[r]] = Uds[r].cpu().numpy()
    assert np.max(np.abs(Ug - Uo)) <= 1e-8 * np.max(np.abs(Uo))
    assert np.max(np.abs(Udg - Udo)) <= 1e-8 * np.max(np.abs(Udo))
