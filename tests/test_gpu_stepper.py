"""GPU parity of iga_alpha_step (generalized-alpha, eq. (ga) P:697-739,
with the §5 fixed budget of Newton / GMRES iterations) against the oracle stepper
(oracle/stepper.py) driving the oracle assembly and the oracle GMRES.  Both run the same
rho_inf, dt, Newton count and GMRES(30) + block-Jacobi ILU(0) (32-row blocks, the library default) settings.

Tolerance: each Newton step carries the GMRES parity difference (<= 1e-8 relative, see
test_gpu_krylov.py) into the update; after 2 steps x 2 Newton iterations U and Udot agree within
1e-8 of their max magnitude, the Newton residual norms within 1e-8 relative.
"""
import numpy as np
import pytest

import oracle
import workloads
from oracle import krylov, stepper

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RHO = 0.5     # the workloads' (a, b) = (5/6, 4/9 dt) are rho_inf = 0.5


def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1305_4452_b200 as iga
    return iga


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.device("cuda", 0))


@pytest.mark.parametrize("cid,n,steps,newton", [(3, 12, 2, 2), (3, 20, 1, 3), (6, 6, 2, 2), (8, 5, 1, 2)])
def test_alpha_steps_match_oracle(cid, n, steps, newton):
    iga = _gpu()
    w = workloads.make(cid, n=n)
    dt = w.b * 9.0 / 4.0
    osp = oracle.Space.from_workload(w)

    def assemble(Ua, Uda, a, b):
        K, T, F = osp.assemble_dense(w.phys, w.params, a, b, Ua, Uda)
        return oracle.dense_to_csr(K, T), np.asarray(F)

    def solve(J, R):
        rp, ci, v = J
        x, _, _ = krylov.gmres(np.asarray(rp, np.int64), np.asarray(ci, np.int32), np.asarray(v), R, restart=30,
                               maxit=30, rtol=0.0, precond=2, block_rows=32)
        return x

    U0 = np.array(w.U, dtype=np.float64)
    Ud0 = np.array(w.Udot, dtype=np.float64)
    Uo, Udo = U0.copy(), Ud0.copy()
    onorms = []
    for _ in range(steps):
        Uo, Udo, nr = stepper.alpha_step(assemble, solve, Uo, Udo, RHO, dt, newton)
        onorms.append(nr)

    sp = iga.Space.from_workload(w)
    rp, ci = sp.csr_pattern()
    val = torch.empty(ci.numel(), dtype=torch.float64, device=rp.device)
    ph = iga.make_phys(w.phys, w.params)
    U, Ud = _dev(U0), _dev(Ud0)
    for s in range(steps):
        st = sp.alpha_step(ph, U, Ud, rp, ci, val, RHO, dt, newton_its=newton)
        sp.check()
        np.testing.assert_allclose(st["res_norm"], onorms[s], rtol=1e-8)
        assert all(i == 30 for i in st["gmres_its"])
    Ug, Udg = U.cpu().numpy(), Ud.cpu().numpy()
    assert np.max(np.abs(Ug - Uo)) <= 1e-8 * np.max(np.abs(Uo))
    assert np.max(np.abs(Udg - Udo)) <= 1e-8 * np.max(np.abs(Udo))


def test_full_size_config3_step():
    """Config 3 at full size (1024^2): one step of the paper's protocol (2 Newton x 30 GMRES).
    Eq. (ga)'s last line holds on the result, and Newton reduces the residual."""
    iga = _gpu()
    w = workloads.make(3)
    dt = w.b * 9.0 / 4.0
    sp = iga.Space.from_workload(w)
    rp, ci = sp.csr_pattern()
    val = torch.empty(ci.numel(), dtype=torch.float64, device=rp.device)
    ph = iga.make_phys(w.phys, w.params)
    U0 = _dev(w.U)
    Ud0 = _dev(np.random.default_rng(3).uniform(-1, 1, w.U.size))
    U, Ud = U0.clone(), Ud0.clone()
    st = sp.alpha_step(ph, U, Ud, rp, ci, val, RHO, dt, newton_its=2)
    sp.check()
    am, af, g = stepper.alpha_params(RHO)
    rhs = U0 + dt * ((1 - g) * Ud0 + g * Ud)
    assert float((U - rhs).abs().max()) <= 1e-12 * float(U.abs().max())
    assert st["res_norm"][1] < 0.1 * st["res_norm"][0]
    assert all(i == 30 for i in st["gmres_its"]) and max(st["gmres_relres"]) < 1e-2


def test_alpha_step_rejects_bad_options_and_multirank():
    iga = _gpu()
    w = workloads.make(3, n=6)
    sp = iga.Space.from_workload(w)
    rp, ci = sp.csr_pattern()
    val = torch.empty(ci.numel(), dtype=torch.float64, device=rp.device)
    ph = iga.make_phys(w.phys, w.params)
    U, Ud = _dev(w.U), _dev(w.Udot)
    for kw in ({"rho_inf": 1.5, "dt": 1e-6}, {"rho_inf": 0.5, "dt": 0.0}, {"rho_inf": 0.5, "dt": 1e-6, "newton_its": 9},
               {"rho_inf": 0.5, "dt": 1e-6, "precond": 3}):
        with pytest.raises(iga.IgaError) as ei:
            sp.alpha_step(ph, U, Ud, rp, ci, val, **kw)
        assert ei.value.code == 1
    # a rank of a multi-rank decomposition: the solver is single-rank in this build
    spaces = [iga.Space.from_workload(w, dist={"rank": r, "nranks": 2, "procs": [2, 1],
                                               "transport": iga.XPORT_LOCAL}) for r in range(2)]
    rp2, ci2 = spaces[0].csr_pattern()
    b = torch.zeros(spaces[0].nrows, dtype=torch.float64, device=rp.device)
    v2 = torch.zeros(ci2.numel(), dtype=torch.float64, device=rp.device)
    with pytest.raises(iga.IgaError) as ei:
        spaces[0].gmres(rp2, ci2, v2, b)
    assert ei.value.code == 9
