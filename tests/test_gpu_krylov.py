"""GPU parity of iga_gmres (the Newton step's GMRES + block-Jacobi ILU(0),
P:866-876) against the solver oracle (oracle/krylov.py).  The matrix and right-hand side are the
ORACLE's Jacobian and -F of the workload (no oracle input comes from the CUDA path); both sides run
the same GMRES(m) / preconditioner settings.

Tolerances: one iteration gives x = y_1 M^{-1} b / ||b||, so it checks the
ILU(0) factor and the triangular solves directly, to 1e-12 relative.  After k iterations the two
Krylov processes differ only by fp64 rounding order (CGS2 vs MGS, atomic dot products), which the
Arnoldi recursion amplifies by at most the conditioning of the small least-squares problems:
x within 1e-8 relative, iteration counts within one, true residuals both below rtol.
"""
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


def _system(cid, n):
    w = workloads.make(cid, n=n)
    rng = np.random.default_rng(200 + cid)
    Ud = rng.uniform(-0.1, 0.1, w.U.size) if w.phys in (1, 3, 4) else w.Udot
    osp = oracle.Space.from_workload(w)
    K, T, F = osp.assemble_dense(w.phys, w.params, w.a, w.b, w.U, Ud)
    rp, ci, v = oracle.dense_to_csr(K, T)
    return w, np.asarray(rp, np.int64), np.asarray(ci, np.int32), np.asarray(v, np.float64), -np.asarray(F)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.device("cuda", 0))


SYSTEMS = [(3, 12), (3, 20), (2, 10), (6, 6), (6, 9)]   # nonsingular Jacobians (no Dirichlet rows in 1, 4)


@pytest.mark.parametrize("precond,B", [(0, 0), (1, 0), (2, 1), (2, 0), (2, 37), (2, 256), (2, 2000)])
@pytest.mark.parametrize("cid,n", SYSTEMS)
def test_one_iteration_applies_preconditioner(cid, n, precond, B):
    iga = _gpu()
    w, rp, ci, v, b = _system(cid, n)
    sp = iga.Space.from_workload(w)
    x, it, rr = sp.gmres(_dev(rp), _dev(ci), _dev(v), _dev(b), restart=1, maxit=1, rtol=0.0, precond=precond,
                         block_rows=B)
    xo, ito, rro = krylov.gmres(rp, ci, v, b, restart=1, maxit=1, rtol=0.0, precond=precond, block_rows=B or 32)
    assert it == ito == 1
    xg = x.cpu().numpy()
    assert np.max(np.abs(xg - xo)) <= 1e-12 * np.max(np.abs(xo))
    assert abs(rr - rro) <= 1e-10 * max(rro, 1e-300)


@pytest.mark.parametrize("restart,maxit,rtol", [(30, 30, 0.0), (30, 30, 1e-6), (5, 23, 0.0), (10, 200, 1e-10)])
@pytest.mark.parametrize("cid,n", SYSTEMS)
def test_gmres_matches_oracle(cid, n, restart, maxit, rtol):
    iga = _gpu()
    w, rp, ci, v, b = _system(cid, n)
    sp = iga.Space.from_workload(w)
    rng = np.random.default_rng(9)
    x0 = rng.uniform(-1e-3, 1e-3, b.size)
    x, it, rr = sp.gmres(_dev(rp), _dev(ci), _dev(v), _dev(b), x=_dev(x0), restart=restart, maxit=maxit, rtol=rtol,
                         precond=2, block_rows=64)
    xo, ito, rro = krylov.gmres(rp, ci, v, b, x0=x0, restart=restart, maxit=maxit, rtol=rtol, precond=2,
                                block_rows=64)
    assert abs(it - ito) <= 1
    if rtol > 0:
        assert rr <= rtol * (1 + 1e-6) and rro <= rtol * (1 + 1e-6)
    else:
        assert it == ito
    xg = x.cpu().numpy()
    if it == ito:
        assert np.max(np.abs(xg - xo)) <= 1e-8 * np.max(np.abs(xo))
    # the reported residual is the true one
    r = b - krylov.csr_matvec(rp, ci, v, xg)
    assert abs(np.linalg.norm(r) / np.linalg.norm(b) - rr) <= 1e-9 * max(rr, 1e-14) + 1e-15


def test_zero_rhs_and_bad_args():
    iga = _gpu()
    w, rp, ci, v, b = _system(3, 8)
    sp = iga.Space.from_workload(w)
    x, it, rr = sp.gmres(_dev(rp), _dev(ci), _dev(v), _dev(np.zeros_like(b)), restart=30, maxit=30, rtol=1e-8)
    assert it == 0 and float(x.abs().max()) == 0.0
    with pytest.raises(iga.IgaError):
        sp.gmres(_dev(rp), _dev(ci), _dev(v), _dev(b), precond=7)
    with pytest.raises(iga.IgaError):
        sp.gmres(_dev(rp), _dev(ci), _dev(v), _dev(b), restart=0)


@pytest.mark.parametrize("restart,maxit", [(30, 30), (5, 12)])
def test_exact_start_vector_fixed_budget(restart, maxit):
    """the device-driven fixed-budget GMRES (rtol = 0) with x0 = the exact solution
    (zero initial residual, beta = 0) must leave x unchanged and finite, not turn it into NaN."""
    iga = _gpu()
    w, rp, ci, v, b = _system(3, 8)
    sp = iga.Space.from_workload(w)
    rng = np.random.default_rng(12)
    xs = rng.uniform(-1.0, 1.0, b.size)
    bb = krylov.csr_matvec(rp, ci, v, xs)                 # x0 = xs solves A x = bb up to rounding
    x0 = xs
    x, it, rr = sp.gmres(_dev(rp), _dev(ci), _dev(v), _dev(bb), x=_dev(x0), restart=restart, maxit=maxit, rtol=0.0,
                         precond=2, block_rows=32)
    xg = x.cpu().numpy()
    assert np.all(np.isfinite(xg)), "NaN / Inf in x"
    assert np.max(np.abs(xg - x0)) <= 1e-10 * np.max(np.abs(x0))
    # an exactly zero right-hand side with x0 = 0 on the same fixed-budget path
    z, itz, rrz = sp.gmres(_dev(rp), _dev(ci), _dev(v), _dev(np.zeros_like(b)), x=_dev(np.zeros_like(b)),
                           restart=restart, maxit=maxit, rtol=0.0, precond=2, block_rows=32)
    assert float(z.abs().max()) == 0.0


def test_full_size_newton_step_config3():
    """Config 3 at full size (1024^2 Cahn-Hilliard, 1M rows): the libiga Jacobian and residual,
    then the paper's 30 GMRES iterations; the reported residual is the true one (checked with
    torch's CSR product), and it decreases with the iteration count."""
    iga = _gpu()
    w = workloads.make(3)
    sp = iga.Space.from_workload(w)
    dev = torch.device("cuda", 0)
    rp, ci = sp.csr_pattern()
    ph = iga.make_phys(w.phys, w.params)
    vals, F = sp.form_jacobian(ph, w.a, w.b, _dev(w.U), _dev(w.Udot), want_F=True)
    sp.check()
    b = -F
    prev = np.inf
    for k in (1, 5, 30):
        x, it, rr = sp.gmres(rp, ci, vals, b, restart=30, maxit=k, rtol=0.0, precond=2)
        assert it == k
        A = torch.sparse_csr_tensor(rp, ci.to(torch.int64), vals, size=(b.numel(), b.numel()), device=dev)
        r = b - torch.mv(A, x)
        true = float(torch.linalg.norm(r) / torch.linalg.norm(b))
        assert abs(true - rr) <= 1e-8 * max(rr, 1e-14) + 1e-15
        assert rr < prev
        prev = rr
    assert prev < 1e-3          # the 4th-order CH system: ~3e-4 after the paper's 30 iterations


@pytest.mark.parametrize("restart,maxit,B,precond", [(60, 60, 0, 2), (7, 0, 0, 2), (30, 30, 100000, 2),
                                                     (30, 30, 2000, 2), (70, 70, 0, 1)])
def test_edge_cases(restart, maxit, B, precond):
    """restart > n (finite termination inside one cycle), maxit = 0 (x0 returned, true residual),
    one block covering the whole matrix (device ILU(0) through the CSR warp path = full ILU(0)),
    restart beyond the device-control limit (host path)."""
    iga = _gpu()
    w, rp, ci, v, b = _system(3, 6)               # 36 rows
    sp = iga.Space.from_workload(w)
    x0 = np.random.default_rng(2).uniform(-1e-3, 1e-3, b.size)
    x, it, rr = sp.gmres(_dev(rp), _dev(ci), _dev(v), _dev(b), x=_dev(x0), restart=restart, maxit=maxit, rtol=0.0,
                         precond=precond, block_rows=B)
    xo, ito, rro = krylov.gmres(rp, ci, v, b, x0=x0, restart=restart, maxit=maxit, rtol=0.0, precond=precond,
                                block_rows=B or 32)
    # past n iterations the Krylov space is exhausted: the host path stops at the (Pythagoras)
    # breakdown h_{j+1} = 0, the oracle's MGS norm stays at rounding level and it keeps iterating
    assert it == ito or (restart > b.size and b.size <= it <= ito)
    xg = x.cpu().numpy()
    if maxit == 0:
        assert np.array_equal(xg, x0)
    assert np.max(np.abs(xg - xo)) <= 1e-7 * np.max(np.abs(xo))
    assert abs(rr - rro) <= 1e-6 * max(rro, 1e-13) + 1e-13


def test_ring_and_nsk_systems():
    """GMRES on the Alg. 2 ring (NURBS, periodic) and on the nonsymmetric NSK Jacobian."""
    iga = _gpu()
    for cid, n in ((7, 8), (6, 7)):
        w, rp, ci, v, b = _system(cid, n)
        sp = iga.Space.from_workload(w)
        x, it, rr = sp.gmres(_dev(rp), _dev(ci), _dev(v), _dev(b), restart=30, maxit=30, rtol=0.0)
        xo, ito, rro = krylov.gmres(rp, ci, v, b, restart=30, maxit=30, rtol=0.0, precond=2, block_rows=32)
        assert it == ito == 30
        assert np.max(np.abs(x.cpu().numpy() - xo)) <= 1e-8 * np.max(np.abs(xo)), cid
