"""Pins of the solver oracle (oracle/krylov.py) against what the mathematics fixes, independent of
its own code: the ILU(0) defining property, exact LU without fill, point Jacobi at block size 1,
GMRES finite termination and the GMRES minimal-residual property over the Krylov space."""
import numpy as np
import pytest

from oracle import krylov


def _csr(Ad):
    n = Ad.shape[0]
    rp, ci, v = [0], [], []
    for i in range(n):
        nz = np.nonzero(Ad[i])[0]
        ci.extend(nz.tolist())
        v.extend(Ad[i, nz].tolist())
        rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int32), np.array(v)


def _random_sparse(n, density, seed, diag=4.0, sym_pattern=True):
    rng = np.random.default_rng(seed)
    mask = rng.random((n, n)) < density
    if sym_pattern:
        mask = mask | mask.T
    np.fill_diagonal(mask, True)
    A = np.where(mask, rng.uniform(-1, 1, (n, n)), 0.0)
    A[np.diag_indices(n)] += diag
    return A


def _unpack(rp, ci, lu, n):
    L, U = np.eye(n), np.zeros((n, n))
    for i in range(n):
        for p in range(rp[i], rp[i + 1]):
            j = ci[p]
            if j < i:
                L[i, j] = lu[p]
            else:
                U[i, j] = lu[p]
    return L, U


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ilu0_defining_property(seed):
    """(L U)_ij = a_ij for every (i, j) in NZ(A) (Saad Prop. 10.x: ILU(0) is the factorisation
    whose product matches A on its pattern)."""
    A = _random_sparse(40, 0.12, seed)
    rp, ci, v = _csr(A)
    lu = krylov.ilu0(rp, ci, v)
    L, U = _unpack(rp, ci, lu, 40)
    P = (L @ U)
    mask = A != 0
    assert np.max(np.abs(P[mask] - A[mask])) < 1e-12
    # and it is not the exact LU (fill was dropped) for a pattern with fill
    assert np.max(np.abs(P - A)) > 1e-8


def test_ilu0_no_fill_is_exact_lu():
    rng = np.random.default_rng(5)
    n = 30
    A = np.diag(rng.uniform(3, 4, n)) + np.diag(rng.uniform(-1, 1, n - 1), 1) + np.diag(rng.uniform(-1, 1, n - 1), -1)
    rp, ci, v = _csr(A)
    lu = krylov.ilu0(rp, ci, v)
    L, U = _unpack(rp, ci, lu, n)
    np.testing.assert_allclose(L @ U, A, atol=1e-13)
    b = rng.uniform(-1, 1, n)
    np.testing.assert_allclose(krylov.ilu0_solve(rp, ci, lu, b), np.linalg.solve(A, b), rtol=1e-12)


def test_block_jacobi_blocks():
    A = _random_sparse(24, 0.2, 7)
    rp, ci, v = _csr(A)
    b = np.random.default_rng(1).uniform(-1, 1, 24)
    # block size 1: point Jacobi
    M1 = krylov.make_precond(rp, ci, v, 2, block_rows=1)
    np.testing.assert_allclose(M1(b), b / np.diag(A), rtol=1e-14)
    # block size 8: block-diagonal ILU(0) equals ILU(0) of each diagonal block on its own
    M8 = krylov.make_precond(rp, ci, v, 2, block_rows=8)
    z = M8(b)
    for r0 in range(0, 24, 8):
        Ab = A[r0:r0 + 8, r0:r0 + 8]
        brp, bci, bv = _csr(Ab)
        zb = krylov.ilu0_solve(brp, bci, krylov.ilu0(brp, bci, bv), b[r0:r0 + 8])
        np.testing.assert_allclose(z[r0:r0 + 8], zb, rtol=1e-13)


@pytest.mark.parametrize("precond", [0, 1, 2])
def test_gmres_finite_termination(precond):
    n = 25
    A = _random_sparse(n, 0.15, 11, sym_pattern=False)
    rp, ci, v = _csr(A)
    b = np.random.default_rng(3).uniform(-1, 1, n)
    x, it, rr = krylov.gmres(rp, ci, v, b, restart=n, maxit=n, rtol=1e-14, precond=precond, block_rows=10)
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-9, atol=1e-11)
    assert rr < 1e-11 and it <= n


@pytest.mark.parametrize("m,precond", [(3, 0), (5, 1), (6, 2)])
def test_gmres_minimal_residual(m, precond):
    """x_m minimises ||b - A x|| over x0 + M^{-1} K_m(A M^{-1}, r0): brute force with an explicit
    (orthonormalised) Krylov basis and numpy's least squares."""
    n = 30
    A = _random_sparse(n, 0.15, 13, sym_pattern=False)
    rp, ci, v = _csr(A)
    rng = np.random.default_rng(4)
    b = rng.uniform(-1, 1, n)
    x0 = rng.uniform(-0.1, 0.1, n)
    x, it, _ = krylov.gmres(rp, ci, v, b, x0=x0, restart=m, maxit=m, rtol=0.0, precond=precond, block_rows=7)
    assert it == m
    Minv = krylov.make_precond(rp, ci, v, precond, 7)
    r0 = b - A @ x0
    K = [r0 / np.linalg.norm(r0)]
    for _ in range(m - 1):
        k = A @ Minv(K[-1])
        K.append(k / np.linalg.norm(k))
    Q, _ = np.linalg.qr(np.array(K).T)
    Y = np.array([Minv(Q[:, k]) for k in range(m)]).T        # search space M^{-1} K_m
    c, *_ = np.linalg.lstsq(A @ Y, r0, rcond=None)
    xb = x0 + Y @ c
    np.testing.assert_allclose(x, xb, rtol=1e-8, atol=1e-10)
    # residuals decrease monotonically in m
    prev = np.inf
    for k in range(1, m + 1):
        _, _, rk = krylov.gmres(rp, ci, v, b, x0=x0, restart=m, maxit=k, rtol=0.0, precond=precond, block_rows=7)
        assert rk <= prev * (1 + 1e-12)
        prev = rk


def test_gmres_restart_and_zero_rhs():
    n = 40
    A = _random_sparse(n, 0.1, 17, sym_pattern=False)
    rp, ci, v = _csr(A)
    b = np.random.default_rng(8).uniform(-1, 1, n)
    x, it, rr = krylov.gmres(rp, ci, v, b, restart=5, maxit=200, rtol=1e-10, precond=2, block_rows=10)
    assert rr <= 1e-10 and it < 200
    x, it, rr = krylov.gmres(rp, ci, v, np.zeros(n), restart=5, maxit=10, rtol=1e-10)
    assert it == 0 and np.all(x == 0)
