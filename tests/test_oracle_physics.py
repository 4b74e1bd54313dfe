"""Pins of the oracle's integrands, element integration and assembly: closed forms, invariants,
exact integration, FD Jacobians, manufactured-solution rates.  CPU only."""
import math

import numpy as np
import pytest

import oracle
import workloads


def fd_jacobian(sp, w, U, Udot, a, b, Utau=None, eps=1e-6, cols=None):
    """a dR/dUdot + b dR/dU by central differences of the oracle residual (dense, tiny spaces)."""
    nd = sp.ndof
    cols = range(nd) if cols is None else cols
    J = np.zeros((nd, len(list(cols))))
    for t, j in enumerate(cols):
        col = np.zeros(nd)
        if b != 0.0:
            Up, Um = U.copy(), U.copy()
            h = eps * max(1.0, abs(U[j]))
            Up[j] += h
            Um[j] -= h
            Fp = sp.assemble_dense(w.phys, w.params, 0, 0, Up, Udot, Utau=Utau, want_K=False)[2]
            Fm = sp.assemble_dense(w.phys, w.params, 0, 0, Um, Udot, Utau=Utau, want_K=False)[2]
            col += b * (Fp - Fm) / (2 * h)
        if a != 0.0:
            Vp, Vm = Udot.copy(), Udot.copy()
            h = eps * max(1.0, abs(Udot[j]))
            Vp[j] += h
            Vm[j] -= h
            Fp = sp.assemble_dense(w.phys, w.params, 0, 0, U, Vp, Utau=Utau, want_K=False)[2]
            Fm = sp.assemble_dense(w.phys, w.params, 0, 0, U, Vm, Utau=Utau, want_K=False)[2]
            col += a * (Fp - Fm) / (2 * h)
        J[:, t] = col
    return J


# ---- config 1: Poisson on the unit square ---------------------------------------------------
def test_poisson_invariants():
    w = workloads.make(1)
    sp = oracle.Space.from_workload(w)
    K, T, F = sp.assemble_dense(w.phys, w.params, w.a, w.b, w.U)
    assert np.abs(K - K.T).max() < 1e-15
    assert np.abs(K.sum(1)).max() < 1e-14          # rows sum to 0 (constants in the kernel)
    assert abs(-F.sum() - 8.0) < 1e-9              # sum F_A = int f = 8 (quadrature error 5.7e-11)
    rp, cols, _ = oracle.dense_to_csr(K, T)
    assert len(cols) == 7056
    # u = x: coefficients = Greville abscissae -> U^T K U = int |grad x|^2 = 1
    gre = w.ctrl[:, :, 0].reshape(-1)
    assert abs(gre @ K @ gre - 1.0) < 1e-13
    # u = x^2: coefficients tau_{i+1} tau_{i+2} (blossom) -> int |2x|^2 = 4/3
    U0 = w.knots[0]
    c = np.array([U0[i + 1] * U0[i + 2] for i in range(len(U0) - 3)])
    cx = np.repeat(c, len(c))
    assert abs(cx @ K @ cx - 4.0 / 3.0) < 1e-12


def _poisson_l2_error(n):
    w = workloads.make(1, n=n)
    sp = oracle.Space.from_workload(w)
    K, _, F = sp.assemble_dense(w.phys, w.params, 0.0, 1.0, w.U)
    nf = w.nfun[0]
    idx = np.arange(nf * nf).reshape(nf, nf)
    interior = idx[1:-1, 1:-1].reshape(-1)
    u = np.zeros(nf * nf)
    u[interior] = np.linalg.solve(K[np.ix_(interior, interior)], -F[interior])
    err2 = 0.0
    gx, gw = oracle.gauss_legendre(4)
    for e0 in range(n):
        for e1 in range(n):
            for q0 in range(4):
                for q1 in range(4):
                    xi = [(e0 + 0.5 + 0.5 * gx[q0]) / n, (e1 + 0.5 + 0.5 * gx[q1]) / n]
                    ev = sp.eval_point([e0, e1], xi)
                    uh = ev["R"] @ u[ev["node"]]
                    x, y = ev["x"][0], ev["x"][1]
                    err2 += (uh - math.sin(math.pi * x) * math.sin(math.pi * y)) ** 2 * gw[q0] * gw[q1] \
                        * ev["detJ"] / (4 * n * n)
    return math.sqrt(err2)


@pytest.mark.slow
def test_poisson_manufactured_rate():
    """Manufactured solution u = sin(pi x) sin(pi y): L2 rate >= 2.9 for p = 2."""
    e = [_poisson_l2_error(n) for n in (8, 16, 32)]
    rates = [math.log2(e[i] / e[i + 1]) for i in range(2)]
    assert min(rates) >= 2.9, (e, rates)


# ---- config 2: NURBS annulus, Laplace + mass --------------------------------------------------
@pytest.mark.parametrize("n,tol", [(4, 2e-12), (8, 1e-14)])
def test_annulus_mass_area(n, tol):
    """sigma only: sum M_AB = area of the quarter annulus = 3 pi / 4 (exact geometry)."""
    w = workloads.make(2, n=n)
    sp = oracle.Space.from_workload(w)
    M, _, _ = sp.assemble_dense(0, [0.0, 1.0, 0.0], 0.0, 1.0, w.U, want_F=False)
    assert abs(M.sum() - 0.75 * math.pi) / (0.75 * math.pi) < tol
    assert np.abs(M - M.T).max() < 1e-16
    assert M.min() >= 0.0


def test_annulus_laplace_rows_and_linear_residual():
    w = workloads.make(2, n=4)
    sp = oracle.Space.from_workload(w)
    K, T, _ = sp.assemble_dense(0, [1.0, 0.0, 0.0], 0.0, 1.0, w.U, want_F=False)
    assert np.abs(K.sum(1)).max() < 1e-13 * np.abs(K).max()
    assert np.abs(K - K.T).max() < 1e-14 * np.abs(K).max()
    # linear problem: R(U) = K U (kappa = sigma = 1, f = 0)
    K2, _, F = sp.assemble_dense(w.phys, w.params, 0.0, 1.0, w.U)
    assert np.abs(F - K2 @ w.U).max() < 1e-13 * np.abs(F).max()
    # pattern: touched == Alg. 3 pattern, and tight (mass matrix has no structural zero)
    rp, cols = sp.pattern()
    rp2, cols2, v = oracle.dense_to_csr(K2, T)
    assert np.array_equal(rp, rp2) and np.array_equal(cols, cols2)
    M, _, _ = sp.assemble_dense(0, [0.0, 1.0, 0.0], 0.0, 1.0, w.U, want_F=False)
    assert np.all(M[T.astype(bool)] > 0)


# ---- config 3: Cahn-Hilliard ------------------------------------------------------------------
def test_ch_constant_state_zero_residual_and_mass():
    w = workloads.make(3, n=6)
    sp = oracle.Space.from_workload(w)
    U = np.full(sp.ndof, 0.6)
    _, _, F = sp.assemble_dense(w.phys, w.params, 0, 0, U, np.zeros(sp.ndof), want_K=False)
    assert np.abs(F).max() < 1e-12
    # sum_A R_A = int cdot (periodic; every other term carries grad N_A or lap N_A)
    rng = np.random.default_rng(0)
    Ud = rng.uniform(-1, 1, sp.ndof)
    _, _, F = sp.assemble_dense(w.phys, w.params, 0, 0, w.U, Ud, want_K=False)
    # int cdot^h = sum_B Udot_B int N_B = sum_B Udot_B / N^2 (uniform periodic: int N_B = h^2)
    assert abs(F.sum() - Ud.sum() / 36.0) < 1e-11


def test_ch_linearised_at_constant_is_symmetric():
    """dR/dc at constant c0 = M mu'(c0) L + M(c0) Bilap: symmetric, rows sum to zero."""
    w = workloads.make(3, n=6)
    sp = oracle.Space.from_workload(w)
    U = np.full(sp.ndof, 0.61)
    K, _, _ = sp.assemble_dense(w.phys, w.params, 0.0, 1.0, U, np.zeros(sp.ndof), want_F=False)
    assert np.abs(K - K.T).max() < 1e-11 * np.abs(K).max()
    assert np.abs(K.sum(1)).max() < 1e-10 * np.abs(K).max()


def test_ch_fd_jacobian():
    w = workloads.make(3, n=5)
    sp = oracle.Space.from_workload(w)
    rng = np.random.default_rng(3)
    Ud = rng.uniform(-1, 1, sp.ndof)
    for a, b in ((1.0, 0.0), (0.0, 1.0), (5 / 6, 0.37)):
        K, _, _ = sp.assemble_dense(w.phys, w.params, a, b, w.U, Ud, want_F=False)
        J = fd_jacobian(sp, w, w.U, Ud, a, b, eps=1e-6)
        assert np.abs(K - J).max() < 2e-6 * np.abs(K).max(), (a, b)


# ---- config 4: Neo-Hookean ---------------------------------------------------------------------
def _nh_small(n=2):
    return workloads.make(4, n=n)


def test_nh_zero_displacement_and_linear_elasticity():
    w = _nh_small()
    sp = oracle.Space.from_workload(w)
    U0 = np.zeros(sp.ndof)
    K, _, F = sp.assemble_dense(w.phys, w.params, 0.0, 1.0, U0)
    assert np.abs(F).max() < 1e-15
    lam, mu = w.params
    # independent linear-elasticity stiffness from the pushed-forward basis
    Kle = np.zeros_like(K)
    gx, gw = oracle.gauss_legendre(3)
    n = w.nel[0]
    for e in np.ndindex(n, n, n):
        for q in np.ndindex(3, 3, 3):
            xi = [(e[d] + 0.5 + 0.5 * gx[q[d]]) / n for d in range(3)]
            ev = sp.eval_point(list(e), xi)
            wq = gw[q[0]] * gw[q[1]] * gw[q[2]] / (8 * n ** 3) * ev["detJ"]
            G = ev["dR"]
            for A in range(27):
                for B in range(27):
                    for i in range(3):
                        for j in range(3):
                            v = lam * G[A, i] * G[B, j] + mu * G[A, j] * G[B, i] + (mu * G[A] @ G[B] if i == j else 0)
                            Kle[ev["node"][A] * 3 + i, ev["node"][B] * 3 + j] += v * wq
    assert np.abs(K - Kle).max() < 1e-13 * np.abs(K).max()


def test_nh_invariance_and_symmetry():
    w = _nh_small()
    sp = oracle.Space.from_workload(w)
    K, _, F = sp.assemble_dense(w.phys, w.params, 0.0, 1.0, w.U)
    assert np.abs(K - K.T).max() < 1e-13 * np.abs(K).max()       # major symmetry
    nn = sp.ndof // 3
    for d in range(3):
        t = np.zeros((nn, 3)); t[:, d] = 1.0
        t = t.reshape(-1)
        assert np.abs(K @ t).max() < 1e-12 * np.abs(K).max()      # translations in the kernel
        _, _, F2 = sp.assemble_dense(w.phys, w.params, 0.0, 1.0, w.U + 0.3 * t, want_K=False)
        assert np.abs(F2 - F).max() < 1e-13 * np.abs(F).max()
    # infinitesimal rotations at u = 0 are in the kernel of K(0): u = W X
    K0, _, _ = sp.assemble_dense(w.phys, w.params, 0.0, 1.0, np.zeros(sp.ndof), want_F=False)
    g = [np.array([(w.knots[d][i + 1] + w.knots[d][i + 2]) / 2 for i in range(w.nfun[d])]) for d in range(3)]
    X = np.stack(np.meshgrid(*g, indexing="ij"), -1).reshape(-1, 3)
    for Wm in (np.array([[0, 1, 0], [-1, 0, 0], [0, 0, 0.]]), np.array([[0, 0, 1], [0, 0, 0], [-1, 0, 0.]])):
        r = (X @ Wm.T).reshape(-1)
        assert np.abs(K0 @ r).max() < 1e-12 * np.abs(K0).max()


def test_nh_affine_displacement_interior_rows_vanish():
    w = workloads.make(4, n=3)
    sp = oracle.Space.from_workload(w)
    g = [np.array([(w.knots[d][i + 1] + w.knots[d][i + 2]) / 2 for i in range(w.nfun[d])]) for d in range(3)]
    X = np.stack(np.meshgrid(*g, indexing="ij"), -1)
    Hm = np.array([[0.05, 0.02, -0.01], [0.0, -0.03, 0.04], [0.01, 0.0, 0.02]])
    U = (X @ Hm.T).reshape(-1)                     # u = H X exactly (Greville coefficients)
    _, _, F = sp.assemble_dense(w.phys, w.params, 0.0, 1.0, U, want_K=False)
    nf = w.nfun[0]
    Fr = F.reshape(nf, nf, nf, 3)
    assert np.abs(Fr[1:-1, 1:-1, 1:-1]).max() < 1e-14
    assert np.abs(Fr).max() > 1e-4


def test_nh_fd_jacobian():
    w = _nh_small()
    sp = oracle.Space.from_workload(w)
    K, _, _ = sp.assemble_dense(w.phys, w.params, 0.0, 1.0, w.U, want_F=False)
    cols = list(range(0, sp.ndof, 7))
    J = fd_jacobian(sp, w, w.U, np.zeros(sp.ndof), 0.0, 1.0, eps=1e-6, cols=cols)
    assert np.abs(K[:, cols] - J).max() < 1e-7 * np.abs(K).max()


# ---- config 5: RBVMS Navier-Stokes -------------------------------------------------------------
def _ns_small(n=5):
    return workloads.make(5, n=n)


def test_vms_constant_state_and_continuity_sum():
    w = _ns_small()
    sp = oracle.Space.from_workload(w)
    nn = sp.ndof // 4
    U = np.tile([0.3, -0.2, 0.5, 1.7], nn)
    _, _, F = sp.assemble_dense(w.phys, w.params, 0, 0, U, np.zeros(sp.ndof), want_K=False)
    assert np.abs(F).max() < 1e-13
    _, _, F = sp.assemble_dense(w.phys, w.params, 0, 0, w.U, np.zeros(sp.ndof), want_K=False)
    Fr = F.reshape(nn, 4)
    assert abs(Fr[:, 3].sum()) < 1e-12 * np.abs(Fr[:, 3]).max() * nn      # sum_A R^C_A = int div u = 0
    assert np.abs(Fr).max() > 1e-6


def test_vms_fd_jacobian_frozen_tau():
    w = _ns_small()
    sp = oracle.Space.from_workload(w)
    rng = np.random.default_rng(5)
    Ud = 0.1 * rng.uniform(-1, 1, sp.ndof)
    cols = list(range(0, sp.ndof, 13)) + [3, 7, 11]
    for a, b in ((1.0, 0.0), (0.0, 1.0)):
        K, _, _ = sp.assemble_dense(w.phys, w.params, a, b, w.U, Ud, want_F=False)
        J = fd_jacobian(sp, w, w.U, Ud, a, b, Utau=w.U, eps=1e-6, cols=cols)
        assert np.abs(K[:, cols] - J).max() < 1e-7 * np.abs(K[:, cols]).max(), (a, b)


def test_vms_stokes_limit_skew_coupling():
    """u = 0, tau = 0 (C_t -> inf): K_up = -K_pu^T (Galerkin Stokes)."""
    w = _ns_small()
    sp = oracle.Space.from_workload(w)
    U = np.zeros(sp.ndof)
    # dt = 1e-150 -> tau_M ~ dt -> 0 (and tau_C large, which only enters the u-u grad-div block)
    K, _, _ = sp.assemble_dense(w.phys, [w.params[0], 1e-150, 1.0, 36.0], 0.0, 1.0, U, np.zeros(sp.ndof), want_F=False)
    nn = sp.ndof // 4
    Kr = K.reshape(nn, 4, nn, 4)
    Kup = Kr[:, :3, :, 3].reshape(nn * 3, nn)
    Kpu = Kr[:, 3, :, :3].reshape(nn, nn * 3)
    # tau_M ~ dt tiny -> tau_C = 1/(tau_M g.g) large: only the grad-div term (symmetric in u-u) grows,
    # the u-p / p-u blocks are tau-free up to O(tau_M) corrections
    assert np.abs(Kup + Kpu.T).max() < 1e-9 * np.abs(Kup).max()


# ---- assembly: rows mode == dense mode, touched == pattern -----------------------------------
@pytest.mark.parametrize("cid,n", [(1, 5), (2, 3), (3, 5), (4, 2), (5, 5)])
def test_rows_mode_equals_dense(cid, n):
    w = workloads.make(cid, n=n)
    sp = oracle.Space.from_workload(w)
    rng = np.random.default_rng(cid)
    Ud = rng.uniform(-0.1, 0.1, sp.ndof) if w.phys in (1, 3) else np.zeros(sp.ndof)
    K, T, F = sp.assemble_dense(w.phys, w.params, w.a, w.b, w.U, Ud)
    rp, cols = sp.pattern()
    rp2, cols2, vals = oracle.dense_to_csr(K, T)
    assert np.array_equal(rp, rp2) and np.array_equal(cols, cols2)      # Alg. 3 == touched entries
    rows = np.sort(rng.choice(sp.ndof, size=min(sp.ndof, 40), replace=False))
    r = sp.assemble_rows(w.phys, w.params, w.a, w.b, w.U, rows, Udot=Ud)
    assert r["touched"].all()
    for t, row in enumerate(rows):
        seg = slice(r["rowptr"][t], r["rowptr"][t + 1])
        np.testing.assert_array_equal(r["cols"][seg], cols[rp[row]:rp[row + 1]])
        np.testing.assert_allclose(r["vals"][seg], vals[rp[row]:rp[row + 1]], rtol=0,
                                   atol=1e-14 * max(1e-300, np.abs(vals[rp[row]:rp[row + 1]]).max()))
    np.testing.assert_allclose(r["F"], F[rows], rtol=0, atol=1e-14 * np.abs(F).max())


def test_periodic_pattern_counts():
    """Periodic uniform C^{p-1}: every row has (2p+1)^d m^2 / m entries (stencil 2p+1 per axis)."""
    w = workloads.make(5, n=5)
    sp = oracle.Space.from_workload(w)
    rp, cols = sp.pattern_rows(np.arange(0, sp.ndof, 17))
    assert np.all(np.diff(rp) == 125 * 4)
    w = workloads.make(3, n=8)
    sp = oracle.Space.from_workload(w)
    rp, cols = sp.pattern()
    assert np.all(np.diff(rp) == 25)
    assert len(cols) == 25 * 64
