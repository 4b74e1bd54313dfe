"""Pins of the oracle's Navier-Stokes-Korteweg integrand (P:774-801 strong
form, readings A-25..A-27).  The paper prints no NSK values, so the integrand itself is parity
unpinned (as CH and VMS): these are the invariants the weak form must satisfy on a periodic
domain, and finite differences of the residual against the Jacobian."""
import numpy as np

import oracle
import workloads
from test_oracle_physics import fd_jacobian


def _w(n=6, lam=None):
    w = workloads.make(6, n=n)
    if lam is not None:
        w.params = list(w.params)
        w.params[6] = lam
    return w


def test_constant_state_residual_vanishes():
    """rho, u constant and no time derivative: every flux is constant and every divergence of a
    compactly supported basis function integrates to zero."""
    w = _w()
    sp = oracle.Space.from_workload(w)
    U = np.tile([0.45, 0.3, -0.2], sp.ndof // 3)
    F = sp.assemble_dense(w.phys, w.params, w.a, w.b, U, np.zeros_like(U), want_K=False)[2]
    assert np.abs(F).max() < 1e-14


def test_conservation_sums():
    """Summing the rows over the test functions (partition of unity, Sum_A grad N_A = 0) leaves
    only the time-derivative integrals -- fluxes, pressure, viscous and Korteweg terms are
    conservative.  With u = c constant and u_t = d constant those integrals have closed forms
    through int N_B = h^2 (uniform periodic quadratics, h = 1/n):
    Sum_A R^C_A = h^2 Sum_B rho_t,B,  Sum_A R^M_{A,i} = h^2 (c_i Sum_B rho_t,B + d_i Sum_B rho_B)."""
    n = 6
    w = _w(n=n, lam=1e-2)
    sp = oracle.Space.from_workload(w)
    rng = np.random.default_rng(11)
    U = w.U.reshape(-1, 3).copy()
    c, d = np.array([0.3, -0.2]), np.array([0.05, 0.07])
    U[:, 1:] = c                                  # rho keeps the bubbles; u constant
    V = np.zeros_like(U)
    V[:, 0] = rng.uniform(-1, 1, len(U))          # rho_t arbitrary
    V[:, 1:] = d
    F = sp.assemble_dense(w.phys, w.params, w.a, w.b, U.reshape(-1), V.reshape(-1), want_K=False)[2].reshape(-1, 3)
    h2 = 1.0 / n ** 2
    want = [h2 * V[:, 0].sum(), *(h2 * (c * V[:, 0].sum() + d * U[:, 0].sum()))]
    np.testing.assert_allclose(F.sum(0), want, rtol=0, atol=1e-13 * np.abs(F).max() * len(F))


def test_one_dimensional_density_has_no_transverse_pressure():
    """rho = rho(x0) only, u = 0, no time derivatives: the x1-momentum rows integrate
    N_{A,1} against functions of x0 only, which vanishes on the periodic x1 axis."""
    w = _w(lam=1e-2)
    sp = oracle.Space.from_workload(w)
    n = w.nfun
    x0 = (np.arange(n[0]) + 0.5) / n[0]
    rho = 0.35 + 0.2 * np.sin(2 * np.pi * x0)
    U = np.zeros((n[0], n[1], 3))
    U[..., 0] = rho[:, None]
    F = sp.assemble_dense(w.phys, w.params, w.a, w.b, U.reshape(-1), np.zeros(U.size), want_K=False)[2]
    F = F.reshape(n[0], n[1], 3)
    assert np.abs(F[..., 2]).max() < 1e-13 * max(np.abs(F).max(), 1e-300)
    assert np.abs(F[..., 1]).max() > 1e-6            # the x0 momentum does see the pressure gradient


def test_nsk_fd_jacobian():
    """J = a dR/dUdot + b dR/dU against central differences, for the a part, the b part and a
    mix, with a capillarity large enough that the Korteweg terms dominate their rows."""
    w = _w(n=5, lam=1e-2)
    sp = oracle.Space.from_workload(w)
    for a, b in ((1.0, 0.0), (0.0, 1.0), (5 / 6, 0.37)):
        K, _, _ = sp.assemble_dense(w.phys, w.params, a, b, w.U, w.Udot, want_F=False)
        J = fd_jacobian(sp, w, w.U, w.Udot, a, b, eps=1e-6)
        assert np.abs(K - J).max() < 2e-6 * np.abs(K).max(), (a, b)
