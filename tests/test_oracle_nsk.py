"""Pins of the oracle's Navier-Stokes-Korteweg integrand (P:774-801 strong
form, readings A-25..A-27).  The paper prints no NSK values; the weak form (reading A-25) is pinned
to the strong form it prints by a manufactured-solution convergence test (sympy-differentiated
strong residual vs the assembled weak residual, O(h^4)), plus the invariants the weak form must
satisfy on a periodic domain and finite differences of the residual against the Jacobian."""
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


def _strong_form(params):
    """The paper's strong form for manufactured smooth periodic fields,
    differentiated symbolically (sympy): returns numpy callables for the fields, their time
    derivatives and the residuals S_C = rho_t + div(rho u),
    S_M = (rho u)_t + div(rho u (x) u + p I) - div tau - div zeta."""
    import sympy as sp
    x, y = sp.symbols("x y", real=True)
    av, bv, Rg, th, mub, lamb, lam = [sp.Float(v) for v in params[:7]]
    tp = 2 * sp.pi
    rho = sp.Float(0.45) + sp.Float(0.1) * sp.sin(tp * x) * sp.cos(tp * y)
    u = [sp.Float(0.2) * sp.sin(tp * y), sp.Float(-0.15) * sp.cos(tp * x)]
    rho_t = sp.Float(0.3) * sp.cos(tp * x)
    u_t = [sp.Float(0.1) * sp.sin(tp * (x + y)), sp.Float(0.05) * sp.cos(tp * y)]
    X = [x, y]
    p = Rg * bv * rho * th / (bv - rho) - av * rho ** 2
    div_u = sum(sp.diff(u[k], X[k]) for k in range(2))
    lap_rho = sum(sp.diff(rho, X[k], 2) for k in range(2))
    g2 = sum(sp.diff(rho, X[k]) ** 2 for k in range(2))
    tau = [[mub * (sp.diff(u[i], X[j]) + sp.diff(u[j], X[i])) + (lamb * div_u if i == j else 0) for j in range(2)]
           for i in range(2)]
    zeta = [[(lam * (rho * lap_rho + g2 / 2) if i == j else 0) - lam * sp.diff(rho, X[i]) * sp.diff(rho, X[j])
             for j in range(2)] for i in range(2)]
    SC = rho_t + sum(sp.diff(rho * u[k], X[k]) for k in range(2))
    SM = [rho_t * u[i] + rho * u_t[i]
          + sum(sp.diff(rho * u[i] * u[j] + (p if i == j else 0) - tau[i][j] - zeta[i][j], X[j]) for j in range(2))
          for i in range(2)]
    f = lambda e: sp.lambdify((x, y), e, "numpy")
    return [f(rho), f(u[0]), f(u[1])], [f(rho_t), f(u_t[0]), f(u_t[1])], [f(SC), f(SM[0]), f(SM[1])]


def _interpolate(osp, n, funcs):
    """Least-squares fit of periodic spline coefficients to smooth functions at every element's
    Gauss points (basis values from the oracle's own, separately pinned, basis evaluation)."""
    g, _ = oracle.gauss_legendre(3)
    rows, vals = [], []
    nd = osp.ndof // 3
    for e0 in range(n):
        for e1 in range(n):
            for q0 in g:
                for q1 in g:
                    xi = ((e0 + (q0 + 1) / 2) / n, (e1 + (q1 + 1) / 2) / n)
                    r = osp.eval_point((e0, e1), xi)
                    row = np.zeros(nd)
                    np.add.at(row, r["node"], r["R"])
                    rows.append(row)
                    vals.append(xi)
    A = np.array(rows)
    pts = np.array(vals)
    coef = np.zeros((nd, len(funcs)))
    for k, fn in enumerate(funcs):
        coef[:, k] = np.linalg.lstsq(A, np.broadcast_to(fn(pts[:, 0], pts[:, 1]), len(pts)), rcond=None)[0]
    return coef


def test_weak_form_converges_to_the_papers_strong_form():
    """Pin of the NSK weak form (reading A-25) against the strong form the paper prints: for smooth
    periodic manufactured fields and test functions phi, sum_A phi_A . R_A(U_h, Udot_h) -> the
    integral of phi . S(u) as h -> 0 (integration by parts on the periodic domain).  A dropped or
    mis-signed flux, pressure, viscous or Korteweg term leaves an O(1) gap; the discretisation
    error shrinks with h."""
    w0 = _w(n=8, lam=1e-3)
    fields, dfields, strong = _strong_form(w0.params)
    tp = 2 * np.pi
    phis = [lambda x, y: np.cos(tp * x) * np.sin(tp * y), lambda x, y: np.sin(tp * x) + 0 * y,
            lambda x, y: np.cos(tp * (x - y))]
    m = 256                                     # trapezoid rule: spectral for smooth periodic integrands
    xs = (np.arange(m) + 0.5) / m
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    exact = sum(np.mean(phis[k](X, Y) * strong[k](X, Y)) for k in range(3))
    errs = []
    for n in (8, 16, 32):
        w = _w(n=n, lam=1e-3)
        osp = oracle.Space.from_workload(w)
        U = _interpolate(osp, n, fields).reshape(-1)
        V = _interpolate(osp, n, dfields).reshape(-1)
        P = _interpolate(osp, n, phis).reshape(-1)
        F = osp.assemble_dense(w.phys, w.params, w.a, w.b, U, V, want_K=False)[2]
        errs.append(abs(P @ F - exact))
    # measured: 3.3e-4, 2.1e-5, 1.3e-6 (O(h^4)); the Korteweg term alone contributes 5.6e-3 and the
    # pressure 0.29 to the integral, the viscous terms ~1e-3
    scale = sum(np.mean(np.abs(phis[k](X, Y) * strong[k](X, Y))) for k in range(3))
    assert errs[2] < 2e-5 * scale, (errs, scale)
    assert errs[1] < errs[0] / 8 and errs[2] < errs[1] / 8, errs
