"""Pins of the oracle's third-order basis (orc_eval_point3): eqs.
(dddrational) P:248-255, the inverse-map third derivative P:328-340 and (dddspatial) P:311-315.
Each pin comes from outside the oracle's formulas: closed forms, reproduction identities of the
isoparametric space, and finite differences of its (already pinned) second derivatives."""
import math

import numpy as np

import oracle
import workloads
from test_oracle_basis import _space1d_curve


def test_uniform_cubic_third_derivative_closed_form():
    """Interior uniform cubic B-splines on a span of length h: N''' = (-1, 3, -3, 1) / h^3."""
    h = 0.125                     # 8 elements: elements 3 and 4 carry four uniform cubics
    knots = [0, 0, 0] + [i * h for i in range(9)] + [1, 1, 1]
    sp = oracle.Space(2, [3, 3], [np.array(knots, float), np.array(knots, float)], [0, 0], [2, 2], 1, [4, 4],
                      oracle.PARAMETRIC, None, None)
    for t in (0.2, 0.5, 0.9):
        ev = sp.eval_point3([3, 4], [3 * h + t * h, 4 * h + 0.3 * h])
        # d^3/dx0^3 of M_A = N'''(x0) N(x1): sum over the a1 direction of the tensor product gives N'''
        d3 = ev["dddR"][:, 0, 0, 0].reshape(4, 4).sum(1)
        np.testing.assert_allclose(d3, np.array([-1, 3, -3, 1]) / h ** 3, rtol=0, atol=1e-9)
        # quadratic directions vanish: d^3/dx1^3 of a cubic in x1 is constant per function, sum = 0
        assert abs(ev["dddR"][:, 1, 1, 1].sum()) < 1e-8


def test_xi_squared_third_derivatives():
    """x = xi^2 (degree-2 Bezier map): xi = sqrt(x), xi_xxx = 3/(8 xi^5); R_A(x) = B_A(sqrt(x))
    differentiated three times in x in closed form -- pins P:328-340 and (dddspatial)."""
    sp = _space1d_curve([0, 0, 0, 1, 1, 1], 2, [0.0, 0.0, 1.0], None)
    B = [lambda t: (1 - t) ** 2, lambda t: 2 * t * (1 - t), lambda t: t * t]
    dB = [lambda t: -2 * (1 - t), lambda t: 2 - 4 * t, lambda t: 2 * t]
    ddB = [2.0, -4.0, 2.0]
    for xi in (0.3, 0.5, 0.8):
        ev = sp.eval_point3([0], [xi])
        xs, xss, xsss = 1 / (2 * xi), -1 / (4 * xi ** 3), 3 / (8 * xi ** 5)
        for A in range(3):
            # d3/dx3 f(xi(x)) = f''' xs^3 + 3 f'' xs xss + f' xsss  (f''' = 0 for quadratics)
            want = 3 * ddB[A] * xs * xss + dB[A](xi) * xsss
            assert abs(ev["dddR"][A, 0, 0, 0] - want) < 1e-10 * max(1.0, abs(want))


def _annulus_points(n=4, k=5, seed=3):
    w = workloads.make(2, n=n)
    sp = oracle.Space.from_workload(w)
    rng = np.random.default_rng(seed)
    pts = []
    for _ in range(k):
        e = [int(rng.integers(0, n)), int(rng.integers(0, n))]
        t = rng.uniform(0.15, 0.85, 2)
        pts.append((e, [(e[0] + t[0]) / n, (e[1] + t[1]) / n]))
    return w, sp, pts


def test_annulus_reproduction_third_order():
    """Isoparametric reproduction on the exact NURBS annulus (non-affine, rational): sum_A R_A = 1
    and sum_A x_A R_A = x hold identically, so every third spatial derivative of both vanishes --
    a dropped or mis-indexed term in (dddrational), xi_{,nlo} or (dddspatial) breaks it."""
    w, sp, pts = _annulus_points()
    ctrl = np.asarray(w.ctrl).reshape(-1, 2)
    for e, xi in pts:
        ev = sp.eval_point3(e, xi)
        d3 = ev["dddR"][:, :2, :2, :2]
        scale = np.abs(d3).max()
        assert scale > 1.0
        assert np.abs(d3.sum(0)).max() < 1e-11 * scale
        xA = ctrl[ev["node"]]
        for m in range(2):
            assert np.abs(np.tensordot(xA[:, m], d3, axes=(0, 0))).max() < 1e-11 * scale * np.abs(xA).max()
        # symmetry of the third derivative in (i, j, k)
        for p_ in [(0, 2, 1, 3), (0, 1, 3, 2), (0, 3, 2, 1)]:
            assert np.abs(d3 - np.transpose(d3, p_)).max() < 1e-11 * scale
        # lower orders unchanged w.r.t. the pinned evaluation
        ev2 = sp.eval_point(e, xi)
        np.testing.assert_allclose(ev["ddR"], ev2["ddR"], rtol=0, atol=1e-12 * np.abs(ev2["ddR"]).max())


def test_annulus_third_derivative_fd():
    """(dddspatial) against central differences of the pinned Hessian in physical coordinates
    (points moved through the inverse map by Newton on the FD-differentiated map)."""
    w, sp, pts = _annulus_points(k=3, seed=9)
    for e, xi in pts:
        ev = sp.eval_point3(e, xi)

        def hess_at_x(xp):
            z = np.array(xi, float)
            for _ in range(30):
                evz = sp.eval_point(e, z)
                J = np.zeros((2, 2))
                for al in range(2):
                    dz = np.zeros(2)
                    dz[al] = 1e-7
                    J[:, al] = (sp.eval_point(e, z + dz)["x"][:2] - sp.eval_point(e, z - dz)["x"][:2]) / 2e-7
                z = z - np.linalg.solve(J, evz["x"][:2] - xp)
            return sp.eval_point(e, z)["ddR"][:, :2, :2]

        x0 = ev["x"][:2]
        for k in range(2):
            def d(hs):
                dx = np.zeros(2)
                dx[k] = hs
                return (hess_at_x(x0 + dx) - hess_at_x(x0 - dx)) / (2 * hs)
            fd = (4 * d(1e-3) - d(2e-3)) / 3               # Richardson, O(h^4)
            got = ev["dddR"][:, :2, :2, k]
            np.testing.assert_allclose(got, fd, rtol=0, atol=2e-5 * np.abs(got).max())
