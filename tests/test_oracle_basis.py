"""Pins of the oracle's basis / knot / quadrature / geometry layer against what the paper and
mathematics fix (not against the oracle itself).  CPU only."""
import itertools
import math
import os

import numpy as np
import pytest

import oracle
import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---- Gauss-Legendre (A-6): closed forms + exactness ---------------------------------------
def test_gauss_legendre_closed_forms():
    x, w = oracle.gauss_legendre(3)
    np.testing.assert_allclose(x, [-math.sqrt(3 / 5), 0.0, math.sqrt(3 / 5)], rtol=0, atol=2e-16)
    np.testing.assert_allclose(w, [5 / 9, 8 / 9, 5 / 9], rtol=0, atol=2e-16)
    x, w = oracle.gauss_legendre(4)
    a = math.sqrt(3 / 7 - 2 / 7 * math.sqrt(6 / 5))
    b = math.sqrt(3 / 7 + 2 / 7 * math.sqrt(6 / 5))
    np.testing.assert_allclose(x, [-b, -a, a, b], rtol=0, atol=3e-16)
    wa, wb = (18 + math.sqrt(30)) / 36, (18 - math.sqrt(30)) / 36
    np.testing.assert_allclose(w, [wb, wa, wa, wb], rtol=0, atol=3e-16)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7])
def test_gauss_legendre_exact_degree(n):
    x, w = oracle.gauss_legendre(n)
    for deg in range(2 * n):
        exact = 0.0 if deg % 2 else 2.0 / (deg + 1)
        assert abs(np.sum(w * x ** deg) - exact) < 1e-14
    # and NOT exact one degree above (the rule is Gauss, not something larger)
    deg = 2 * n
    assert abs(np.sum(w * x ** deg) - 2.0 / (deg + 1)) > 1e-8


# ---- Alg. 1 (Fig. 2) ------------------------------------------------------------------------
def _read_fig2():
    out = {}
    for line in open(os.path.join(GOLDEN, "fig2_unclamped_knots.txt")):
        if line.startswith("#") or not line.strip():
            continue
        key, vals = line.split(":")
        out[key.strip()] = np.array([float(v) for v in vals.split()])
    return out


@pytest.mark.parametrize("k", [0, 1, 2])
def test_unclamp_fig2(k):
    g = _read_fig2()
    got = oracle.unclamp_knots(7, 3, k, g["open"])
    # A-3: fp64 Alg. 1 is not bit-exact to the printed decimals; compare to 1 ulp
    assert np.all(np.abs(got - g[str(k)]) <= np.spacing(np.maximum(np.abs(g[str(k)]), 1.0)))


# ---- Alg. 3 (Fig. 3) ------------------------------------------------------------------------
def _read_fig3():
    rows = []
    U = p = None
    for line in open(os.path.join(GOLDEN, "fig3_pattern.txt")):
        if line.startswith("#") or not line.strip():
            continue
        if line.startswith("knots:"):
            U = [float(v) for v in line.split(":")[1].split()]
        elif line.startswith("p:"):
            p = int(line.split(":")[1])
        else:
            rows.append([c == "o" for c in line.strip()])
    return U, p, np.array(rows)


def test_stencil_fig3():
    U, p, pat = _read_fig3()
    n = len(U) - p - 1
    got = np.zeros((n, n), bool)
    for i in range(n):
        l, r = oracle.basis_stencil(i, p, U)
        got[i, l:r + 1] = True
    assert np.array_equal(got, pat)
    # symmetry of the adjacency
    assert np.array_equal(got, got.T)


def test_stencil_vs_support_overlap():
    """Alg. 3 == brute-force support overlap (nonzero at a common interior point)."""
    rng = np.random.default_rng(0)
    for trial in range(20):
        p = int(rng.integers(1, 4))
        interior = np.sort(rng.integers(1, 8, size=int(rng.integers(2, 9)))).astype(float)
        U = np.concatenate([[0.0] * (p + 1), interior, [8.0] * (p + 1)])
        # cap multiplicity at p (keep C^0)
        vals, cnt = np.unique(interior, return_counts=True)
        if np.any(cnt > p):
            continue
        n = len(U) - p - 1
        pts = np.linspace(0, 8, 4001)[:-1] + 1e-4
        B = np.array([[oracle.coxdeboor(i, p, U, x) for x in pts] for i in range(n)]) != 0
        for i in range(n):
            l, r = oracle.basis_stencil(i, p, U)
            overl = [j for j in range(n) if np.any(B[i] & B[j])]
            assert overl == list(range(l, r + 1)), (U, p, i)


# ---- Cox-de Boor: closed forms ------------------------------------------------------------
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_bernstein(p):
    U = [0.0] * (p + 1) + [1.0] * (p + 1)
    for t in (0.1, 0.37, 0.5, 0.9):
        for i in range(p + 1):
            exact = math.comb(p, i) * t ** i * (1 - t) ** (p - i)
            assert abs(oracle.coxdeboor(i, p, U, t) - exact) < 1e-15
            # derivative of the Bernstein polynomial
            d = math.comb(p, i) * (i * t ** (i - 1) * (1 - t) ** (p - i) if i > 0 else 0.0) \
                - math.comb(p, i) * ((p - i) * t ** i * (1 - t) ** (p - i - 1) if i < p else 0.0)
            assert abs(oracle.coxdeboor(i, p, U, t, 1) - d) < 1e-13


def test_quadratic_half():
    U = [0, 0, 0, 1, 1, 1]
    assert [oracle.coxdeboor(i, 2, U, 0.5) for i in range(3)] == [0.25, 0.5, 0.25]
    assert [oracle.coxdeboor(i, 2, U, 0.5, 1) for i in range(3)] == [-1.0, 0.0, 1.0]


@pytest.mark.parametrize("p", [2, 3])
def test_uniform_interior_closed_form(p):
    h = 0.25
    U = workloads.open_uniform_knots(p, 12, 0.0, 3.0)   # h = 0.25
    # interior element e = 6: span s = p + 6, functions s-p..s, local t in [0,1]
    s = p + 6
    if p == 2:
        f = [lambda t: (1 - t) ** 2 / 2, lambda t: (-2 * t * t + 2 * t + 1) / 2, lambda t: t * t / 2]
        f1 = [lambda t: -(1 - t), lambda t: -2 * t + 1, lambda t: t]
        f2 = [lambda t: 1.0, lambda t: -2.0, lambda t: 1.0]
    else:
        f = [lambda t: (1 - t) ** 3 / 6, lambda t: (3 * t ** 3 - 6 * t * t + 4) / 6,
             lambda t: (-3 * t ** 3 + 3 * t * t + 3 * t + 1) / 6, lambda t: t ** 3 / 6]
        f1 = [lambda t: -(1 - t) ** 2 / 2, lambda t: (9 * t * t - 12 * t) / 6,
              lambda t: (-9 * t * t + 6 * t + 3) / 6, lambda t: t * t / 2]
        f2 = [lambda t: (1 - t), lambda t: (18 * t - 12) / 6, lambda t: (-18 * t + 6) / 6, lambda t: t]
    for t in (0.05, 0.3, 0.5, 0.77):
        xi = U[s] + t * h
        for a in range(p + 1):
            i = s - p + a
            assert abs(oracle.coxdeboor(i, p, U, xi) - f[a](t)) < 1e-15
            assert abs(oracle.coxdeboor(i, p, U, xi, 1) - f1[a](t) / h) < 1e-13
            assert abs(oracle.coxdeboor(i, p, U, xi, 2) - f2[a](t) / h ** 2) < 1e-11


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_partition_of_unity_and_fd(p):
    rng = np.random.default_rng(p)
    interior = np.sort(rng.uniform(0, 1, 6))
    U = np.concatenate([[0.0] * (p + 1), interior, [1.0] * (p + 1)])
    n = len(U) - p - 1
    for x in rng.uniform(0.001, 0.999, 25):
        vals = [oracle.coxdeboor(i, p, U, x) for i in range(n)]
        assert abs(sum(vals) - 1.0) < 1e-14
        assert min(vals) >= 0.0
        assert abs(sum(oracle.coxdeboor(i, p, U, x, 1) for i in range(n))) < 1e-10
        if p >= 2:
            assert abs(sum(oracle.coxdeboor(i, p, U, x, 2) for i in range(n))) < 1e-7
        # FD of the derivative (away from knots)
        if np.min(np.abs(U - x)) > 1e-3:
            e = 1e-6
            for i in range(n):
                fd = (oracle.coxdeboor(i, p, U, x + e) - oracle.coxdeboor(i, p, U, x - e)) / (2 * e)
                assert abs(fd - oracle.coxdeboor(i, p, U, x, 1)) < 1e-6 * max(1.0, abs(fd))
                if p >= 2:
                    fd2 = (oracle.coxdeboor(i, p, U, x + e, 1) - oracle.coxdeboor(i, p, U, x - e, 1)) / (2 * e)
                    assert abs(fd2 - oracle.coxdeboor(i, p, U, x, 2)) < 1e-5 * max(1.0, abs(fd2))


# ---- rational / geometry ---------------------------------------------------------------------
def _space1d_curve(U, p, ctrl, weights):
    return oracle.Space(1, [p], [np.array(U, float)], [0], [p - 1], 1, [p + 1], oracle.NURBS,
                        np.array(ctrl, float).reshape(-1, 1), None if weights is None else np.array(weights, float))


def test_arc_rational_values():
    """Quarter arc: w(1/2) = 0.853553..., R = (0.292893, 0.414214, 0.292893)."""
    s2 = math.sqrt(2)
    sp = oracle.Space(1, [2], [np.array([0, 0, 0, 1, 1, 1.0])], [0], [1], 1, [3], oracle.PARAMETRIC,
                      None, np.array([1.0, 1 / s2, 1.0]))
    ev = sp.eval_point([0], [0.5])
    w = 0.25 + 0.5 / s2 + 0.25
    assert abs(w - 0.8535533905932737) < 1e-15
    np.testing.assert_allclose(ev["R"], [0.25 / w, 0.5 / s2 / w, 0.25 / w], rtol=1e-15)
    np.testing.assert_allclose(ev["R"], [0.292893218813, 0.414213562373, 0.292893218813], atol=1e-12)
    assert abs(ev["R"].sum() - 1) < 1e-15
    assert abs(ev["dR"][:, 0].sum()) < 1e-14


def test_unit_weights_reduce_to_bsplines():
    U = workloads.open_uniform_knots(3, 5)
    n = len(U) - 4
    ctrl = np.linspace(0, 1, n)
    a = _space1d_curve(U, 3, ctrl, np.ones(n))
    b = _space1d_curve(U, 3, ctrl, None)
    for e in range(5):
        for t in (0.1, 0.6):
            xi = U[3 + e] + t * 0.2
            ea, eb = a.eval_point([e], [xi]), b.eval_point([e], [xi])
            assert np.array_equal(ea["R"], eb["R"])
            for ii, i in enumerate(range(e, e + 4)):
                assert abs(ea["R"][ii] - oracle.coxdeboor(i, 3, U, xi)) < 1e-15


def test_affine_scaling_map():
    """x = s*xi + c: xi_{,x} = 1/s, detJ = s^d, grad N = dN/dxi / s, hess = d2N/dxi2 / s^2."""
    s_ = 2.5
    U = workloads.open_uniform_knots(2, 4)
    gre = np.array([(U[i + 1] + U[i + 2]) / 2 for i in range(len(U) - 3)])
    n = len(gre)
    ctrl = np.zeros((n, n, 2))
    ctrl[:, :, 0] = s_ * gre[:, None] + 1.0
    ctrl[:, :, 1] = s_ * gre[None, :] - 3.0
    sp = oracle.Space(2, [2, 2], [U, U], [0, 0], [1, 1], 1, [3, 3], oracle.NURBS, ctrl, np.ones((n, n)))
    par = oracle.Space(2, [2, 2], [U, U], [0, 0], [1, 1], 1, [3, 3], oracle.PARAMETRIC, None, None)
    e, xi = [1, 2], [0.3, 0.6]
    a, b = sp.eval_point(e, xi), par.eval_point(e, xi)
    assert abs(a["detJ"] - s_ ** 2) < 1e-13
    np.testing.assert_allclose(a["x"][:2], [s_ * 0.3 + 1, s_ * 0.6 - 3], atol=1e-14)
    np.testing.assert_allclose(a["R"], b["R"], atol=1e-15)
    np.testing.assert_allclose(a["dR"], b["dR"] / s_, atol=1e-12)
    np.testing.assert_allclose(a["ddR"], b["ddR"] / s_ ** 2, atol=1e-10)


def test_xi_squared_inverse_map():
    """1D map x = xi^2 on [0,1]: xi = sqrt(x), xi_x = 1/(2 xi), xi_xx = -1/(4 xi^3).
    Pins eqs. (dspatial) and (ddspatial) including the inverse-map second derivative P:316-327."""
    sp = _space1d_curve([0, 0, 0, 1, 1, 1], 2, [0.0, 0.0, 1.0], None)
    for xi in (0.3, 0.5, 0.8):
        ev = sp.eval_point([0], [xi])
        assert abs(ev["x"][0] - xi * xi) < 1e-15
        assert abs(ev["detJ"] - 2 * xi) < 1e-14
        x = xi * xi
        # Bernstein B_i(sqrt(x)) differentiated twice in x, closed form
        B = [lambda t: (1 - t) ** 2, lambda t: 2 * t * (1 - t), lambda t: t * t]
        dB = [lambda t: -2 * (1 - t), lambda t: 2 - 4 * t, lambda t: 2 * t]
        ddB = [lambda t: 2.0, lambda t: -4.0, lambda t: 2.0]
        xs, xss = 1 / (2 * xi), -1 / (4 * xi ** 3)
        for A in range(3):
            assert abs(ev["R"][A] - B[A](xi)) < 1e-15
            assert abs(ev["dR"][A, 0] - dB[A](xi) * xs) < 1e-13
            assert abs(ev["ddR"][A, 0, 0] - (ddB[A](xi) * xs ** 2 + dB[A](xi) * xss)) < 1e-12
        del x


def test_annulus_geometry_and_pushforward_fd():
    """Exact quarter annulus (A-20): |x| = 1 + xi0; physical gradient/Hessian vs FD in x."""
    w = workloads.make(2, n=4)
    sp = oracle.Space.from_workload(w)
    rng = np.random.default_rng(1)
    for _ in range(6):
        e = [int(rng.integers(0, 4)), int(rng.integers(0, 4))]
        t = rng.uniform(0.2, 0.8, 2)
        xi = [(e[0] + t[0]) / 4, (e[1] + t[1]) / 4]
        ev = sp.eval_point(e, xi)
        r = math.hypot(ev["x"][0], ev["x"][1])
        assert abs(r - (1 + xi[0])) < 2e-15 * 4
        assert ev["detJ"] > 1.4
        # FD in physical coordinates: perturb x via the inverse map (Newton on the map)
        def R_at_x(xp):
            z = np.array(xi, float)
            for _ in range(30):
                evz = sp.eval_point(e, z)
                J = np.zeros((2, 2))
                # x_{i,alpha} by FD of the map (independent of the oracle's derivative code)
                for al in range(2):
                    dz = np.zeros(2); dz[al] = 1e-7
                    J[:, al] = (sp.eval_point(e, z + dz)["x"][:2] - sp.eval_point(e, z - dz)["x"][:2]) / 2e-7
                z = z - np.linalg.solve(J, evz["x"][:2] - xp)
            return sp.eval_point(e, z)["R"]
        x0 = ev["x"][:2]
        for i in range(2):
            def d1d2(hs):
                dx = np.zeros(2); dx[i] = hs
                Rp, Rm = R_at_x(x0 + dx), R_at_x(x0 - dx)
                return (Rp - Rm) / (2 * hs), (Rp - 2 * ev["R"] + Rm) / hs ** 2
            (a1, a2), (b1, b2) = d1d2(2e-3), d1d2(1e-3)
            fd, fd2 = (4 * b1 - a1) / 3, (4 * b2 - a2) / 3      # Richardson: O(h^4)
            np.testing.assert_allclose(ev["dR"][:, i], fd, atol=1e-8)
            np.testing.assert_allclose(ev["ddR"][:, i, i], fd2, atol=1e-5)
        assert abs(ev["R"].sum() - 1) < 1e-14
        assert np.abs(ev["dR"].sum(0)).max() < 1e-12
        assert np.abs(ev["ddR"].sum(0)).max() < 1e-10


def test_parametric_equals_greville_identity():
    """A-19: the NURBS identity map with Greville control points equals parametric mode (1e-13)."""
    w = workloads.make(1, n=6)
    a = oracle.Space.from_workload(w)
    b = oracle.Space(2, w.degree, w.knots, [0, 0], [1, 1], 1, w.quad, oracle.PARAMETRIC, None, None)
    Ka, _, Fa = a.assemble_dense(w.phys, w.params, w.a, w.b, w.U)
    Kb, _, Fb = b.assemble_dense(w.phys, w.params, w.a, w.b, w.U)
    assert np.abs(Ka - Kb).max() < 1e-13 * np.abs(Ka).max()
    assert np.abs(Fa - Fb).max() < 1e-13 * np.abs(Fa).max()
