"""Pins of Alg. 2 (curve unclamping for periodic mapped geometry) in the oracle:
the curve is unchanged on its domain (the defining property of unclamping -- a change of basis,
not of geometry), the knots equal Alg. 1's (whose worked examples are the paper's Fig. f:period
captions, pinned in test_oracle_basis.py), and a C^k-periodic clamped net comes out with its
last k+1 points equal to its first k+1 (the periodic identification)."""
import numpy as np
import pytest

import oracle
import workloads


def _curve(U, Pw, p, xi):
    n = Pw.shape[0] - 1
    N = np.array([oracle.coxdeboor(i, p, U, xi) for i in range(n + 1)])
    hw = N @ Pw
    return hw[:-1] / hw[-1]


@pytest.mark.parametrize("p,k", [(2, 0), (2, 1), (3, 0), (3, 1), (3, 2), (4, 3), (4, 1)])
def test_curve_unchanged(p, k):
    rng = np.random.default_rng(10 * p + k)
    nel = 7
    U = workloads.open_uniform_knots(p, nel, 0.0, 1.0)
    n = len(U) - p - 2
    P = rng.uniform(-1, 1, (n + 1, 2))
    w = rng.uniform(0.5, 1.5, n + 1)
    Pw = np.concatenate([P * w[:, None], w[:, None]], axis=1)
    U2, Pw2 = oracle.unclamp_curve(n, p, k, U, Pw)
    np.testing.assert_allclose(U2, oracle.unclamp_knots(n, p, k, U), rtol=0, atol=1e-15)
    for xi in np.linspace(0.0, 1.0, 23)[1:-1]:
        np.testing.assert_allclose(_curve(U2, Pw2, p, xi), _curve(U, Pw, p, xi), rtol=1e-12, atol=1e-12)
    # Alg. 2 moves control points iff its point loops run (k >= 1)
    assert np.allclose(Pw2, Pw) == (k == 0)


def test_c1_periodic_quadratic_wraps():
    """A clamped quadratic net with P_0 = P_n = (P_{n-1} + P_1)/2 (C^1 seam, homogeneous) comes
    out of Alg. 2 with Pw'_{n-1} = Pw'_0 and Pw'_n = Pw'_1."""
    rng = np.random.default_rng(3)
    p, nel = 2, 9
    U = workloads.open_uniform_knots(p, nel)
    n = len(U) - p - 2
    Pw = np.zeros((n + 1, 3))
    Pw[1:n] = np.concatenate([rng.uniform(-1, 1, (n - 1, 2)), rng.uniform(0.5, 1.5, (n - 1, 1))], axis=1)
    Pw[1:n, :2] *= Pw[1:n, 2:]
    Pw[0] = Pw[n] = 0.5 * (Pw[n - 1] + Pw[1])
    _, Pw2 = oracle.unclamp_curve(n, p, 1, U, Pw)
    np.testing.assert_allclose(Pw2[n - 1], Pw2[0], atol=1e-14)
    np.testing.assert_allclose(Pw2[n], Pw2[1], atol=1e-14)


def test_space_rejects_non_periodic_geometry():
    w = workloads.make(7, n=6)
    oracle.Space.from_workload(w)                 # the ring is C^1 periodic
    bad = w.ctrl.copy()
    bad[:, 0, 1] += 0.01                           # break the seam condition
    with pytest.raises(ValueError):
        oracle.Space(w.dim, w.degree, w.knots, w.periodic, w.continuity, w.dof, w.quad, w.geometry, bad, w.weights)


def test_ring_seam_is_the_clamped_endpoint():
    """The unclamped periodic map passes through the clamped net's end point P_0 (= P_n) at the
    seam xi_1 = 0 (a clamped curve interpolates its end points), and reaches it again as
    xi_1 -> 1 with a continuous Jacobian determinant (C^1 across the seam).  (eval_point takes
    parametric coordinates; the last span is approached from inside.)"""
    w = workloads.make(7, n=8)
    osp = oracle.Space.from_workload(w)
    last = osp.nel[1] - 1
    eps = 1e-9
    a = osp.eval_point((0, 0), (0.0, 0.0))
    np.testing.assert_allclose(a["x"][:2], w.ctrl[0, 0], atol=1e-13)
    b = osp.eval_point((0, last), (0.0, 1.0 - eps))
    np.testing.assert_allclose(b["x"][:2], w.ctrl[0, 0], atol=1e-7)
    for xi0 in (0.2, 0.55):
        e0 = int(xi0 * osp.nel[0])
        a = osp.eval_point((e0, 0), (xi0, eps))
        b = osp.eval_point((e0, last), (xi0, 1.0 - eps))
        np.testing.assert_allclose(a["x"], b["x"], atol=1e-7)
        assert abs(a["detJ"] - b["detJ"]) < 1e-6 * abs(a["detJ"])
