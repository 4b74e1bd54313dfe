"""Pins of the generalized-alpha oracle (oracle/stepper.py) against closed forms."""
import numpy as np
import pytest

from oracle import stepper


def _linear(M, K):
    def assemble(U, Ud, a, b):
        return a * M + b * K, M @ Ud + K @ U
    return assemble


def _exact(J, R):
    return np.linalg.solve(J, R)


def test_parameters_from_rho():
    # rho = 0.5: the values the workloads use (a = 5/6, b = 4/9 dt)
    am, af, g = stepper.alpha_params(0.5)
    assert abs(am - 5 / 6) < 1e-15 and abs(af - 2 / 3) < 1e-15 and abs(af * g - 4 / 9) < 1e-15
    assert stepper.alpha_params(1.0) == (0.5, 0.5, 0.5)


def test_rho_one_is_crank_nicolson():
    rng = np.random.default_rng(0)
    n = 6
    A = rng.uniform(-1, 1, (n, n))
    M = A @ A.T + n * np.eye(n)
    B = rng.uniform(-1, 1, (n, n))
    K = B @ B.T + np.eye(n)
    U = rng.uniform(-1, 1, n)
    Ud = rng.uniform(-1, 1, n)            # need not be consistent: CN does not use it
    dt = 0.3
    U1, Ud1, _ = stepper.alpha_step(_linear(M, K), _exact, U, Ud, 1.0, dt, 1)
    ref = np.linalg.solve(M + dt / 2 * K, (M - dt / 2 * K) @ U)
    np.testing.assert_allclose(U1, ref, rtol=1e-12, atol=1e-13)
    # and the last line of (ga) holds
    np.testing.assert_allclose(U1, U + dt * (0.5 * Ud + 0.5 * Ud1), rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("rho", [0.0, 0.3, 0.5, 0.8, 1.0])
def test_spectral_radius_at_infinity(rho):
    """u' = -lam u: the one-step map of (u, u') has spectral radius -> rho_inf as lam dt -> inf."""
    lam, dt = 1.0, 1e9
    M, K = np.array([[1.0]]), np.array([[lam]])
    cols = []
    for u0, v0 in ((1.0, 0.0), (0.0, 1.0 / dt)):       # state (u, dt u')
        U1, Ud1, _ = stepper.alpha_step(_linear(M, K), _exact, np.array([u0]), np.array([v0]), rho, dt, 1)
        cols.append([U1[0], Ud1[0] * dt])           # scale u' by dt: the map is then O(1)
    A = np.array(cols).T
    assert abs(np.max(np.abs(np.linalg.eigvals(A))) - rho) < 1e-4   # rho = 0: a Jordan pair, O(sqrt(1/(lam dt)))


@pytest.mark.parametrize("rho", [0.5, 0.9])
def test_second_order(rho):
    M, K = np.array([[1.0]]), np.array([[1.0]])
    errs = []
    for dt in (0.1, 0.05, 0.025):
        U, Ud = np.array([1.0]), np.array([-1.0])
        for _ in range(int(round(1.0 / dt))):
            U, Ud, _ = stepper.alpha_step(_linear(M, K), _exact, U, Ud, rho, dt, 1)
        errs.append(abs(U[0] - np.exp(-1.0)))
    assert 3.6 < errs[0] / errs[1] < 4.4 and 3.6 < errs[1] / errs[2] < 4.4


def test_newton_on_nonlinear_problem():
    """R = Udot + U^3: Newton residual norms fall quadratically; one exact iteration solves a
    linear problem (second norm at rounding level)."""
    def assemble(U, Ud, a, b):
        return np.diag(a + 3 * b * U ** 2), Ud + U ** 3
    U = np.linspace(0.5, 1.0, 5)
    _, _, norms = stepper.alpha_step(assemble, _exact, U, -U ** 3, 0.5, 0.1, 5)
    assert norms[1] < norms[0] * 1e-1 and norms[2] < norms[1] ** 1.8 * 10 and norms[3] < 1e-12
    M, K = np.eye(3), np.diag([1.0, 2.0, 3.0])
    _, _, n2 = stepper.alpha_step(_linear(M, K), _exact, np.ones(3), np.zeros(3), 0.5, 0.1, 2)
    assert n2[1] < 1e-13 * n2[0]
