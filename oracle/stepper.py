"""CPU oracle of the generalized-alpha time step with a fixed-budget Newton loop (SURVEY §8(f)
ranks 2-3; §4 eq. (ga), and the §5 protocol).

TEST INFRASTRUCTURE ONLY: imported by tests/ (and bench.py's baseline legs), never by the product
package.  Plain numpy, fp64.

The step follows eq. (ga) in the paper's notation: given U_n, Udot_n find
Udot_{n+1} with
    R(U_{n+af}, Udot_{n+am}) = 0,
    U_{n+af}    = U_n    + af (U_{n+1}    - U_n),
    Udot_{n+am} = Udot_n + am (Udot_{n+1} - Udot_n),
    U_{n+1}     = U_n + dt ((1 - gamma) Udot_n + gamma Udot_{n+1}),
with am = (3 - rho)/(2 (1 + rho)), af = 1/(1 + rho), gamma = 1/2 + am - af.
Reading A-29 (the paper names neither the Newton unknown nor the predictor; Jansen et al. 2000,
which it cites, fixes both): Newton runs on Udot_{n+1}, so dR/dUdot_{n+1} = am dR/dUdot +
af gamma dt dR/dU -- the (a, b) of iga_form_jacobian -- and starts from the constant-U predictor
U_{n+1} = U_n, Udot_{n+1} = (gamma - 1)/gamma Udot_n (which satisfies the last line of (ga)).
The §5 protocol runs a FIXED number of Newton iterations (2) of a fixed number of GMRES
iterations (30), with no convergence test.

Pins (tests/test_oracle_stepper.py): rho = 1 is Crank-Nicolson -- the closed-form
step of a linear system M Udot + K U = 0; |amplification| -> rho as lambda dt -> infinity (the
defining property of rho); second-order convergence on udot = -lambda u; one exact
Newton iteration solves a linear problem.
"""
from __future__ import annotations

import numpy as np


def alpha_params(rho_inf):
    am = 0.5 * (3.0 - rho_inf) / (1.0 + rho_inf)
    af = 1.0 / (1.0 + rho_inf)
    gamma = 0.5 + am - af
    return am, af, gamma


def alpha_step(assemble, solve, U, Udot, rho_inf, dt, newton_its):
    """One step.  assemble(U, Udot, a, b) -> (J, R) with J = a dR/dUdot + b dR/dU;
    solve(J, R) -> x ~ J^{-1} R.  Returns (U_{n+1}, Udot_{n+1}, [||R|| at each Newton iterate])."""
    am, af, gamma = alpha_params(rho_inf)
    U = np.asarray(U, dtype=np.float64)
    Udot = np.asarray(Udot, dtype=np.float64)
    U1 = U.copy()                                   # predictor (A-29)
    Ud1 = (gamma - 1.0) / gamma * Udot
    norms = []
    for _ in range(newton_its):
        Ua = U + af * (U1 - U)
        Uda = Udot + am * (Ud1 - Udot)
        J, R = assemble(Ua, Uda, am, af * gamma * dt)
        norms.append(float(np.linalg.norm(R)))
        dx = solve(J, R)                            # J dx = R, Newton: Udot_{n+1} -= dx
        Ud1 = Ud1 - dx
        U1 = U1 - gamma * dt * dx
    return U1, Ud1, norms
