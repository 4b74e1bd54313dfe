"""Pins of the reading-dependent integrand state (VMS stabilisation, Cahn-Hilliard mobility and
chemical potential) against values computed independently of the oracle.

Sources (none of them is the oracle's code):
  * SURVEY.md Appendix A "Sanity ranges for config 5 (h = 2 pi / 128)": G = 1660.05 I,
    tau_M in [4.893e-3, 4.993e-3] for |u| <= 1, tau_C in [0.0402, 0.0410]  (reading A-14:
    tau_M = (C_t/dt^2 + u.G u + C_I nu^2 G:G)^(-1/2), tau_C = 1/(tau_M g.g));
  * SURVEY.md Appendix A (Cahn-Hilliard): over c in [0.58, 0.68], M in [0.2176, 0.2436] and
    mu' in [-5685, -4213] (reading A-10);
  * the interior diagonal of the config-3 Jacobian at the measurement
    (a, b) and c = 0.63: mass 2.40e-7, mu'-Laplacian -5.85e-4, bi-Laplacian 0.934 -- and the
    1D integrals of the uniform quadratic B-spline it lists (int N^2 = 11h/20, int N'^2 = 1/h,
    int N''^2 = 6/h^3, int N N'' = -1/h), from which the same three numbers follow in closed form.

Each check raises AssertionError.  tests/test_oracle_state_pins.py runs them on the oracle and,
in subprocesses, on deliberately mutated oracle builds, which must fail them.
"""
import math

import numpy as np

import oracle
import workloads


def _vms_space():
    w = workloads.make(5)                 # config 5, 128^3, h = 2 pi / 128
    return w, oracle.Space.from_workload(w)


def _pt(w, e, off=(0.3, 0.55, 0.8)):
    h = 2.0 * math.pi / 128
    return [(e[d] + off[d]) * h for d in range(3)]


def check_vms_tau():
    w, o = _vms_space()
    U0 = np.zeros(w.U.size)
    e = (5, 70, 127)
    # |u| = 0
    s = o.point_state(oracle.NS_VMS, w.params, U0, e, _pt(w, e))
    G = s["G"]
    assert np.all(np.abs(np.diag(G) - 1660.05) < 0.005), G
    assert np.all(G[~np.eye(3, dtype=bool)] == 0.0), G
    assert abs(s["tauM"] - 4.993e-3) < 5e-7, s["tauM"]
    assert 0.0402 <= s["tauC"] < 0.0403, s["tauC"]
    # |u| = 1 in each direction and along the diagonal (G is isotropic here)
    for d in ([1, 0, 0], [0, 1, 0], [0, 0, 1], [1 / math.sqrt(3)] * 3, [0.6, -0.8, 0.0]):
        U1 = U0.copy()
        for c in range(3):
            U1[c::4] = d[c]
        s1 = o.point_state(oracle.NS_VMS, w.params, U1, e, _pt(w, e))
        assert abs(s1["tauM"] - 4.893e-3) < 5e-7, (d, s1["tauM"])
        assert 0.0410 <= s1["tauC"] < 0.0411, (d, s1["tauC"])
    # u' = -tau_M r_M with r_M = udot at u = 0, p = 0 (A-14); p' = -tau_C r_C with r_C = 0
    Ud = np.zeros(w.U.size)
    Ud[0::4] = 1.0
    s2 = o.point_state(oracle.NS_VMS, w.params, U0, e, _pt(w, e), Udot=Ud)
    assert abs(s2["up"][0] + 4.993e-3) < 5e-7 and s2["up"][1] == 0.0 and s2["up"][2] == 0.0, s2["up"]
    # every sampled point of the actual config-5 state: |u| <= ~1.02 (Taylor-Green + 1 % noise)
    rng = np.random.default_rng(11)
    lo = (40000.0 + 1.05 ** 2 * 1660.05 + 36.0 / 1600.0 ** 2 * 3 * 1660.05 ** 2) ** -0.5
    for _ in range(12):
        e = tuple(int(x) for x in rng.integers(0, 128, 3))
        s3 = o.point_state(oracle.NS_VMS, w.params, w.U, e, _pt(w, e, tuple(rng.uniform(0, 1, 3))), Udot=w.Udot)
        assert lo <= s3["tauM"] <= 4.9928e-3, s3["tauM"]
        assert 0.0402 <= s3["tauC"] <= 0.04115, s3["tauC"]


def check_ch_state():
    w = workloads.make(3)                 # config 3, 1024^2, theta = 1.5, alpha = 3000
    o = oracle.Space.from_workload(w)
    e = (3, 1000)
    xi = [(e[0] + 0.4) / 1024, (e[1] + 0.7) / 1024]
    for c, M, mup in ((0.58, 0.2436, -5685.0), (0.68, 0.2176, -4213.0)):
        s = o.point_state(oracle.CAHN_HILLIARD, w.params, np.full(w.U.size, c), e, xi)
        assert abs(s["M"] - M) < 5e-5, (c, s["M"])
        assert abs(s["mup"] - mup) < 1.0, (c, s["mup"])
    # interior diagonal of the Jacobian at c = 0.63, split by term group (reading A-17)
    h = 1.0 / 1024
    a, b = w.a, w.b
    c0 = 0.63
    row = np.array([(512 * 1024 + 300)], np.int64)
    U = np.full(w.U.size, c0)

    def diag(a_, b_, params):
        r = o.assemble_rows(w.phys, params, a_, b_, U, row, Udot=np.zeros_like(U))
        j = int(np.nonzero(r["cols"] == row[0])[0][0])
        return r["vals"][j]

    mass = diag(a, 0.0, w.params)
    bilap = diag(0.0, b, [w.params[0], 0.0])            # alpha = 0 => mu' = 0: bi-Laplacian alone
    mulap = diag(0.0, b, w.params) - bilap
    # SURVEY App. C magnitudes (3 digits) ...
    assert abs(mass - 2.40e-7) < 0.005e-7, mass
    assert abs(mulap + 5.85e-4) < 0.005e-4, mulap
    assert abs(bilap - 0.934) < 0.0005, bilap
    # ... and their closed forms from the 1D integrals (exact under 3-point Gauss)
    M = c0 * (1 - c0)
    mup = 3 * 3000.0 * (1.0 / (2 * 1.5 * M) - 2.0)
    assert abs(mass - a * (11 * h / 20) ** 2) <= 1e-12 * mass
    assert abs(bilap - b * M * (2 * (6 / h ** 3) * (11 * h / 20) + 2 / h ** 2)) <= 1e-11 * bilap
    assert abs(mulap - b * M * mup * 2 * (1 / h) * (11 * h / 20)) <= 1e-9 * abs(mulap)


if __name__ == "__main__":
    import sys
    {"vms": check_vms_tau, "ch": check_ch_state}[sys.argv[1]]()
