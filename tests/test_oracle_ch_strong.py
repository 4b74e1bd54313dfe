"""Pin of the oracle's Cahn-Hilliard weak form (A-11) against the strong form the paper prints
(P:745-747): c_t - div(M_c grad(mu_c - lap c)) = 0 on the periodic domain.  M_c and mu_c are not
given by the paper (reading A-10: M = c(1-c), mu' = 3 alpha (1/(2 theta c(1-c)) - 2)), so this pins
the weak form's derivation (integration by parts, signs, the M' lap c grad N . grad c term) given
that reading: for smooth manufactured c(x, y), c_t(x, y) and test functions phi,
sum_A phi_A R_A(c_h, c_t,h) -> int phi S(c) as h -> 0."""
import numpy as np
import pytest

import oracle
import workloads

sp = pytest.importorskip("sympy")


def _interp(osp, n, funcs):
    g, _ = oracle.gauss_legendre(3)
    rows, pts = [], []
    for e0 in range(n):
        for e1 in range(n):
            for q0 in g:
                for q1 in g:
                    xi = ((e0 + (q0 + 1) / 2) / n, (e1 + (q1 + 1) / 2) / n)
                    r = osp.eval_point((e0, e1), xi)
                    row = np.zeros(osp.ndof)
                    np.add.at(row, r["node"], r["R"])
                    rows.append(row)
                    pts.append(xi)
    A, P = np.array(rows), np.array(pts)
    return [np.linalg.lstsq(A, np.broadcast_to(f(P[:, 0], P[:, 1]), len(P)), rcond=None)[0] for f in funcs]


def test_weak_form_converges_to_the_papers_strong_form():
    x, y = sp.symbols("x y", real=True)
    w0 = workloads.make(3, n=8)
    theta, alpha = w0.params[0], w0.params[1] / 1000.0        # alpha = 3: all terms of one scale
    params = [theta, alpha]
    tp = 2 * sp.pi
    c = sp.Float(0.5) + sp.Float(0.2) * sp.sin(tp * x) * sp.cos(tp * y)
    ct = sp.Float(10.0) * sp.cos(tp * (x + y))
    M = c * (1 - c)
    mup = 3 * sp.Float(alpha) * (1 / (2 * sp.Float(theta) * c * (1 - c)) - 2)
    lapc = sp.diff(c, x, 2) + sp.diff(c, y, 2)
    flux = [M * (mup * sp.diff(c, v) - sp.diff(lapc, v)) for v in (x, y)]
    S = ct - sp.diff(flux[0], x) - sp.diff(flux[1], y)
    fc, fct, fS = (sp.lambdify((x, y), e, "numpy") for e in (c, ct, S))
    phi = lambda X, Y: np.sin(2 * np.pi * X) * np.cos(2 * np.pi * Y) + 0.3 * np.cos(2 * np.pi * (X + Y))
    m = 256
    xs = (np.arange(m) + 0.5) / m
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    exact = np.mean(phi(X, Y) * fS(X, Y))
    scale = np.mean(np.abs(phi(X, Y) * fS(X, Y)))
    errs = []
    for n in (8, 16, 32):
        w = workloads.make(3, n=n)
        osp = oracle.Space.from_workload(w)
        U, V, P = _interp(osp, n, [fc, fct, phi])
        F = osp.assemble_dense(w.phys, params, 0.0, 1.0, U, V, want_K=False)[2]
        errs.append(abs(P @ F - exact))
    # measured 2.13, 0.50, 0.12 against an integral of 71.7: O(h^2) (the Delta N Delta c term of C^1
    # quadratics); a dropped or mis-signed term leaves an O(1) relative gap
    assert errs[2] < 5e-3 * scale, (errs, scale, exact)
    assert errs[1] < errs[0] / 3 and errs[2] < errs[1] / 3, errs
