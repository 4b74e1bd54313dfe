"""Consistency pin of the oracle's RBVMS Navier-Stokes residual (config 5, reading
A-14).  The stabilisation (tau, the fine-scale model) is a reading the paper does not print, but a
VMS residual must vanish on an exact solution of the incompressible Navier-Stokes equations: the
Galerkin terms integrate to zero and every fine-scale term is proportional to the strong residual.
The Arnold-Beltrami-Childress flow u = (A sin z + C cos y, B sin x + A cos z, C sin y + B cos x) on
[0, 2 pi]^3 is one (curl u = u, lap u = -u): with u_t = -nu u and p = -|u|^2 / 2 all NS residuals
vanish.  Interpolated into the C^1 quadratic space, the assembled residual must shrink with h
relative to the size of its individual terms (a wrong sign or a dropped convective, pressure,
viscous or continuity term leaves an O(1) remainder)."""
import math

import numpy as np

import oracle
import workloads

A_, B_, C_ = 1.0, 0.7, 0.4


def _abc(x, y, z):
    u = A_ * np.sin(z) + C_ * np.cos(y)
    v = B_ * np.sin(x) + A_ * np.cos(z)
    w = C_ * np.sin(y) + B_ * np.cos(x)
    return u, v, w, -(u * u + v * v + w * w) / 2


def _interp_matrix(osp, d, n, L):
    """1D collocation matrix of the unique periodic functions at the element midpoints."""
    U = osp.knots(d)
    p = 2
    nopen = len(U) - p - 1
    nu = osp.nu[d]
    pts = (np.arange(n) + 0.5) / n * L
    Cm = np.zeros((n, nu))
    for k, xk in enumerate(pts):
        for i in range(nopen):
            Cm[k, i % nu] += oracle.coxdeboor(i, p, U, xk)
    return pts, np.linalg.inv(Cm)


def _residual(n, fields_fn, nu):
    w = workloads.make(5, n=n)
    osp = oracle.Space.from_workload(w)
    L = 2 * math.pi
    pts, Ci = _interp_matrix(osp, 0, n, L)
    X, Y, Z = np.meshgrid(pts, pts, pts, indexing="ij")
    vals = fields_fn(X, Y, Z)
    coef = [np.einsum("ai,bj,ck,ijk->abc", Ci, Ci, Ci, f) for f in vals]
    U = np.stack(coef, axis=-1).reshape(-1)
    Ud = np.zeros_like(U).reshape(-1, 4)
    Ud[:, :3] = -nu * U.reshape(-1, 4)[:, :3]
    rows = np.arange(osp.ndof, dtype=np.int64)
    return osp.assemble_rows(w.phys, w.params, w.a, w.b, U, rows, Udot=Ud.reshape(-1), want_K=False)["F"], w


def test_vms_residual_vanishes_on_an_exact_navier_stokes_solution():
    nu = workloads.make(5, n=4).params[0]
    rel = []
    for n in (6, 12, 24):
        F, w = _residual(n, _abc, nu)
        # scale: the residual of the same fields with the pressure sign flipped (pressure term x 2)
        Fp, _ = _residual(n, lambda x, y, z: (*_abc(x, y, z)[:3], -_abc(x, y, z)[3]), nu)
        rel.append(np.linalg.norm(F) / np.linalg.norm(Fp))
    # measured 1.8e-5, 7.7e-7, 4.4e-8; the viscous and time terms (nu = 1/1600) alone are ~6e-4 of
    # the scale, so a wrong sign in any term is far above the remainder
    assert rel[2] < 1e-6, rel
    assert rel[1] < rel[0] / 8 and rel[2] < rel[1] / 8, rel
