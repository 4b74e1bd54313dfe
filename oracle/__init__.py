"""ctypes front-end of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.  See oracle.c's
header for what it computes and the passages it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
# tests/test_oracle_state_pins.py points this at deliberately MUTATED oracle builds (seeded
# mutations of the readings) to show that the pins fail on them; never set otherwise.
_SO_OVERRIDE = os.environ.get("IGA_ORACLE_SO_OVERRIDE")

LAPLACE, CAHN_HILLIARD, NEOHOOKE, NS_VMS, NSK = 0, 1, 2, 3, 4
PARAMETRIC, NURBS = 0, 1


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2, no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", _SO, _SRC, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(_SO_OVERRIDE if _SO_OVERRIDE else build())
        L = _lib
        P = C.c_void_p
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        lp = C.POINTER(C.c_int64)
        L.orc_space_new.restype = P
        L.orc_space_new.argtypes = [C.c_int, ip, ip, dp, ip, ip, C.c_int, ip, C.c_int, dp, dp]
        L.orc_space_free.argtypes = [P]
        L.orc_ndof.restype = C.c_int64
        L.orc_ndof.argtypes = [P]
        L.orc_space_info.argtypes = [P, ip, ip, ip, ip]
        L.orc_space_knots.argtypes = [P, C.c_int, dp]
        L.orc_pattern_rows.restype = C.c_int64
        L.orc_pattern_rows.argtypes = [P, C.c_int64, lp, lp, C.POINTER(C.c_int32)]
        L.orc_eval_point.restype = C.c_int
        L.orc_eval_point.argtypes = [P, ip, dp, dp, dp, dp, lp, dp, dp]
        L.orc_eval_point3.restype = C.c_int
        L.orc_eval_point3.argtypes = [P, ip, dp, dp, dp, dp, dp, lp, dp, dp]
        L.orc_point_state.restype = C.c_int
        L.orc_point_state.argtypes = [P, C.c_int, dp, dp, dp, ip, dp, dp]
        L.orc_element.restype = C.c_int
        L.orc_element.argtypes = [P, C.c_int, dp, C.c_double, C.c_double, dp, dp, dp, ip, dp, dp, lp]
        L.orc_assemble_dense.restype = C.c_int
        L.orc_assemble_dense.argtypes = [P, C.c_int, dp, C.c_double, C.c_double, dp, dp, dp, dp,
                                         C.POINTER(C.c_ubyte), dp]
        L.orc_assemble_rows.restype = C.c_int64
        L.orc_assemble_rows.argtypes = [P, C.c_int, dp, C.c_double, C.c_double, dp, dp, dp, C.c_int64,
                                        lp, lp, C.POINTER(C.c_int32), dp, dp, C.POINTER(C.c_ubyte)]
        L.orc_coxdeboor.restype = C.c_double
        L.orc_coxdeboor.argtypes = [C.c_int, C.c_int, dp, C.c_double]
        L.orc_coxdeboor_deriv.restype = C.c_double
        L.orc_coxdeboor_deriv.argtypes = [C.c_int, C.c_int, dp, C.c_double, C.c_int]
        L.orc_gauss_legendre.argtypes = [C.c_int, dp, dp]
        L.orc_unclamp_knots.argtypes = [C.c_int, C.c_int, C.c_int, dp]
        L.orc_unclamp_curve.argtypes = [C.c_int, C.c_int, C.c_int, dp, dp, C.c_int, C.c_long]
        L.orc_basis_stencil.argtypes = [C.c_int, C.c_int, dp, C.c_int, ip, ip]
    return _lib


def _d(a):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _l(a):
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


# ---- primitives ---------------------------------------------------------------------------
def coxdeboor(i: int, p: int, U, xi: float, k: int = 0) -> float:
    U = _f64(U)
    return lib().orc_coxdeboor_deriv(i, p, _d(U), float(xi), k)


def gauss_legendre(n: int):
    x = np.zeros(n)
    w = np.zeros(n)
    lib().orc_gauss_legendre(n, _d(x), _d(w))
    return x, w


def unclamp_knots(n: int, p: int, k: int, U):
    U = np.array(U, dtype=np.float64)
    lib().orc_unclamp_knots(n, p, k, _d(U))
    return U


def unclamp_curve(n: int, p: int, k: int, U, Pw):
    """Alg. 2 on a copy: returns (U', Pw') for n+1 homogeneous points Pw[n+1][h]."""
    U = np.array(U, dtype=np.float64)
    Pw = np.array(Pw, dtype=np.float64)
    h = Pw.shape[1]
    lib().orc_unclamp_curve(n, p, k, _d(U), _d(Pw), h, h)
    return U, Pw


def basis_stencil(i: int, p: int, U):
    U = _f64(U)
    l = C.c_int()
    r = C.c_int()
    lib().orc_basis_stencil(i, p, _d(U), len(U), C.byref(l), C.byref(r))
    return l.value, r.value


# ---- space --------------------------------------------------------------------------------
class Space:
    """The oracle's view of an IGA space built from a workloads.Workload-like description."""

    def __init__(self, dim, degree, knots, periodic, continuity, dof, quad, geometry, ctrl, weights):
        self.dim = dim
        self.dof = dof
        p = np.array(list(degree) + [0] * (3 - dim), dtype=np.int32)
        nk = np.array([len(k) for k in knots] + [0] * (3 - dim), dtype=np.int32)
        kc = np.concatenate([np.asarray(k, dtype=np.float64) for k in knots])
        per = np.array(list(periodic) + [0] * (3 - dim), dtype=np.int32)
        cont = np.array(list(continuity) + [0] * (3 - dim), dtype=np.int32)
        qd = np.array(list(quad) + [1] * (3 - dim), dtype=np.int32)
        self._keep = (p, nk, kc, per, cont, qd)
        c = _f64(None if ctrl is None else np.asarray(ctrl).reshape(-1))
        w = _f64(None if weights is None else np.asarray(weights).reshape(-1))
        self._keep2 = (c, w)
        h = lib().orc_space_new(dim, _i(p), _i(nk), _d(kc), _i(per), _i(cont), dof, _i(qd), geometry,
                                _d(c), _d(w))
        if not h:
            raise ValueError("oracle: invalid space description")
        self.h = h
        nu = np.zeros(3, np.int32)
        nel = np.zeros(3, np.int32)
        nq = np.zeros(3, np.int32)
        nf = np.zeros(3, np.int32)
        lib().orc_space_info(h, _i(nu), _i(nel), _i(nq), _i(nf))
        self.nu, self.nel, self.nq, self.nfun = nu[:dim].tolist(), nel[:dim].tolist(), nq[:dim].tolist(), nf[:dim].tolist()
        self.ndof = int(lib().orc_ndof(h))
        self.nk = nk[:dim].tolist()

    @classmethod
    def from_workload(cls, w):
        return cls(w.dim, w.degree, w.knots, w.periodic, w.continuity, w.dof, w.quad, w.geometry,
                   w.ctrl, w.weights)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_space_free(self.h)
            self.h = None

    def knots(self, d):
        out = np.zeros(self.nk[d])
        lib().orc_space_knots(self.h, d, _d(out))
        return out

    def pattern_rows(self, rows):
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        rl = np.zeros(len(rows), np.int64)
        tot = lib().orc_pattern_rows(self.h, len(rows), _l(rows), _l(rl), None)
        cols = np.zeros(tot, np.int32)
        lib().orc_pattern_rows(self.h, len(rows), _l(rows), _l(rl), cols.ctypes.data_as(C.POINTER(C.c_int32)))
        rp = np.zeros(len(rows) + 1, np.int64)
        rp[1:] = np.cumsum(rl)
        return rp, cols

    def pattern(self):
        return self.pattern_rows(np.arange(self.ndof, dtype=np.int64))

    def eval_point(self, e, xi):
        nen_max = 125
        R = np.zeros(nen_max)
        dR = np.zeros(nen_max * 3)
        ddR = np.zeros(nen_max * 9)
        node = np.zeros(nen_max, np.int64)
        x = np.zeros(3)
        det = C.c_double()
        ee = np.array(list(e) + [0] * (3 - len(e)), np.int32)
        xx = np.array(list(xi) + [0.0] * (3 - len(xi)), np.float64)
        n = lib().orc_eval_point(self.h, _i(ee), _d(xx), _d(R), _d(dR), _d(ddR), _l(node), _d(x), C.byref(det))
        if n < 0:
            raise ValueError("oracle: detJ <= 0")
        return dict(R=R[:n], dR=dR[:3 * n].reshape(n, 3), ddR=ddR[:9 * n].reshape(n, 3, 3), node=node[:n],
                    x=x, detJ=det.value)

    def eval_point3(self, e, xi):
        """All spatial derivatives of R_A up to third order (orc_eval_point3)."""
        nen_max = 125
        R = np.zeros(nen_max)
        d1 = np.zeros(nen_max * 3)
        d2 = np.zeros(nen_max * 9)
        d3 = np.zeros(nen_max * 27)
        node = np.zeros(nen_max, np.int64)
        x = np.zeros(3)
        det = C.c_double()
        ee = np.array(list(e) + [0] * (3 - len(e)), np.int32)
        xx = np.array(list(xi) + [0.0] * (3 - len(xi)), np.float64)
        n = lib().orc_eval_point3(self.h, _i(ee), _d(xx), _d(R), _d(d1), _d(d2), _d(d3), _l(node), _d(x), C.byref(det))
        if n < 0:
            raise ValueError("oracle: detJ <= 0")
        return dict(R=R[:n], dR=d1[:3 * n].reshape(n, 3), ddR=d2[:9 * n].reshape(n, 3, 3),
                    dddR=d3[:27 * n].reshape(n, 3, 3, 3), node=node[:n], x=x, detJ=det.value)

    def point_state(self, kind, params, U, e, xi, Udot=None):
        """Integrand point state at parametric point xi of element e (orc_point_state): VMS ->
        dict(tauM, tauC, G, gg, up, pp); Cahn-Hilliard -> dict(M, Mp, Mpp, mup, mupp)."""
        prm = np.zeros(8)
        prm[:len(params)] = params
        U = _f64(U)
        Udot = _f64(Udot) if Udot is not None else np.zeros_like(U)
        out = np.zeros(16)
        ee = np.array(list(e) + [0] * (3 - len(e)), np.int32)
        xx = np.array(list(xi) + [0.0] * (3 - len(xi)), np.float64)
        n = lib().orc_point_state(self.h, kind, _d(prm), _d(U), _d(Udot), _i(ee), _d(xx), _d(out))
        if n < 0:
            raise ValueError(f"oracle point state failed ({n})")
        if kind == NS_VMS:
            return dict(tauM=out[0], tauC=out[1], G=out[2:11].reshape(3, 3), gg=out[11], up=out[12:15], pp=out[15])
        return dict(M=out[0], Mp=out[1], Mpp=out[2], mup=out[3], mupp=out[4])

    def element(self, kind, params, a, b, U, Udot=None, e=(0, 0, 0), Utau=None, want_K=True):
        prm = np.zeros(8)
        prm[:len(params)] = params
        U = _f64(U)
        Udot = _f64(Udot) if Udot is not None else np.zeros_like(U)
        Utau = _f64(Utau)
        nmax = 125 * 4
        Ke = np.zeros(nmax * nmax) if want_K else None
        Fe = np.zeros(nmax)
        nodes = np.zeros(125, np.int64)
        ee = np.array(list(e) + [0] * (3 - len(e)), np.int32)
        n = lib().orc_element(self.h, kind, _d(prm), a, b, _d(U), _d(Udot), _d(Utau), _i(ee), _d(Ke), _d(Fe),
                              _l(nodes))
        if n < 0:
            raise ValueError(f"oracle element failed ({n})")
        m = self.dof
        k = n * m
        return (Ke[:k * k].reshape(k, k) if want_K else None), Fe[:k], nodes[:n]

    def assemble_dense(self, kind, params, a, b, U, Udot=None, Utau=None, want_K=True, want_F=True):
        prm = np.zeros(8)
        prm[:len(params)] = params
        U = _f64(U)
        Udot = _f64(Udot) if Udot is not None else np.zeros_like(U)
        Utau = _f64(Utau)
        nd = self.ndof
        K = np.zeros((nd, nd)) if want_K else None
        T = np.zeros((nd, nd), np.uint8) if want_K else None
        F = np.zeros(nd) if want_F else None
        rc = lib().orc_assemble_dense(self.h, kind, _d(prm), a, b, _d(U), _d(Udot), _d(Utau), _d(K),
                                      None if T is None else T.ctypes.data_as(C.POINTER(C.c_ubyte)), _d(F))
        if rc < 0:
            raise ValueError(f"oracle dense assembly failed ({rc})")
        return K, T, F

    def assemble_rows(self, kind, params, a, b, U, rows, Udot=None, Utau=None, want_K=True, want_F=True):
        """Complete rows (CSR over the Alg. 3 pattern) for a sorted row subset."""
        prm = np.zeros(8)
        prm[:len(params)] = params
        U = _f64(U)
        Udot = _f64(Udot) if Udot is not None else np.zeros_like(U)
        Utau = _f64(Utau)
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        rp, cols = self.pattern_rows(rows)
        vals = np.zeros(len(cols)) if want_K else None
        touched = np.zeros(len(cols), np.uint8) if want_K else None
        F = np.zeros(len(rows)) if want_F else None
        nv = lib().orc_assemble_rows(self.h, kind, _d(prm), a, b, _d(U), _d(Udot), _d(Utau), len(rows),
                                     _l(rows), _l(rp), cols.ctypes.data_as(C.POINTER(C.c_int32)), _d(vals), _d(F),
                                     None if touched is None else touched.ctypes.data_as(C.POINTER(C.c_ubyte)))
        if nv < 0:
            raise ValueError(f"oracle row assembly failed ({nv})")
        return dict(rowptr=rp, cols=cols, vals=vals, F=F, touched=touched, nvisited=int(nv))


def dense_to_csr(K, T):
    """Compress the touched entries of a dense matrix (ascending columns) -> (rowptr, cols, vals)."""
    nd = K.shape[0]
    rp = np.zeros(nd + 1, np.int64)
    cols = []
    vals = []
    for r in range(nd):
        c = np.nonzero(T[r])[0]
        cols.append(c)
        vals.append(K[r, c])
        rp[r + 1] = rp[r] + len(c)
    return rp, np.concatenate(cols).astype(np.int32), np.concatenate(vals)
