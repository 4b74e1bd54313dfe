"""paper_1305_4452_b200 -- thin Python binding of libiga (include/iga.h).

Argument marshalling only: every step of the assembly runs in libiga's CUDA kernels for
sm_100a.  torch provides device memory and streams.  There is no CPU fallback: if libiga.so
is missing or no CUDA device is present, the calls raise.

    sp = Space(dim, degree, knots, periodic, continuity, dof, quad, geometry, ctrl, weights)
    row_ptr, col_idx = sp.csr_pattern()
    F = sp.form_residual(phys, U, Udot)
    vals, F = sp.form_jacobian(phys, a, b, U, Udot, want_F=True)
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# IGA_LIB: an alternative build of the same library (A/B experiments); default the in-tree one
LIB_PATH = os.environ.get("IGA_LIB", os.path.join(_HERE, "libiga.so"))

PHYS_LAPLACE, PHYS_CAHN_HILLIARD, PHYS_NEOHOOKE, PHYS_NS_VMS = 0, 1, 2, 3
GEOM_PARAMETRIC, GEOM_NURBS = 0, 1
_STATUS = ["OK", "ERR_PARAM", "ERR_DOMAIN", "ERR_SINGULAR_MAP", "ERR_PATTERN", "ERR_NONFINITE",
           "ERR_CUDA", "ERR_COMM", "ERR_NOMEM", "ERR_STATE"]


class IgaError(RuntimeError):
    def __init__(self, code, msg):
        self.code = code
        super().__init__(f"libiga {_STATUS[code] if 0 <= code < len(_STATUS) else code}: {msg}")


class _Desc(C.Structure):
    _fields_ = [("dim", C.c_int), ("degree", C.c_int * 3), ("n_knots", C.c_int * 3),
                ("knots", C.POINTER(C.c_double) * 3), ("periodic", C.c_int * 3),
                ("periodic_continuity", C.c_int * 3), ("dof", C.c_int), ("quad", C.c_int * 3),
                ("geometry", C.c_int), ("ctrl", C.POINTER(C.c_double)), ("weights", C.POINTER(C.c_double))]


class _Dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("procs", C.c_int * 3), ("transport", C.c_int),
                ("nccl_id", C.c_ubyte * 128)]


class _Msg(C.Structure):
    _fields_ = [("peer", C.c_int), ("subbox", C.c_int), ("rows", C.c_int64), ("values", C.c_int64),
                ("box_lo", C.c_int * 3), ("box_n", C.c_int * 3)]


XPORT_NCCL, XPORT_LOCAL = 0, 1


class _Krylov(C.Structure):
    _fields_ = [("restart", C.c_int), ("maxit", C.c_int), ("rtol", C.c_double), ("precond", C.c_int),
                ("block_rows", C.c_int)]


PC_NONE, PC_JACOBI, PC_BJACOBI_ILU0 = 0, 1, 2


class _Alpha(C.Structure):
    _fields_ = [("rho_inf", C.c_double), ("dt", C.c_double), ("newton_its", C.c_int), ("krylov", _Krylov)]


class _StepStats(C.Structure):
    _fields_ = [("res_norm", C.c_double * 8), ("gmres_its", C.c_int * 8), ("gmres_relres", C.c_double * 8)]


class _Phys(C.Structure):
    _fields_ = [("kind", C.c_int), ("p", C.c_double * 8)]


_lib = None

EXPORTS = ["iga_space_create", "iga_space_destroy", "iga_space_info", "iga_csr_pattern", "iga_form_residual",
           "iga_form_jacobian", "iga_form_jacobian_host", "iga_space_check", "iga_last_launch_count",
           "iga_last_error", "iga_version", "iga_profile_enable", "iga_profile_reset", "iga_profile_read",
           "iga_microbench", "iga_space_set_option", "iga_form_jacobian_group", "iga_form_residual_group",
           "iga_dist_plan", "iga_nccl_unique_id", "iga_basis_eval", "iga_gmres", "iga_alpha_step", "iga_gmres_group", "iga_alpha_step_group",
           "iga_krylov_plan"]


def lib():
    """Load libiga.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1305_4452_b200.build` "
                              "(libiga has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        dp = C.POINTER(C.c_double)
        lp = C.POINTER(C.c_int64)
        L.iga_space_create.argtypes = [C.POINTER(_Desc), C.POINTER(_Dist), C.c_int, C.POINTER(vp)]
        L.iga_space_destroy.argtypes = [vp]
        L.iga_space_info.argtypes = [vp, lp, lp, lp, lp, lp, lp, lp, lp]
        L.iga_csr_pattern.argtypes = [vp, vp, vp, vp]
        L.iga_form_residual.argtypes = [vp, C.POINTER(_Phys), vp, vp, vp, vp]
        L.iga_form_jacobian.argtypes = [vp, C.POINTER(_Phys), C.c_double, C.c_double, vp, vp, vp, vp, vp]
        L.iga_form_jacobian_host.argtypes = [vp, C.POINTER(_Phys), C.c_double, C.c_double, vp, vp, vp, vp, vp]
        L.iga_space_check.argtypes = [vp, vp]
        L.iga_last_launch_count.argtypes = [vp]
        L.iga_last_launch_count.restype = C.c_int
        L.iga_profile_enable.argtypes = [vp, C.c_int]
        L.iga_profile_reset.argtypes = [vp]
        L.iga_profile_read.argtypes = [vp, C.c_int, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double)]
        L.iga_profile_read.restype = C.c_int
        L.iga_space_set_option.argtypes = [vp, C.c_char_p, C.c_longlong]
        L.iga_space_set_option.restype = C.c_int
        L.iga_microbench.argtypes = [C.c_int, C.c_int, C.c_longlong]
        L.iga_microbench.restype = C.c_double
        L.iga_form_jacobian_group.argtypes = [C.c_int, C.POINTER(vp), C.POINTER(_Phys), C.c_double, C.c_double,
                                              C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), vp]
        L.iga_form_residual_group.argtypes = [C.c_int, C.POINTER(vp), C.POINTER(_Phys), C.POINTER(vp), C.POINTER(vp),
                                              C.POINTER(vp), vp]
        L.iga_dist_plan.argtypes = [C.POINTER(_Desc), C.POINTER(_Dist), lp, lp, lp, lp, lp, C.c_int,
                                    C.POINTER(_Msg), C.POINTER(C.c_int), C.POINTER(_Msg), C.POINTER(C.c_int)]
        L.iga_nccl_unique_id.argtypes = [C.POINTER(C.c_ubyte * 128)]
        L.iga_basis_eval.argtypes = [vp, C.c_int, vp, vp]
        L.iga_gmres.argtypes = [vp, vp, vp, vp, vp, vp, C.POINTER(_Krylov), C.POINTER(C.c_int), dp, vp]
        L.iga_gmres_group.argtypes = [C.c_int, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                      C.POINTER(vp), C.POINTER(_Krylov), C.POINTER(C.c_int), dp, vp]
        L.iga_krylov_plan.argtypes = [C.POINTER(_Desc), C.POINTER(_Dist), lp, lp, lp, lp, C.c_int,
                                      C.POINTER(_Msg), C.POINTER(C.c_int), C.POINTER(_Msg), C.POINTER(C.c_int)]
        L.iga_alpha_step_group.argtypes = [C.c_int, C.POINTER(vp), C.POINTER(_Phys), C.POINTER(_Alpha), C.POINTER(vp),
                                           C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                                           C.POINTER(_StepStats), vp]
        L.iga_alpha_step.argtypes = [vp, C.POINTER(_Phys), C.POINTER(_Alpha), vp, vp, vp, vp, vp, C.POINTER(_StepStats), vp]
        L.iga_last_error.restype = C.c_char_p
        L.iga_version.restype = C.c_char_p
        for f in ("iga_space_create", "iga_space_destroy", "iga_space_info", "iga_csr_pattern", "iga_form_residual",
                  "iga_form_jacobian", "iga_form_jacobian_host", "iga_space_check", "iga_profile_enable",
                  "iga_profile_reset", "iga_form_jacobian_group", "iga_form_residual_group", "iga_dist_plan",
                  "iga_nccl_unique_id", "iga_basis_eval", "iga_gmres", "iga_alpha_step", "iga_gmres_group", "iga_alpha_step_group",
                  "iga_krylov_plan"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(code):
    if code != 0:
        raise IgaError(code, lib().iga_last_error().decode())


def _ptr(t):
    """Raw data pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t.ctypes.data)


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def make_phys(kind: int, params) -> _Phys:
    ph = _Phys()
    ph.kind = kind
    for i, v in enumerate(params):
        ph.p[i] = float(v)
    return ph


MICROBENCH = {0: "dfma_flops", 1: "dmma_flops", 2: "dfma_dmma_mixed_flops", 3: "red_f64_warp_contig_per_s",
              4: "red_f64_sector_per_s", 5: "red_f64_scattered_per_s", 6: "store_bytes_per_s",
              7: "smem_atomic_f64_per_s", 8: "bulkred_96B_ops_per_s", 9: "red_f64_c5pattern_per_s",
              10: "bulkred_384B_ops_per_s", 11: "lds128_bcast_warp_loads_per_s", 12: "ldg128_bcast_warp_loads_per_s"}


def microbench(device: int = 0, which=None, param: int = 0) -> dict:
    """K8 ceilings measured on `device` (see iga.h)."""
    out = {}
    for k in (MICROBENCH if which is None else [which]):
        out[MICROBENCH[k]] = float(lib().iga_microbench(device, k, param))
    return out


def _make_desc(dim, degree, knots, periodic, continuity, dof, quad, geometry, ctrl=None, weights=None):
    """iga_space_desc from host arrays; returns (desc, keep-alive list)."""
    d = _Desc()
    d.dim = dim
    keep = []
    for a in range(3):
        if a < dim:
            k = np.ascontiguousarray(knots[a], dtype=np.float64)
            keep.append(k)
            d.degree[a] = int(degree[a])
            d.n_knots[a] = len(k)
            d.knots[a] = k.ctypes.data_as(C.POINTER(C.c_double))
            d.periodic[a] = int(periodic[a])
            d.periodic_continuity[a] = int(continuity[a])
            d.quad[a] = int(quad[a]) if quad is not None else 0
    d.dof = dof
    d.geometry = geometry
    if ctrl is not None:
        c = np.ascontiguousarray(ctrl, dtype=np.float64).reshape(-1)
        keep.append(c)
        d.ctrl = c.ctypes.data_as(C.POINTER(C.c_double))
    if weights is not None:
        w = np.ascontiguousarray(weights, dtype=np.float64).reshape(-1)
        keep.append(w)
        d.weights = w.ctypes.data_as(C.POINTER(C.c_double))
    return d, keep


def _make_dist(dist) -> _Dist:
    """dist = {"rank", "nranks", "procs", ["transport"], ["nccl_id": 128 bytes]}"""
    dd = _Dist()
    dd.rank, dd.nranks = int(dist["rank"]), int(dist["nranks"])
    for a in range(3):
        dd.procs[a] = int(dist["procs"][a]) if a < len(dist["procs"]) else 1
    dd.transport = int(dist.get("transport", XPORT_NCCL))
    uid = dist.get("nccl_id")
    if uid is not None:
        for i, b in enumerate(bytes(uid)[:128]):
            dd.nccl_id[i] = b
    return dd


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId for an IGA_XPORT_NCCL decomposition (broadcast it to every rank)."""
    buf = (C.c_ubyte * 128)()
    _check(lib().iga_nccl_unique_id(C.byref(buf)))
    return bytes(buf)


def dist_plan(w, dist) -> dict:
    """Host-only box decomposition + exchange plan of rank dist["rank"] for workload `w` (no GPU)."""
    d, keep = _make_desc(w.dim, w.degree, w.knots, w.periodic, w.continuity, w.dof, w.quad, w.geometry, w.ctrl,
                         w.weights)
    dd = _make_dist(dist)
    arrs = [(C.c_int64 * 3)() for _ in range(5)]
    snd, rcv = (_Msg * 8)(), (_Msg * 8)()
    ns, nr = C.c_int(), C.c_int()
    _check(lib().iga_dist_plan(C.byref(d), C.byref(dd), *arrs, 8, snd, C.byref(ns), rcv, C.byref(nr)))

    def msgs(a, n):
        return [{"peer": a[k].peer, "subbox": a[k].subbox, "rows": a[k].rows, "values": a[k].values,
                 "box_lo": list(a[k].box_lo), "box_n": list(a[k].box_n)} for k in range(n)]
    own_lo, own_hi, el_lo, el_hi, ext_n = [list(x) for x in arrs]
    return {"own_lo": own_lo, "own_hi": own_hi, "el_lo": el_lo, "el_hi": el_hi, "ext_n": ext_n,
            "send": msgs(snd, ns.value), "recv": msgs(rcv, nr.value)}


def krylov_plan(w, dist) -> dict:
    """Host-only ghost-exchange plan of the distributed GMRES for rank dist["rank"] (no GPU)."""
    d, keep = _make_desc(w.dim, w.degree, w.knots, w.periodic, w.continuity, w.dof, w.quad, w.geometry, w.ctrl,
                         w.weights)
    dd = _make_dist(dist)
    arrs = [(C.c_int64 * 3)() for _ in range(4)]
    snd, rcv = (_Msg * 32)(), (_Msg * 32)()
    ns, nr = C.c_int(), C.c_int()
    _check(lib().iga_krylov_plan(C.byref(d), C.byref(dd), *arrs, 32, snd, C.byref(ns), rcv, C.byref(nr)))

    def msgs(a, n):
        out = []
        for k in range(n):
            sb = a[k].subbox
            out.append({"peer": a[k].peer, "offset": [sb // 9 - 1, (sb // 3) % 3 - 1, sb % 3 - 1], "rows": a[k].rows,
                        "box_lo": list(a[k].box_lo), "box_n": list(a[k].box_n)})
        return out
    own_lo, own_hi, ext_n, ghost = [list(x) for x in arrs]
    return {"own_lo": own_lo, "own_hi": own_hi, "ext_n": ext_n, "ghost": ghost,
            "send": msgs(snd, ns.value), "recv": msgs(rcv, nr.value)}


def _pp(ts):
    return (C.c_void_p * len(ts))(*[(t.data_ptr() if t is not None else None) for t in ts])


def form_jacobian_group(spaces, phys, a, b, Us, Udots=None, vals=None, Fs=None, want_F=False, stream=None):
    """In-process multi-rank Jacobian (IGA_XPORT_LOCAL): spaces[k] = rank k; returns (vals, Fs)."""
    import torch
    n = len(spaces)
    if vals is None:
        vals = [torch.empty(sp.nnz, dtype=torch.float64, device=Us[k].device) for k, sp in enumerate(spaces)]
    if want_F and Fs is None:
        Fs = [torch.empty(sp.nrows, dtype=torch.float64, device=Us[k].device) for k, sp in enumerate(spaces)]
    hs = (C.c_void_p * n)(*[sp.h.value for sp in spaces])
    _check(lib().iga_form_jacobian_group(n, hs, C.byref(phys), float(a), float(b), _pp(Us),
                                         _pp(Udots) if Udots is not None else None, _pp(vals),
                                         _pp(Fs) if Fs is not None else None, _stream(stream)))
    return vals, Fs


def gmres_group(spaces, row_ptrs, col_idxs, vals, bs, xs=None, restart=30, maxit=30, precond=PC_BJACOBI_ILU0,
                block_rows=32, stream=None):
    """Distributed fixed-budget GMRES of in-process ranks (iga_gmres_group); returns (xs, iters, relres)."""
    import torch
    n = len(spaces)
    if xs is None:
        xs = [torch.zeros_like(bb) for bb in bs]
    arr = lambda ts: (C.c_void_p * n)(*[t.data_ptr() for t in ts])
    hs = (C.c_void_p * n)(*[sp.h.value for sp in spaces])
    opt = _Krylov(int(restart), int(maxit), 0.0, int(precond), int(block_rows))
    it = C.c_int(0)
    rr = C.c_double(0.0)
    _check(lib().iga_gmres_group(n, hs, arr(row_ptrs), arr(col_idxs), arr(vals), arr(bs), arr(xs), C.byref(opt),
                                 C.byref(it), C.byref(rr), _stream(stream)))
    return xs, int(it.value), float(rr.value)


def alpha_step_group(spaces, phys, Us, Udots, row_ptrs, col_idxs, vals, rho_inf, dt, newton_its=2, restart=30,
                     maxit=30, precond=PC_BJACOBI_ILU0, block_rows=32, stream=None):
    """One generalized-alpha step of in-process ranks (iga_alpha_step_group); Us / Udots advance in place."""
    n = len(spaces)
    arr = lambda ts: (C.c_void_p * n)(*[t.data_ptr() for t in ts])
    hs = (C.c_void_p * n)(*[sp.h.value for sp in spaces])
    opt = _Alpha(float(rho_inf), float(dt), int(newton_its),
                 _Krylov(int(restart), int(maxit), 0.0, int(precond), int(block_rows)))
    stt = _StepStats()
    _check(lib().iga_alpha_step_group(n, hs, C.byref(phys), C.byref(opt), arr(row_ptrs), arr(col_idxs), arr(vals),
                                      arr(Us), arr(Udots), C.byref(stt), _stream(stream)))
    k = int(newton_its)
    return {"res_norm": list(stt.res_norm[:k]), "gmres_its": list(stt.gmres_its[:k]),
            "gmres_relres": list(stt.gmres_relres[:k])}


def form_residual_group(spaces, phys, Us, Udots=None, Fs=None, stream=None):
    import torch
    n = len(spaces)
    if Fs is None:
        Fs = [torch.empty(sp.nrows, dtype=torch.float64, device=Us[k].device) for k, sp in enumerate(spaces)]
    hs = (C.c_void_p * n)(*[sp.h.value for sp in spaces])
    _check(lib().iga_form_residual_group(n, hs, C.byref(phys), _pp(Us), _pp(Udots) if Udots is not None else None,
                                         _pp(Fs), _stream(stream)))
    return Fs


class Space:
    """An IGA space on one CUDA device (iga_space_create).  Inputs are host arrays."""

    def __init__(self, dim, degree, knots, periodic, continuity, dof, quad, geometry, ctrl=None, weights=None,
                 device: int = 0, dist=None):
        L = lib()
        d, self._keep = _make_desc(dim, degree, knots, periodic, continuity, dof, quad, geometry, ctrl, weights)
        dd = _make_dist(dist) if dist is not None else None
        h = C.c_void_p()
        _check(L.iga_space_create(C.byref(d), C.byref(dd) if dd is not None else None, device, C.byref(h)))
        self.h = h
        self.dim, self.dof, self.device = dim, dof, device
        self.degree = [int(degree[a]) for a in range(dim)]
        self.quad = [int(quad[a]) if quad is not None and quad[a] else int(degree[a]) + 1 for a in range(dim)]
        v = [C.c_int64() for _ in range(4)]
        lo, hi, elo, ehi = [(C.c_int64 * 3)() for _ in range(4)]
        _check(L.iga_space_info(h, *[C.byref(x) for x in v], lo, hi, elo, ehi))
        self.ndof, self.nrows, self.nnz, self.nqp = [x.value for x in v]
        self.owned_lo, self.owned_hi = list(lo), list(hi)
        self.elem_lo, self.elem_hi = list(elo), list(ehi)

    @classmethod
    def from_workload(cls, w, device: int = 0, dist=None):
        return cls(w.dim, w.degree, w.knots, w.periodic, w.continuity, w.dof, w.quad, w.geometry, w.ctrl,
                   w.weights, device=device, dist=dist)

    def close(self):
        if getattr(self, "h", None):
            lib().iga_space_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- calls -------------------------------------------------------------------------------
    def csr_pattern(self, row_ptr=None, col_idx=None, stream=None):
        import torch
        dev = torch.device("cuda", self.device)
        if row_ptr is None:
            row_ptr = torch.empty(self.nrows + 1, dtype=torch.int64, device=dev)
        if col_idx is None:
            col_idx = torch.empty(self.nnz, dtype=torch.int32, device=dev)
        _check(lib().iga_csr_pattern(self.h, _ptr(row_ptr), _ptr(col_idx), _stream(stream)))
        return row_ptr, col_idx

    def form_residual(self, phys, U, Udot=None, F=None, stream=None):
        import torch
        if F is None:
            F = torch.empty(self.nrows, dtype=torch.float64, device=U.device)
        _check(lib().iga_form_residual(self.h, C.byref(phys), _ptr(U), _ptr(Udot), _ptr(F), _stream(stream)))
        return F

    def form_jacobian(self, phys, a, b, U, Udot=None, vals=None, F=None, want_F=False, stream=None):
        import torch
        if vals is None:
            vals = torch.empty(self.nnz, dtype=torch.float64, device=U.device)
        if want_F and F is None:
            F = torch.empty(self.nrows, dtype=torch.float64, device=U.device)
        _check(lib().iga_form_jacobian(self.h, C.byref(phys), float(a), float(b), _ptr(U), _ptr(Udot), _ptr(vals),
                                       _ptr(F), _stream(stream)))
        return vals, F

    def form_jacobian_host(self, phys, a, b, U_host, Udot_host, vals_host, F_host=None, stream=None):
        _check(lib().iga_form_jacobian_host(self.h, C.byref(phys), float(a), float(b), _ptr(U_host),
                                            _ptr(Udot_host), _ptr(vals_host), _ptr(F_host), _stream(stream)))
        return vals_host, F_host

    def basis_eval(self, order=3, out=None, stream=None):
        """Spatial derivatives of every local basis function up to `order` at every Gauss point
        (iga_basis_eval); returns a tensor [nelem_local, nen, ncomp, nq]."""
        import torch
        nen = int(np.prod([p + 1 for p in self.degree]))
        nq = int(np.prod(self.quad))
        ncomp = sum(self.dim ** k for k in range(order + 1))
        nel = int(np.prod([self.elem_hi[a] - self.elem_lo[a] for a in range(self.dim)]))
        if out is None:
            out = torch.empty((nel, nen, ncomp, nq), dtype=torch.float64, device=torch.device("cuda", self.device))
        _check(lib().iga_basis_eval(self.h, int(order), _ptr(out), _stream(stream)))
        return out

    def gmres(self, row_ptr, col_idx, val, b, x=None, restart=30, maxit=30, rtol=1e-8, precond=PC_BJACOBI_ILU0,
              block_rows=32, stream=None):
        """Solve J x = b with this space's assembled CSR (iga_gmres: right-preconditioned GMRES,
        block-Jacobi ILU(0)); x (device fp64) is the initial guess (zeros if None) and is
        overwritten.  Returns (x, iterations, true relative residual)."""
        import torch
        if x is None:
            x = torch.zeros_like(b)
        opt = _Krylov(int(restart), int(maxit), float(rtol), int(precond), int(block_rows))
        it = C.c_int(0)
        rr = C.c_double(0.0)
        _check(lib().iga_gmres(self.h, _ptr(row_ptr), _ptr(col_idx), _ptr(val), _ptr(b), _ptr(x), C.byref(opt),
                               C.byref(it), C.byref(rr), _stream(stream)))
        return x, int(it.value), float(rr.value)

    def alpha_step(self, phys, U, Udot, row_ptr, col_idx, val, rho_inf, dt, newton_its=2, restart=30, maxit=30,
                   rtol=0.0, precond=PC_BJACOBI_ILU0, block_rows=32, stream=None):
        """One generalized-alpha step with the fixed Newton / GMRES budget (iga_alpha_step); U and
        Udot (device fp64) advance in place from step n to n+1; val is the Jacobian buffer.
        Returns {"res_norm": [...], "gmres_its": [...], "gmres_relres": [...]} per Newton iterate."""
        opt = _Alpha(float(rho_inf), float(dt), int(newton_its),
                     _Krylov(int(restart), int(maxit), float(rtol), int(precond), int(block_rows)))
        stt = _StepStats()
        _check(lib().iga_alpha_step(self.h, C.byref(phys), C.byref(opt), _ptr(row_ptr), _ptr(col_idx), _ptr(val),
                                    _ptr(U), _ptr(Udot), C.byref(stt), _stream(stream)))
        k = int(newton_its)
        return {"res_norm": list(stt.res_norm[:k]), "gmres_its": list(stt.gmres_its[:k]),
                "gmres_relres": list(stt.gmres_relres[:k])}

    def check(self, stream=None):
        _check(lib().iga_space_check(self.h, _stream(stream)))

    def last_launch_count(self) -> int:
        return int(lib().iga_last_launch_count(self.h))

    def set_option(self, key: str, value: int):
        _check(lib().iga_space_set_option(self.h, key.encode(), int(value)))

    def profile(self, on: bool = True):
        _check(lib().iga_profile_enable(self.h, int(on)))

    def profile_reset(self):
        _check(lib().iga_profile_reset(self.h))

    def profile_read(self) -> dict:
        """{kernel name: (launches, total ms)} since the last reset (synchronises)."""
        mx = 32
        names = C.create_string_buffer(32 * mx)
        cnt = (C.c_int * mx)()
        ms = (C.c_double * mx)()
        n = lib().iga_profile_read(self.h, mx, names, cnt, ms)
        if n < 0:
            raise IgaError(1, lib().iga_last_error().decode())
        out = {}
        for k in range(min(n, mx)):
            nm = names.raw[32 * k:32 * k + 32].split(b"\0", 1)[0].decode()
            out[nm] = (int(cnt[k]), float(ms[k]))
        return out
