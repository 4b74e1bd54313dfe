"""GPU parity of the third-order basis evaluation (iga_basis_eval) against
the oracle's orc_eval_point3 at every Gauss point of every element: R_A and all spatial
derivatives up to third order, each order within 1e-11 of that order's max |value| at the point.
Covers the rational / non-affine path (NURBS annulus), parametric 2D (open and periodic knots),
3D open and periodic."""
import ctypes as C

import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-11


def _gauss(n):
    x, w = np.zeros(n), np.zeros(n)
    oracle.lib().orc_gauss_legendre(n, x.ctypes.data_as(C.POINTER(C.c_double)), w.ctypes.data_as(C.POINTER(C.c_double)))
    return x


def _spans(U, p, nfun):
    return [i for i in range(p, nfun) if U[i] < U[i + 1]]


@pytest.mark.parametrize("cid,n", [(1, 5), (2, 3), (2, 6), (3, 5), (4, 2), (5, 5)])
def test_basis3_parity(cid, n):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1305_4452_b200 as iga
    w = workloads.make(cid, n=n)
    sp = iga.Space.from_workload(w)
    out = sp.basis_eval(3).cpu().numpy()
    sp.check()
    osp = oracle.Space.from_workload(w)
    d = w.dim
    # unclamped knots / spans / Gauss points per axis, as the oracle defines them
    axes = []
    for a in range(d):
        nk = len(w.knots[a])
        U = np.zeros(nk)
        oracle.lib().orc_space_knots(osp.h, a, U.ctypes.data_as(C.POINTER(C.c_double)))
        p = w.degree[a]
        sp_ = _spans(U, p, nk - p - 1)
        axes.append((U, sp_, _gauss(w.quad[a])))
    nel = [len(ax[1]) for ax in axes]
    nq = [len(ax[2]) for ax in axes]
    assert out.shape[0] == int(np.prod(nel)) and out.shape[3] == int(np.prod(nq))
    worst = 0.0
    for el in range(out.shape[0]):
        e = list(np.unravel_index(el, nel))
        for q in range(out.shape[3]):
            qq = list(np.unravel_index(q, nq))
            xi = []
            for a in range(d):
                U, spans, gx = axes[a]
                lo, hi = U[spans[e[a]]], U[spans[e[a]] + 1]
                xi.append(0.5 * (lo + hi) + 0.5 * (hi - lo) * gx[qq[a]])
            ev = osp.eval_point3(e, xi)
            ref = [ev["R"][:, None], ev["dR"][:, :d], ev["ddR"][:, :d, :d].reshape(-1, d * d),
                   ev["dddR"][:, :d, :d, :d].reshape(-1, d ** 3)]
            got = out[el, :, :, q]
            c0 = 0
            for k, r in enumerate(ref):
                g = got[:, c0:c0 + r.shape[1]]
                c0 += r.shape[1]
                scale = max(np.abs(r).max(), 1e-300)
                err = np.abs(g - r).max() / scale
                worst = max(worst, err)
                assert err <= TOL, (cid, el, q, k, err)
    assert worst <= TOL
