"""Seeded synthetic inputs for the five BASELINE.json configs (shared by tests, bench, smoke).

This module holds NONE of the method's arithmetic (no basis evaluation, no quadrature,
no integrand, no assembly).  It only draws the numbers both the CUDA path and the CPU
oracle are handed bit-identically: open knot vectors, control points / weights of the
synthetic geometries, physics parameters, and the solution coefficient arrays U, Udot.

Recipes (SURVEY.md §8(d) table and readings A-19..A-23):

cfg 1  Poisson validation (SPEC demo): [0,1]^2, open uniform p=2 knots, N x N elements,
       identity geometry as NURBS with Greville control points and unit weights (A-19);
       LAPLACE kappa=1, sigma=0, f = 2 pi^2 sin(pi x) sin(pi y); U = 0; (a,b) = (0,1).
cfg 2  NURBS quarter annulus r in [1,2], theta in [0,pi/2] (P:55-58 exact geometry),
       cubic C^2, N x N; homogeneous control points are the exact blossoms of the
       quadratic (angular) x linear (radial) numerators (A-20); LAPLACE kappa=sigma=1, f=0;
       U ~ U[-1,1] i.i.d. seed 2; (a,b) = (0,1).
cfg 3  Cahn-Hilliard, [0,1]^2 periodic C^1 quadratic (the library unclamps the open knot
       vector with Alg. 1), parametric geometry; c = 0.63 + U[-0.05,0.05] seed 3,
       cdot = 0; theta=1.5, alpha=3000; a = alpha_m = 5/6, b = alpha_f*gamma*dt = (4/9)*1e-6
       (rho_inf = 0.5).
cfg 4  Neo-Hookean, [0,1]^3 open C^1 quadratic, parametric, 3 dofs/node, E=1, nu=0.3
       (lambda, mu by A-13); u = 0.05 sum_{m<8} a_m sin(pi k_m.X + phi_m) sampled at the
       Greville abscissae (A-22, A-23); (a,b) = (0,1).
cfg 5  RBVMS Navier-Stokes, [0,2pi]^3 periodic C^1 quadratic, 4 dofs/node (u,v,w,p);
       Taylor-Green velocity + 0.01*U[-1,1] seed 5 and its pressure at Greville points;
       Udot = 0; nu = 1/1600, dt = 1e-2, C_t = 4, C_I = 36; a = 5/6, b = (4/9)*1e-2.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np

PHYS_LAPLACE, PHYS_CAHN_HILLIARD, PHYS_NEOHOOKE, PHYS_NS_VMS, PHYS_NSK = 0, 1, 2, 3, 4
GEOM_PARAMETRIC, GEOM_NURBS = 0, 1

# full-size element counts per axis (BASELINE.json configs[0..4])
FULL_N = {1: 16, 2: 256, 3: 1024, 4: 64, 5: 128, 6: 256, 7: 256, 8: 256}
NAMES = {1: "poisson2d_p2_16x16", 2: "annulus_lapmass_p3_256x256", 3: "cahn_hilliard2d_p2_1024x1024",
         4: "neohooke3d_p2_64x64x64", 5: "ns_vms3d_p2_128x128x128", 6: "nsk2d_p2_256x256",
         7: "ring_alg2_lapmass_p2_256x256", 8: "cahn_hilliard3d_p2_256x256x256"}


@dataclass
class Workload:
    cid: int
    name: str
    dim: int
    degree: list
    knots: list            # open (clamped) knot vectors, one np.float64 array per axis
    periodic: list
    continuity: list       # C^k across the periodic seam (only read when periodic)
    dof: int
    quad: list
    geometry: int
    ctrl: np.ndarray | None      # [n0][n1][n2][dim] Euclidean control points, or None
    weights: np.ndarray | None   # [n0][n1][n2] projective weights, or None (=> 1)
    phys: int
    params: list
    a: float
    b: float
    U: np.ndarray          # [n0*n1*n2*dof] dof innermost, last axis fastest
    Udot: np.ndarray
    nel: list = field(default_factory=list)
    nfun: list = field(default_factory=list)   # unique functions per axis

    @property
    def ndof(self) -> int:
        return int(np.prod(self.nfun)) * self.dof

    @property
    def nqp(self) -> int:
        return int(np.prod(self.nel)) * int(np.prod(self.quad))

    @property
    def nelem(self) -> int:
        return int(np.prod(self.nel))


def open_uniform_knots(p: int, n: int, a: float = 0.0, b: float = 1.0) -> np.ndarray:
    """p+1 copies of a, a+(b-a)i/n for i=1..n-1, p+1 copies of b (SURVEY O-1)."""
    inner = [a + (b - a) * i / n for i in range(1, n)]
    return np.array([a] * (p + 1) + inner + [b] * (p + 1), dtype=np.float64)


def _greville(U: np.ndarray, p: int) -> np.ndarray:
    """Sample locations (Greville abscissae) of an OPEN knot vector: (t_{i+1}+..+t_{i+p})/p."""
    n = len(U) - p - 1
    return np.array([sum(U[i + 1:i + p + 1]) / p for i in range(n)], dtype=np.float64)


def _periodic_greville(a: float, b: float, n: int, p: int) -> np.ndarray:
    """Sample locations for the n unique functions of a uniform C^{p-1} periodic space on [a,b]:
    function g is centred at a + (g + (1-p)/2) h (h=(b-a)/n), i.e. the Greville abscissa of the
    uniformly extended knots.  Only used to place the synthetic field samples."""
    h = (b - a) / n
    return np.array([a + (g + 0.5 * (1 - p)) * h for g in range(n)], dtype=np.float64)


def _blossom_quadratic_in_cubic(c0: float, c1: float, c2: float, t: np.ndarray) -> float:
    """Blossom of f(x)=c0+c1 x+c2 x^2 viewed as a cubic, at knots t1,t2,t3 (A-20)."""
    t1, t2, t3 = t
    return c0 + c1 * (t1 + t2 + t3) / 3.0 + c2 * (t1 * t2 + t1 * t3 + t2 * t3) / 3.0


def annulus_geometry(U0: np.ndarray, U1: np.ndarray, p: int = 3):
    """Exact quarter-annulus NURBS in the cubic space (A-20): xi0 radial r = 1 + xi0, xi1 angular.

    Homogeneous numerators of the quadratic arc (P0=(1,0),P1=(1,1),P2=(0,1), w=(1,1/sqrt2,1)):
      wx(t) = (1-t)^2 + sqrt2 t(1-t),  wy(t) = sqrt2 t(1-t) + t^2,  w(t) = (1-t)^2 + sqrt2 t(1-t) + t^2
    expanded in the monomial basis; each B-spline coefficient is the blossom at its p interior knots.
    """
    s2 = math.sqrt(2.0)
    # monomial coefficients (c0, c1, c2)
    wx = (1.0, -2.0 + s2, 1.0 - s2)
    wy = (0.0, s2, 1.0 - s2)
    ww = (1.0, -2.0 + s2, 2.0 - s2)
    n0 = len(U0) - p - 1
    n1 = len(U1) - p - 1
    R = np.array([_blossom_quadratic_in_cubic(1.0, 1.0, 0.0, U0[i + 1:i + p + 1]) for i in range(n0)])
    WX = np.array([_blossom_quadratic_in_cubic(*wx, U1[j + 1:j + p + 1]) for j in range(n1)])
    WY = np.array([_blossom_quadratic_in_cubic(*wy, U1[j + 1:j + p + 1]) for j in range(n1)])
    W = np.array([_blossom_quadratic_in_cubic(*ww, U1[j + 1:j + p + 1]) for j in range(n1)])
    ctrl = np.zeros((n0, n1, 2))
    ctrl[:, :, 0] = R[:, None] * (WX / W)[None, :]
    ctrl[:, :, 1] = R[:, None] * (WY / W)[None, :]
    weights = np.broadcast_to(W[None, :], (n0, n1)).copy()
    return ctrl, weights


def make(cid: int, n=None, seed: int | None = None) -> Workload:
    """Build config `cid` (1..5) with n elements per axis (default: the full BASELINE size); n may
    be a list with one count per axis (weak-scaling meshes of bench.py --gpus N)."""
    dims = {1: 2, 2: 2, 3: 2, 4: 3, 5: 3, 6: 2, 7: 2, 8: 3}[cid] if cid in FULL_N else 0
    if n is None:
        n = FULL_N[cid]
    nn = list(n) if isinstance(n, (list, tuple)) else [int(n)] * dims
    w = _make(cid, nn, seed)
    if any(x != nn[0] for x in nn) or nn[0] != FULL_N.get(cid):
        w.name = NAMES[cid].rsplit("_", 1)[0] + "_" + "x".join(str(x) for x in nn)
    return w


def _make(cid: int, nn: list, seed: int | None = None) -> Workload:
    n = nn[0]
    if seed is None:
        seed = cid
    rng = np.random.default_rng(seed)
    if cid == 1:
        p, d = 2, 2
        U = [open_uniform_knots(p, nn[a]) for a in range(d)]
        g = [_greville(u, p) for u in U]
        nf = [len(x) for x in g]
        ctrl = np.zeros((nf[0], nf[1], 2))
        ctrl[:, :, 0] = g[0][:, None]
        ctrl[:, :, 1] = g[1][None, :]
        w = Workload(1, NAMES[1], d, [p] * d, U, [0] * d, [p - 1] * d, 1, [p + 1] * d, GEOM_NURBS,
                     ctrl, np.ones(nf), PHYS_LAPLACE, [1.0, 0.0, 1.0], 0.0, 1.0,
                     np.zeros(nf[0] * nf[1]), np.zeros(nf[0] * nf[1]), list(nn), nf)
    elif cid == 2:
        p, d = 3, 2
        U = [open_uniform_knots(p, nn[a]) for a in range(d)]
        ctrl, weights = annulus_geometry(U[0], U[1], p)
        nf = [ctrl.shape[0], ctrl.shape[1]]
        nd = nf[0] * nf[1]
        w = Workload(2, NAMES[2], d, [p] * d, U, [0] * d, [p - 1] * d, 1, [p + 1] * d, GEOM_NURBS,
                     ctrl, weights, PHYS_LAPLACE, [1.0, 1.0, 0.0], 0.0, 1.0,
                     rng.uniform(-1.0, 1.0, nd), np.zeros(nd), list(nn), nf)
    elif cid == 3:
        p, d = 2, 2
        U = [open_uniform_knots(p, nn[a]) for a in range(d)]
        nf = [nn[0], nn[1]]
        nd = nf[0] * nf[1]
        c = 0.63 + rng.uniform(-0.05, 0.05, nd)
        dt = 1e-6
        w = Workload(3, NAMES[3], d, [p] * d, U, [1] * d, [p - 1] * d, 1, [p + 1] * d, GEOM_PARAMETRIC,
                     None, None, PHYS_CAHN_HILLIARD, [1.5, 3000.0], 5.0 / 6.0, (4.0 / 9.0) * dt,
                     c, np.zeros(nd), list(nn), nf)
    elif cid == 4:
        p, d = 2, 3
        U = [open_uniform_knots(p, nn[a]) for a in range(d)]
        g = [_greville(u, p) for u in U]
        nf = [len(x) for x in g]
        # A-22: idx, phi, amplitude drawn in this order from default_rng(4)
        kvecs = [k for k in itertools.product((0, 1), repeat=3) if any(k)]
        idx = rng.integers(0, 7, 8)
        phi = rng.uniform(0.0, 2.0 * math.pi, 8)
        amp = rng.uniform(-1.0, 1.0, (8, 3))
        X = np.stack(np.meshgrid(g[0], g[1], g[2], indexing="ij"), axis=-1)   # [n0,n1,n2,3]
        disp = np.zeros(X.shape)
        for m in range(8):
            kv = np.array(kvecs[idx[m]], dtype=np.float64)
            s = np.sin(math.pi * (X @ kv) + phi[m])
            disp += amp[m][None, None, None, :] * s[..., None]
        disp *= 0.05
        E, nu = 1.0, 0.3
        lam = E * nu / ((1 + nu) * (1 - 2 * nu))
        mu = E / (2 * (1 + nu))
        w = Workload(4, NAMES[4], d, [p] * d, U, [0] * d, [p - 1] * d, 3, [p + 1] * d, GEOM_PARAMETRIC,
                     None, None, PHYS_NEOHOOKE, [lam, mu], 0.0, 1.0,
                     disp.reshape(-1).copy(), np.zeros(disp.size), list(nn), nf)
    elif cid == 5:
        p, d = 2, 3
        L = 2.0 * math.pi
        U = [open_uniform_knots(p, nn[a], 0.0, L) for a in range(d)]
        gs = [_periodic_greville(0.0, L, nn[a], p) for a in range(d)]
        x, y, z = np.meshgrid(gs[0], gs[1], gs[2], indexing="ij")
        vel = np.stack([np.sin(x) * np.cos(y) * np.cos(z),
                        -np.cos(x) * np.sin(y) * np.cos(z),
                        np.zeros_like(x)], axis=-1)
        vel = vel + 0.01 * rng.uniform(-1.0, 1.0, vel.shape)
        pres = (np.cos(2 * x) + np.cos(2 * y)) * (np.cos(2 * z) + 2.0) / 16.0
        Uarr = np.concatenate([vel, pres[..., None]], axis=-1).reshape(-1).copy()
        dt = 1e-2
        w = Workload(5, NAMES[5], d, [p] * d, U, [1] * d, [p - 1] * d, 4, [p + 1] * d, GEOM_PARAMETRIC,
                     None, None, PHYS_NS_VMS, [1.0 / 1600.0, dt, 4.0, 36.0], 5.0 / 6.0, (4.0 / 9.0) * dt,
                     Uarr, np.zeros(Uarr.size), list(nn), list(nn))
    elif cid == 6:
        # Navier-Stokes-Korteweg (not a BASELINE config): [0,1]^2 periodic C^1
        # quadratic, parametric, unknowns (rho, u1, u2); three vapour bubbles in liquid (the paper's
        # three-bubble test) as a smooth density field at the Greville points, small
        # seeded velocity and time derivatives; van der Waals a = 3, b = 1, R = 8/27, theta = 0.85
        # (sub-critical), mu_bar = 1/512, lambda_bar = -2/3 mu_bar, capillarity lambda = 1/512^2
        # (readings A-25..A-27); generalized-alpha (a, b) with dt = 1e-3.
        p, d = 2, 2
        U = [open_uniform_knots(p, nn[a]) for a in range(d)]
        gs = [_periodic_greville(0.0, 1.0, nn[a], p) for a in range(d)]
        x, y = np.meshgrid(gs[0], gs[1], indexing="ij")
        rho = np.full(x.shape, 0.6)
        for (cx, cy, r) in ((0.30, 0.30, 0.10), (0.62, 0.60, 0.15), (0.25, 0.72, 0.08)):
            dist = np.hypot(x - cx, y - cy)
            rho -= 0.25 * (1.0 + np.tanh((r - dist) / 0.04))
        vel = 0.01 * rng.uniform(-1.0, 1.0, x.shape + (2,))
        Uarr = np.concatenate([rho[..., None], vel], axis=-1).reshape(-1).copy()
        Udot = 0.01 * rng.uniform(-1.0, 1.0, Uarr.size)
        dt = 1e-3
        mub = 1.0 / 512.0
        w = Workload(6, NAMES[6], d, [p] * d, U, [1] * d, [p - 1] * d, 3, [p + 1] * d, GEOM_PARAMETRIC,
                     None, None, PHYS_NSK, [3.0, 1.0, 8.0 / 27.0, 0.85, mub, -2.0 / 3.0 * mub, 1.0 / 512.0 ** 2],
                     5.0 / 6.0, (4.0 / 9.0) * dt, Uarr, Udot, list(nn), list(nn))
    elif cid == 7:
        # Periodic mapped geometry (Alg. 2): a ring, axis 0 radial (open p = 2,
        # r = 1 + Greville abscissa in [1, 2]), axis 1 angular, periodic C^1 quadratic.  Unique
        # homogeneous points Q_g = w_g (r cos t_g, r sin t_g, 1), t_g = 2 pi g / nu, w_g ~ U[0.8, 1.2]
        # seed 7 (a smooth rational closed curve near the circle); the caller hands the CLAMPED net
        # of that periodic curve: P_j = Q_j (1 <= j <= n-2), P_{n-1} = Q_0 and P_0 = P_n =
        # (Q_0 + Q_1)/2 -- the C^1 seam condition of uniform clamped quadratics, homogeneous.  Both
        # sides unclamp it with Alg. 2.  LAPLACE kappa = sigma = 1, f = 0, U ~ U[-1, 1]; (a, b) = (0, 1).
        p, d = 2, 2
        U = [open_uniform_knots(p, nn[a]) for a in range(d)]
        r = 1.0 + _greville(U[0], p)
        nf0, nopen1 = len(r), nn[1] + p
        nu1 = nopen1 - 2
        t = 2.0 * math.pi * np.arange(nu1) / nu1
        wq = rng.uniform(0.8, 1.2, nu1)
        Q = np.zeros((nf0, nu1, 3))
        Q[:, :, 0] = r[:, None] * np.cos(t)[None, :] * wq[None, :]
        Q[:, :, 1] = r[:, None] * np.sin(t)[None, :] * wq[None, :]
        Q[:, :, 2] = wq[None, :]
        n = nopen1 - 1
        Pw = np.zeros((nf0, nopen1, 3))
        Pw[:, 1:n - 1] = Q[:, 1:n - 1]
        Pw[:, n - 1] = Q[:, 0]
        Pw[:, 0] = Pw[:, n] = 0.5 * (Q[:, 0] + Q[:, 1])
        ctrl = Pw[:, :, :2] / Pw[:, :, 2:]
        weights = Pw[:, :, 2].copy()
        nd = nf0 * nu1
        w = Workload(7, NAMES[7], d, [p] * d, U, [0, 1], [p - 1] * d, 1, [p + 1] * d, GEOM_NURBS,
                     ctrl, weights, PHYS_LAPLACE, [1.0, 1.0, 0.0], 0.0, 1.0,
                     rng.uniform(-1.0, 1.0, nd), np.zeros(nd), list(nn), [nf0, nu1])
    elif cid == 8:
        # 3D Cahn-Hilliard (the Fig. 5 run): [0,1]^3 periodic C^1
        # quadratic, 256^3 elements, random initial condition as in config 3 (c = 0.63 +
        # U[-0.05, 0.05], seed 8), cdot = 0, theta = 1.5, alpha = 3000, rho_inf = 0.5, dt = 1e-6.
        p, d = 2, 3
        U = [open_uniform_knots(p, nn[a]) for a in range(d)]
        nf = [nn[0], nn[1], nn[2]]
        nd = nf[0] * nf[1] * nf[2]
        c = 0.63 + rng.uniform(-0.05, 0.05, nd)
        dt = 1e-6
        w = Workload(8, NAMES[8], d, [p] * d, U, [1] * d, [p - 1] * d, 1, [p + 1] * d, GEOM_PARAMETRIC,
                     None, None, PHYS_CAHN_HILLIARD, [1.5, 3000.0], 5.0 / 6.0, (4.0 / 9.0) * dt,
                     c, np.zeros(nd), list(nn), nf)
    else:
        raise ValueError(f"unknown config {cid}")
    return w


def probe_rows(w: Workload, nblocks_random: int = 4, block: int = 3, seed: int = 5) -> np.ndarray:
    """Sorted global dof rows for probe-block parity at full size (SURVEY O-10, reduced):
    block^d node boxes at the low corner / seam, the middle (a partition plane), the
    quarter point, the high corner, plus `nblocks_random` seeded random boxes; all dofs."""
    nf = w.nfun
    d = w.dim
    rng = np.random.default_rng(seed)
    starts = []
    for frac in (0.0, 0.5, 0.25):
        starts.append([int(frac * f) for f in nf])
    starts.append([f - block for f in nf])
    for _ in range(nblocks_random):
        starts.append([int(rng.integers(0, f - block + 1)) for f in nf])
    rows = set()
    for s in starts:
        for off in itertools.product(range(block), repeat=d):
            node = 0
            for ax in range(d):
                node = node * nf[ax] + min(max(s[ax] + off[ax], 0), nf[ax] - 1)
            for c in range(w.dof):
                rows.add(node * w.dof + c)
    return np.array(sorted(rows), dtype=np.int64)


def custom(dim: int, degree, knots, periodic=None, continuity=None, dof: int = 1, phys: int = PHYS_LAPLACE,
           params=(1.0, 1.0, 0.0), a: float = 0.0, b: float = 1.0, geometry: int = GEOM_PARAMETRIC,
           field: str = "uniform", seed: int = 0, name: str = "custom") -> Workload:
    """A seeded workload on explicit OPEN knot vectors (GPU parity of the knot-driven cases: repeated
    interior knots, non-uniform spacing, periodic C^k with k < p-1, p = 1, mixed degrees).

    geometry NURBS (open axes only): control points at the Greville abscissae of each axis plus a
    smooth seeded shear, weights ~ U[0.8, 1.2] -- a non-affine rational map (both sides check
    detJ > 0).  field: "uniform" U ~ U[-1, 1]; "ch" c = 0.63 + U[-0.05, 0.05]; "small" 0.02 U[-1, 1]
    (hyperelastic displacements).  Udot ~ 0.1 U[-1, 1]."""
    rng = np.random.default_rng(seed)
    deg = list(degree) if isinstance(degree, (list, tuple)) else [int(degree)] * dim
    kn = [np.asarray(k, dtype=np.float64) for k in knots]
    per = list(periodic) if periodic is not None else [0] * dim
    cont = list(continuity) if continuity is not None else [p - 1 for p in deg]
    nopen = [len(kn[d]) - deg[d] - 1 for d in range(dim)]
    nf = [nopen[d] - (cont[d] + 1) if per[d] else nopen[d] for d in range(dim)]
    nel = [len(np.unique(kn[d])) - 1 for d in range(dim)]
    ctrl = weights = None
    if geometry == GEOM_NURBS:
        assert not any(per), "custom NURBS geometry: open axes only (periodic nets go through Alg. 2, config 7)"
        g = [_greville(kn[d], deg[d]) for d in range(dim)]
        grids = np.meshgrid(*g, indexing="ij")
        ctrl = np.stack(grids, axis=-1).copy()
        span = [kn[d][-1] - kn[d][0] for d in range(dim)]
        for d in range(dim):
            o = (d + 1) % dim
            ctrl[..., d] += 0.04 * span[d] * np.sin(np.pi * (grids[o] - kn[o][0]) / span[o])
        weights = rng.uniform(0.8, 1.2, nopen)
    nd = int(np.prod(nf)) * dof
    if field == "ch":
        U = 0.63 + rng.uniform(-0.05, 0.05, nd)
    elif field == "small":
        U = 0.02 * rng.uniform(-1.0, 1.0, nd)
    else:
        U = rng.uniform(-1.0, 1.0, nd)
    Udot = 0.1 * rng.uniform(-1.0, 1.0, nd)
    return Workload(0, name, dim, deg, kn, per, cont, dof, [p + 1 for p in deg], geometry, ctrl, weights, phys,
                    list(params), a, b, U, Udot, nel, nf)


def probe_rows_o10(w: Workload, block: int = 5, nrandom: int = 64, seed: int = 5) -> np.ndarray:
    """SURVEY O-10 probe set: block^d node boxes (all dofs) centred, per axis, at every combination
    of {periodic seam / first node 0, the partition plane N/2, the interior N/4} (3^d structured
    probes), plus `nrandom` seeded random boxes.  Open axes clamp a box to the node range, periodic
    axes wrap it.  Returns sorted unique global dof rows."""
    nf, d = w.nfun, w.dim
    rng = np.random.default_rng(seed)
    centres = [list(c) for c in itertools.product(*[(0, f // 2, f // 4) for f in nf])]
    for _ in range(nrandom):
        centres.append([int(rng.integers(0, f)) for f in nf])
    half = block // 2
    rows = set()
    for c in centres:
        for off in itertools.product(range(-half, block - half), repeat=d):
            node = 0
            for ax in range(d):
                g = c[ax] + off[ax]
                if w.periodic[ax]:
                    g %= nf[ax]
                else:
                    g = min(max(g, 0), nf[ax] - 1)
                node = node * nf[ax] + g
            for m in range(w.dof):
                rows.add(node * w.dof + m)
    return np.array(sorted(rows), dtype=np.int64)
