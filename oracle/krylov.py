"""CPU oracle of the Newton step's linear solve.

TEST INFRASTRUCTURE ONLY: imported by tests/ and bench.py's baseline legs, never by the product
package.  Plain numpy / Python loops, fp64, small matrices only.

What it follows (§5 solver protocol): "30 GMRES iterations per Newton
iteration" with "block Jacobi with one block per process, ILU(0) ... in each block"; GMRES is the
Saad-Schultz method the paper cites.  The algorithms are the textbook ones, step by step:

* ilu0(): Saad, "Iterative Methods for Sparse Linear Systems", Alg. 10.4 (ILU(0), IKJ variant):
      for i = 2..n:  for k = 1..i-1 with (i,k) in NZ(A):
          a_ik := a_ik / a_kk
          for j = k+1..n with (i,j) in NZ(A):  a_ij := a_ij - a_ik * a_kj
  restricted to a diagonal block (block Jacobi: entries outside the block are dropped).
* gmres(): right-preconditioned restarted GMRES(m) (Saad Alg. 9.5) with modified Gram-Schmidt
  Arnoldi (Saad Alg. 6.2) and the Givens-rotation least-squares update (Saad §6.5.3).
  Reading A-28: a cycle ends at m iterations, at `maxit` total iterations, or when
  |g_{j+1}| <= rtol ||b||; the returned relres is the TRUE ||b - A x|| / ||b||.

Pins (tests/test_oracle_krylov.py): the ILU(0) defining property (L U)_ij = a_ij on NZ(A);
exact LU when the pattern admits no fill (banded tridiagonal); block size 1 = point Jacobi;
GMRES finite termination (n iterations, no restart -> numpy.linalg.solve); GMRES(m)'s iterate
equals the brute-force least-squares minimiser of ||b - A x|| over x0 + M^{-1} K_m.
"""
from __future__ import annotations

import math

import numpy as np


def _block_of(n, block_rows):
    """[r0, r1) of every row's block: block_rows = int (runs of that many rows), None (one block)
    or a list of block start rows (explicit partition, e.g. per-rank runs of a distributed solve)."""
    lo = np.zeros(n, np.int64)
    hi = np.zeros(n, np.int64)
    if block_rows is None or (np.isscalar(block_rows) and not block_rows):
        starts = [0]
    elif np.isscalar(block_rows):
        starts = list(range(0, n, int(block_rows)))
    else:
        starts = sorted(int(v) for v in block_rows)
    starts = [v for v in starts if v < n] + [n]
    for k in range(len(starts) - 1):
        lo[starts[k]:starts[k + 1]] = starts[k]
        hi[starts[k]:starts[k + 1]] = starts[k + 1]
    return lo, hi


def ilu0(rp, ci, val, block_rows=None):
    """Block-Jacobi ILU(0) factors of the CSR matrix (rp, ci, val) with sorted columns: returns
    `lu` on the same pattern (unit-lower L strictly below the diagonal, U on and above), only
    the entries inside each diagonal block (see _block_of) are meaningful."""
    n = len(rp) - 1
    blo, bhi = _block_of(n, block_rows)
    lu = np.array(val, dtype=np.float64, copy=True)
    pos = [dict() for _ in range(n)]               # column -> position, per row
    for i in range(n):
        for p in range(rp[i], rp[i + 1]):
            pos[i][int(ci[p])] = p
    for i in range(n):
        r0, r1 = int(blo[i]), int(bhi[i])
        for p in range(rp[i], rp[i + 1]):
            k = int(ci[p])
            if k >= i:
                break
            if k < r0:
                continue
            lu[p] = lu[p] / lu[pos[k][k]]
            for q in range(p + 1, rp[i + 1]):
                j = int(ci[q])
                if j >= r1:
                    continue
                kj = pos[k].get(j)
                if kj is not None:
                    lu[q] = lu[q] - lu[p] * lu[kj]
    return lu


def ilu0_solve(rp, ci, lu, r, block_rows=None):
    """z = (L U)^{-1} r blockwise: forward substitution with unit L, back substitution with U."""
    n = len(rp) - 1
    blo, bhi = _block_of(n, block_rows)
    z = np.zeros(n)
    for r0 in sorted(set(blo.tolist())):
        r1 = int(bhi[r0])
        for i in range(r0, r1):
            s = r[i]
            for p in range(rp[i], rp[i + 1]):
                k = int(ci[p])
                if r0 <= k < i:
                    s -= lu[p] * z[k]
            z[i] = s
        for i in range(r1 - 1, r0 - 1, -1):
            s = z[i]
            d = None
            for p in range(rp[i], rp[i + 1]):
                j = int(ci[p])
                if j == i:
                    d = lu[p]
                elif i < j < r1:
                    s -= lu[p] * z[j]
            z[i] = s / d
    return z


def csr_matvec(rp, ci, val, x):
    n = len(rp) - 1
    y = np.zeros(n)
    for i in range(n):
        y[i] = np.dot(val[rp[i]:rp[i + 1]], x[ci[rp[i]:rp[i + 1]]])
    return y


def make_precond(rp, ci, val, precond, block_rows=32):
    """M^{-1} as a function: 0 identity, 1 point Jacobi, 2 block-Jacobi ILU(0)."""
    n = len(rp) - 1
    if precond == 0:
        return lambda r: np.array(r, dtype=np.float64, copy=True)
    if precond == 1:
        d = np.array([val[rp[i] + list(ci[rp[i]:rp[i + 1]]).index(i)] for i in range(n)])
        return lambda r: r / d
    lu = ilu0(rp, ci, val, block_rows)
    return lambda r: ilu0_solve(rp, ci, lu, r, block_rows)


def gmres(rp, ci, val, b, x0=None, restart=30, maxit=30, rtol=1e-8, precond=2, block_rows=32):
    """Right-preconditioned GMRES(m), Saad Alg. 9.5 with MGS Arnoldi.  Returns (x, iters, relres)."""
    n = len(rp) - 1
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    Minv = make_precond(rp, ci, val, precond, block_rows)
    A = lambda v: csr_matvec(rp, ci, val, v)
    bnorm = np.linalg.norm(b)
    target = rtol * (bnorm if bnorm > 0 else 1.0)
    m = restart
    it = 0
    while True:
        r = b - A(x)
        beta = np.linalg.norm(r)
        if beta <= target or it >= maxit:
            break
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs, sn = np.zeros(m), np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        j = 0
        while j < m and it < maxit:
            Z[j] = Minv(V[j])
            w = A(Z[j])
            for i in range(j + 1):                      # modified Gram-Schmidt
                H[i, j] = np.dot(w, V[i])
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            hj1 = H[j + 1, j]
            if hj1 > 0:
                V[j + 1] = w / hj1
            for i in range(j):                          # previous rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = math.hypot(H[j, j], H[j + 1, j])
            cs[j] = H[j, j] / den if den > 0 else 1.0
            sn[j] = H[j + 1, j] / den if den > 0 else 0.0
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            j += 1
            it += 1
            if abs(g[j]) <= target or hj1 == 0:
                break
        y = np.zeros(j)
        for i in range(j - 1, -1, -1):                  # R y = g
            y[i] = (g[i] - np.dot(H[i, i + 1:j], y[i + 1:j])) / H[i, i]
        x = x + Z[:j].T @ y
        if abs(g[j]) <= target or it >= maxit:
            break
    relres = np.linalg.norm(b - A(x)) / (bnorm if bnorm > 0 else 1.0)
    return x, it, relres
