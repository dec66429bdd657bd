"""ORACLE (test infrastructure only): the two normal-equation solvers.

Restates reference `solvers.py:41-145`: QR solve of the dense 36x36 pose
system with rank test + Tikhonov damping, and block-Jacobi PCG on the
3x3-block sparse surface system (zero start, fixed budget, best-residual
iterate, breakdown rules).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg

RANK_DEFICIENT_RTOL = 1e-10   # solvers.py:16
DAMPING_SCALE = 1e-6          # solvers.py:17
PCG_BREAKDOWN_EPS = 1e-14     # solvers.py:18


def dense_solve(a, b):
    """Returns (delta, damped, damping)  (solvers.py:41-56)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = a.shape[0]
    q, r = np.linalg.qr(a)
    d = np.abs(np.diag(r))
    damped, lam = False, 0.0
    if d.min() < RANK_DEFICIENT_RTOL * max(d.max(), 1e-300):
        damped = True
        lam = DAMPING_SCALE * np.trace(a) / n
        if lam <= 0.0:
            lam = DAMPING_SCALE
        q, r = np.linalg.qr(a + lam * np.eye(n))
    return scipy.linalg.solve_triangular(r, q.T @ b), damped, lam


def bsr_matvec(diag, off, rows, cols, x):
    """y = D x + scatter_rows(off @ x[cols])  (solvers.py:79-84)."""
    y = np.einsum("nij,nj->ni", diag, x)
    if len(rows):
        np.add.at(y, rows, np.einsum("mij,mj->mi", off, x[cols]))
    return y


def pcg(diag, off, rows, cols, rhs, iterations=4):
    """Returns (best_x, iterations_done, breakdown, residual_norms)  (solvers.py:104-145)."""
    n = diag.shape[0]
    try:
        minv = np.linalg.inv(diag)
    except np.linalg.LinAlgError:
        minv = np.linalg.pinv(diag)
    x = np.zeros((n, 3))
    r = np.array(rhs, dtype=np.float64, copy=True)
    z = np.einsum("nij,nj->ni", minv, r)
    p = z.copy()
    rz = float(np.sum(r * z))
    norms = [float(np.linalg.norm(r))]
    best, best_norm = x.copy(), norms[0]
    done, breakdown = 0, False
    for _ in range(iterations):
        ap = bsr_matvec(diag, off, rows, cols, p)
        pap = float(np.sum(p * ap))
        if pap <= PCG_BREAKDOWN_EPS * max(float(np.sum(p * p)), 1e-300):
            breakdown = True
            break
        alpha = rz / pap
        x = x + alpha * p
        r = r - alpha * ap
        done += 1
        nr = float(np.linalg.norm(r))
        norms.append(nr)
        if nr < best_norm:
            best_norm, best = nr, x.copy()
        z = np.einsum("nij,nj->ni", minv, r)
        rz_new = float(np.sum(r * z))
        if rz <= 0.0:
            breakdown = True
            break
        p = z + (rz_new / rz) * p
        rz = rz_new
    return best, done, breakdown, norms
