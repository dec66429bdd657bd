"""Drop-in `solvers` (reference solvers.py:21-145), computed on the GPU.

`pcg_solve(BlockSparseSystem)` and `dense_solve(DenseNormalSystem)` accept the
reference's own system objects (any object with the same fields) and return
the reference's (solution, info) tuples.  Validation and error behaviour
follow the reference: malformed systems raise ValueError at construction;
numerical trouble (rank deficiency, PCG breakdown) becomes info flags.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .config import DenseSolveInfo, PcgInfo

RANK_DEFICIENT_RTOL = 1e-10
DAMPING_SCALE = 1e-6
PCG_BREAKDOWN_EPS = 1e-14


@dataclass
class DenseNormalSystem:
    a: np.ndarray
    b: np.ndarray

    def __post_init__(self):
        self.a = np.asarray(self.a, dtype=np.float64)
        self.b = np.asarray(self.b, dtype=np.float64)
        if self.a.ndim != 2 or self.a.shape[0] != self.a.shape[1]:
            raise ValueError("system matrix must be square")
        if not (np.isfinite(self.a).all() and np.isfinite(self.b).all()):
            raise ValueError("non-finite entries in normal system")


@dataclass
class BlockSparseSystem:
    diag: np.ndarray      # (N,3,3)
    off: np.ndarray       # (M,3,3)
    off_rows: np.ndarray  # (M,)
    off_cols: np.ndarray  # (M,)
    rhs: np.ndarray       # (N,3)

    def __post_init__(self):
        self.diag = np.asarray(self.diag, dtype=np.float64)
        self.off = np.asarray(self.off, dtype=np.float64).reshape(-1, 3, 3)
        self.off_rows = np.asarray(self.off_rows, dtype=np.int64)
        self.off_cols = np.asarray(self.off_cols, dtype=np.int64)
        self.rhs = np.asarray(self.rhs, dtype=np.float64)

    @property
    def n_blocks(self) -> int:
        return self.diag.shape[0]


def dense_solve(system, ctx: L.Context | None = None):
    """QR solve with rank test and Tikhonov damping (solvers.py:41-56)."""
    ctx = ctx or L.default_context()
    a = L.f64c(system.a)
    b = L.f64c(system.b)
    n = a.shape[0]
    x = np.empty(n)
    info = L.DenseInfo()
    L.check(ctx.lib.lc_dense_solve(ctx.handle, n, L.ptr(a), L.ptr(b), L.ptr(x), C.byref(info)))
    return x, DenseSolveInfo(bool(info.damped), float(info.damping))


def pcg_solve(system, iterations: int = 4, ctx: L.Context | None = None):
    """Block-Jacobi PCG from zero returning the best-residual iterate
    (solvers.py:104-145)."""
    ctx = ctx or L.default_context()
    diag = L.f64c(system.diag).reshape(-1, 3, 3)
    off = L.f64c(system.off).reshape(-1, 3, 3)
    rows = L.i64c(system.off_rows)
    cols = L.i64c(system.off_cols)
    rhs = L.f64c(system.rhs).reshape(-1, 3)
    n = diag.shape[0]
    x = np.empty((n, 3))
    info = L.PcgInfo()
    L.check(ctx.lib.lc_pcg_solve_bsr(ctx.handle, n, len(rows), L.ptr(diag), L.ptr(off), L.ptr(rows),
                                     L.ptr(cols), L.ptr(rhs), int(iterations), L.ptr(x), C.byref(info)))
    out = PcgInfo(iterations=int(info.iterations), breakdown=bool(info.breakdown),
                  residual_norms=[float(info.residual_norms[k]) for k in range(info.iterations + 1)])
    return x, out
