"""Drop-in Stage II (reference nonrigid_stage.py:160-500) on the GPU.

`solve_nonrigid(problem, v0)` and `snap_vertices(v, problem)` accept the
reference's `NonrigidProblem` (or the mirror below with the same fields);
residual assembly, the matrix-free block-Jacobi PCG, the halving line
search and the snapping walk all run in one persistent CTA.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .config import ContourVertexSet, SnapInfo
from .device import DeviceActor, camera_c, nonrigid_hyper_c, nonrigid_report_from_c


@dataclass
class NonrigidProblem:
    """Per-frame Stage II data (same fields as the reference, nonrigid_stage.py:160-176)."""
    mesh: object
    camera: object
    hyper: object
    skinned: np.ndarray
    pyramid: list
    dt_field: object | None
    visible: np.ndarray
    boundary: ContourVertexSet
    boundary_enabled: np.ndarray
    prev: np.ndarray | None = None
    prev2: np.ndarray | None = None
    directional: bool = True
    enable_photo: bool = True
    enable_sil: bool = True


def _run(problem, v0, do_solve, do_snap, ctx):
    ctx = ctx or L.default_context()
    dev = DeviceActor.for_mesh(problem.mesh, ctx)
    levels = len(problem.pyramid)
    keep = dict(
        mask=None if problem.dt_field is None else L.u8c(problem.dt_field.mask),
        pyr=L.f64c(np.stack([np.asarray(p, dtype=np.float64) for p in problem.pyramid])) if levels else None,
        vs=L.f64c(problem.skinned), vis=L.i64c(problem.visible), bidx=L.i64c(problem.boundary.indices),
        n2d=L.f64c(problem.boundary.normals2d).reshape(-1, 2), en=L.u8c(problem.boundary_enabled),
        prev=None if problem.prev is None else L.f64c(problem.prev),
        prev2=None if problem.prev2 is None else L.f64c(problem.prev2), v0=L.f64c(v0))
    if levels and keep["pyr"].shape[1:] != (problem.camera.height, problem.camera.width, 3):
        raise ValueError("pyramid levels must be (H,W,3) images matching the camera")
    pb = L.NonrigidProblemC()
    pb.mask = L.ptr(keep["mask"])
    pb.n_levels = max(levels, 1)
    pb.pyramid = L.ptr(keep["pyr"])
    pb.skinned = L.ptr(keep["vs"])
    pb.n_visible, pb.visible = len(keep["vis"]), L.ptr(keep["vis"])
    pb.n_boundary, pb.boundary = len(keep["bidx"]), L.ptr(keep["bidx"])
    pb.normals2d, pb.enabled = L.ptr(keep["n2d"]), L.ptr(keep["en"])
    pb.prev, pb.prev2 = L.ptr(keep["prev"]), L.ptr(keep["prev2"])
    pb.directional = int(problem.directional)
    pb.enable_photo = int(getattr(problem, "enable_photo", True) and levels > 0)
    pb.enable_sil = int(getattr(problem, "enable_sil", True))
    pb.hyper = nonrigid_hyper_c(problem.hyper, n_levels=max(levels, 1))
    cam = camera_c(problem.camera)
    v = np.empty_like(keep["v0"])
    rep = L.NonrigidReport()
    L.check(ctx.lib.lc_nonrigid_solve(ctx.handle, dev.handle, C.byref(cam), C.byref(pb), L.ptr(keep["v0"]),
                                      int(do_solve), int(do_snap), L.ptr(v), C.byref(rep)))
    return v, rep


def solve_nonrigid(problem, v0, ctx: L.Context | None = None):
    """Coarse-to-fine Gauss-Newton with a fixed PCG budget (nonrigid_stage.py:372-403).
    Returns (vertices, NonrigidStageReport)."""
    v, rep = _run(problem, v0, True, False, ctx)
    return v, nonrigid_report_from_c(rep)


def snap_vertices(v, problem, ctx: L.Context | None = None):
    """Silhouette snapping (nonrigid_stage.py:417-500). Returns (vertices, SnapInfo)."""
    out, rep = _run(problem, v, False, True, ctx)
    info = SnapInfo(int(rep.snap_walked), int(rep.snap_reached), int(rep.snap_stuck))
    info.moved_vertices = np.flatnonzero(np.any(out != np.asarray(v), axis=1))
    return out, info
