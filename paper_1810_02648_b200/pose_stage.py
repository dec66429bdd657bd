"""Drop-in Stage I (reference pose_stage.py:284-459) on the GPU.

`solve_pose(problem, init)` accepts the reference's `PoseProblem` (or this
module's mirror with the same fields) and runs all Gauss-Newton steps, the
36x36 QR solves and the halving line search in one persistent CTA.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .config import ContourVertexSet, PoseParams
from .device import DeviceActor, camera_c, pose_hyper_c, pose_report_from_c


@dataclass
class PoseProblem:
    """Per-frame Stage I data (same fields as the reference, pose_stage.py:284-297)."""
    skeleton: object
    skinning: object
    camera: object
    detections: object           # joints3d already bone-length rescaled
    dt_field: object | None      # DistanceField (ours or the reference's): `.mask` is read
    contour: ContourVertexSet
    contour_rest: np.ndarray
    hyper: object
    prev_positions: np.ndarray | None = None
    directional: bool = True
    contour_enabled: np.ndarray | None = None


def solve_pose(problem, init, ctx: L.Context | None = None):
    """Damped Gauss-Newton with step halving (pose_stage.py:429-459).
    Returns (PoseParams, PoseStageReport)."""
    ctx = ctx or L.default_context()
    dev = DeviceActor.for_pose(problem.skeleton, problem.skinning, ctx)
    det = problem.detections
    keep = dict(
        mask=None if problem.dt_field is None else L.u8c(problem.dt_field.mask),
        j2d=L.f64c(det.joints2d), j3d=L.f64c(det.joints3d), v2d=L.u8c(det.valid2d), v3d=L.u8c(det.valid3d),
        idx=L.i64c(problem.contour.indices), n2d=L.f64c(problem.contour.normals2d).reshape(-1, 2),
        rest=L.f64c(problem.contour_rest).reshape(-1, 3),
        en=None if problem.contour_enabled is None else L.u8c(problem.contour_enabled),
        prev=None if problem.prev_positions is None else L.f64c(problem.prev_positions))
    pb = L.PoseProblemC()
    pb.mask = L.ptr(keep["mask"])
    pb.joints2d, pb.joints3d = L.ptr(keep["j2d"]), L.ptr(keep["j3d"])
    pb.valid2d, pb.valid3d = L.ptr(keep["v2d"]), L.ptr(keep["v3d"])
    pb.n_contour = len(keep["idx"])
    pb.contour_indices, pb.contour_normals2d = L.ptr(keep["idx"]), L.ptr(keep["n2d"])
    pb.contour_rest, pb.contour_enabled = L.ptr(keep["rest"]), L.ptr(keep["en"])
    pb.prev_positions = L.ptr(keep["prev"])
    pb.directional = int(problem.directional)
    pb.hyper = pose_hyper_c(problem.hyper)
    cam = camera_c(problem.camera)
    x0 = L.f64c(init.to_vector())
    x = np.empty(36)
    rep = L.PoseReport()
    L.check(ctx.lib.lc_pose_solve(ctx.handle, dev.handle, C.byref(cam), C.byref(pb), L.ptr(x0), L.ptr(x),
                                  C.byref(rep)))
    return PoseParams.from_vector(x), pose_report_from_c(rep)


def extract_contour_vertices(verts, actor, camera, ctx: L.Context | None = None) -> ContourVertexSet:
    """Occluding-contour vertices of `verts` (pose_stage.py:151-191); the
    visibility z-buffer is rendered on the device."""
    ctx = ctx or L.default_context()
    dev = DeviceActor.get(actor, ctx) if hasattr(actor, "skeleton") else DeviceActor.for_mesh(actor, ctx)
    v = L.f64c(verts)
    n = C.c_int32()
    idx = np.empty(len(v), dtype=np.int64)
    n2d = np.empty((len(v), 2))
    cam = camera_c(camera)
    L.check(ctx.lib.lc_contour_vertices(ctx.handle, dev.handle, C.byref(cam), L.ptr(v), C.byref(n),
                                        L.ptr(idx), L.ptr(n2d)))
    return ContourVertexSet(idx[:n.value].copy(), n2d[:n.value].copy())


def tracker_sets(verts, actor, camera, stage: int = 2, part_gate: bool = True, dilation: int = 10,
                 with_labels: bool = False, ctx: L.Context | None = None) -> dict:
    """The tracker's own index / set work on `verts` (one lc_surface_sets
    call): contour indices + normals2d (extract_contour_vertices), the rim
    keep flags (outer_rim_mask; stage 1 with the thickness probes and the
    rigidity >= 2 gate of pipeline.py:211, stage 2 without, AND the part
    gating of pipeline.py:241-249 when part_gate), the visible ids (stage 2,
    visible_vertices) and optionally the part label image
    (build_body_part_mask)."""
    ctx = ctx or L.default_context()
    dev = DeviceActor.get(actor, ctx)
    v = L.f64c(verts)
    N = len(v)
    nb, nv = C.c_int32(), C.c_int32()
    idx, vis = np.empty(N, dtype=np.int64), np.empty(N, dtype=np.int64)
    n2d, keep = np.empty((N, 2)), np.empty(N, dtype=np.uint8)
    labels = np.empty((camera.height, camera.width), dtype=np.int32) if with_labels else None
    cam = camera_c(camera)
    L.check(ctx.lib.lc_surface_sets(ctx.handle, dev.handle, C.byref(cam), L.ptr(v), int(stage), int(bool(part_gate)),
                                    int(dilation), C.byref(nb), L.ptr(idx), L.ptr(n2d), L.ptr(keep), C.byref(nv),
                                    L.ptr(vis), L.ptr(labels)))
    out = {"contour": idx[:nb.value].copy(), "normals2d": n2d[:nb.value].copy(),
           "keep": keep[:nb.value].astype(bool)}
    if stage == 2:
        out["visible"] = vis[:nv.value].copy()
    if with_labels:
        out["labels"] = labels
    return out
