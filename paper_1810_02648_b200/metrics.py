"""Tracking-quality metrics on the device (reference `metrics.py:8-106`).

Same names, arguments and errors as the reference module.  The arithmetic runs
in `liblivecap.so` (`csrc/lc_eval.cu`, `csrc/lc_post.cu`):
  - `iou` / `iou_batch`: per-frame pixel counts (`lc_mask_overlap`);
  - `mean_vertex_error`: bit-identical to numpy (`lc_mean_vertex_error`);
  - `umeyama_alignment` / `aligned_joint_error`: a Jacobi SVD of the 3x3
    cross-covariance in place of LAPACK's (`lc_aligned_error`, ~1e-15).
Batched forms (`*_batch`) evaluate a whole sequence in one launch.
"""

from __future__ import annotations

import numpy as np

from . import _lib as L
from .postprocess import iou_batch  # noqa: F401  (re-export)


def iou(mask_a, mask_b, return_empty_flag: bool = False):
    """metrics.py:8-23: two empty masks count as 1.0 (flagged on request)."""
    a = np.asarray(mask_a, dtype=bool)
    b = np.asarray(mask_b, dtype=bool)
    if a.shape != b.shape:
        raise ValueError("mask shapes differ")
    ctx = L.default_context()
    inter = np.zeros(1, dtype=np.uint64)
    uni = np.zeros(1, dtype=np.uint64)
    aa = np.ascontiguousarray(a).view(np.uint8)
    bb = np.ascontiguousarray(b).view(np.uint8)
    L.check(ctx.lib.lc_mask_overlap(ctx.handle, 1, int(a.size), L.ptr(aa), L.ptr(bb), L.ptr(inter), L.ptr(uni)))
    empty = int(uni[0]) == 0
    value = 1.0 if empty else float(np.float64(inter[0]) / np.float64(uni[0]))
    if return_empty_flag:
        return value, bool(empty)
    return value


def mean_vertex_error_batch(pred, gt, indices=None, center: bool = True, ctx: L.Context | None = None):
    """Per-frame `mean_vertex_error` of (F,N,3) stacks (or one (N,3) pair)."""
    ctx = ctx or L.default_context()
    pred = np.asarray(pred, dtype=np.float64)
    gt = np.asarray(gt, dtype=np.float64)
    if pred.shape != gt.shape:
        raise ValueError("vertex array shapes differ")
    single = pred.ndim == 2
    p = L.f64c(pred[None] if single else pred)
    g = L.f64c(gt[None] if single else gt)
    if p.ndim != 3 or p.shape[2] != 3:
        raise ValueError("vertex arrays must be (N,3) or (F,N,3)")
    F, N = p.shape[0], p.shape[1]
    idx = None
    if indices is not None:
        idx = np.asarray(indices)
        if idx.dtype == bool:
            idx = np.flatnonzero(idx)
        idx = np.ascontiguousarray(idx, dtype=np.int64).ravel()
        if len(idx) == 0:
            return np.full(F, np.nan) if not single else float("nan")
        if np.any(idx >= N) or np.any(idx < -N):
            raise IndexError("vertex index out of range")
    out = np.empty(F)
    L.check(ctx.lib.lc_mean_vertex_error(ctx.handle, F, N, L.ptr(p), L.ptr(g), L.ptr(idx),
                                         0 if idx is None else len(idx), int(bool(center)), 0, L.ptr(out)))
    return float(out[0]) if single else out


def mean_vertex_error(pred, gt, indices=None, center: bool = True) -> float:
    """metrics.py:26-46: mean per-vertex distance after removing each cloud's
    mean position (centring on the full clouds, before index selection)."""
    pred = np.asarray(pred, dtype=np.float64)
    gt = np.asarray(gt, dtype=np.float64)
    if pred.shape != gt.shape:
        raise ValueError("vertex array shapes differ")
    return float(mean_vertex_error_batch(pred, gt, indices, center))


def _aligned(pred, gt, with_scaling, ctx=None):
    ctx = ctx or L.default_context()
    src = np.asarray(pred, dtype=np.float64)
    dst = np.asarray(gt, dtype=np.float64)
    if src.shape != dst.shape or src.ndim not in (2, 3):
        raise ValueError("point sets must share shape (N,D)")
    single = src.ndim == 2
    s = L.f64c(src[None] if single else src)
    d = L.f64c(dst[None] if single else dst)
    F, M, D = s.shape
    if D != 3:
        raise ValueError("only 3-D point sets are supported")
    if M < 3:
        raise ValueError("need at least 3 points to align")
    scale, rot, t, err = np.empty(F), np.empty((F, 3, 3)), np.empty((F, 3)), np.empty(F)
    L.check(ctx.lib.lc_aligned_error(ctx.handle, F, M, L.ptr(s), L.ptr(d), int(bool(with_scaling)), 0,
                                     L.ptr(scale), L.ptr(rot), L.ptr(t), L.ptr(err)))
    return single, scale, rot, t, err


def umeyama_alignment(src, dst, with_scaling: bool = True):
    """metrics.py:49-76: least-squares similarity dst ~ scale * R @ src + t
    (proper rotation; needs at least 3 points)."""
    _, scale, rot, t, _ = _aligned(src, dst, with_scaling)
    return float(scale[0]), rot[0], t[0]


def aligned_joint_error(pred, gt, with_scaling: bool = True) -> float:
    """metrics.py:79-83: mean joint distance after the similarity alignment."""
    return float(_aligned(pred, gt, with_scaling)[4][0])


def aligned_joint_error_batch(pred, gt, with_scaling: bool = True, ctx: L.Context | None = None) -> np.ndarray:
    """Per-frame aligned_joint_error of (F,J,3) stacks, one launch."""
    return _aligned(pred, gt, with_scaling, ctx)[4]


def max_angle_error(theta_pred, theta_gt) -> float:
    """metrics.py:86-87 (27 numbers: host)."""
    return float(np.max(np.abs(np.asarray(theta_pred) - np.asarray(theta_gt))))


def sequence_errors(pred_vertices, gt_vertices, class_indices: dict | None = None) -> dict:
    """metrics.py:90-106: overall and per-class mean surface errors."""
    pred_vertices = np.asarray(pred_vertices)
    gt_vertices = np.asarray(gt_vertices)
    per_frame = [float(e) for e in mean_vertex_error_batch(pred_vertices, gt_vertices)] \
        if len(pred_vertices) else []
    out = {"vertex_error": float(np.mean(per_frame)), "vertex_error_per_frame": per_frame}
    if class_indices:
        for name, idx in class_indices.items():
            vals = mean_vertex_error_batch(pred_vertices, gt_vertices, indices=idx) if len(pred_vertices) else []
            out[f"vertex_error_{name}"] = float(np.mean(vals))
    return out
