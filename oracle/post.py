"""ORACLE (test infrastructure only): offline post-processing of sequences.

Restates reference `pipeline.py:308-325` (smooth_trajectory), `:365-375`
(_finalize's smoothing), `:503-507` (frame_latencies) and `metrics.py:8-24`
(iou) and `metrics.py:26-106` (vertex error, Umeyama alignment, sequence
errors) with plain numpy, in the reference's accumulation order.
"""

from __future__ import annotations

import numpy as np


def smooth_trajectory(values, stencil=(0.15, 0.7, 0.15)):
    """pipeline.py:308-325: out[lo:hi] += w * arr[lo+off:hi+off] per stencil tap, / norm."""
    arr = np.asarray(values, dtype=np.float64)
    stencil = np.asarray(stencil, dtype=np.float64)
    if len(stencil) % 2 != 1:
        raise ValueError("stencil length must be odd")
    half = len(stencil) // 2
    f = arr.shape[0]
    out = np.zeros_like(arr)
    norm = np.zeros(f)
    for k, w in enumerate(stencil):
        off = k - half
        lo, hi = max(0, -off), min(f, f - off)
        out[lo:hi] += w * arr[lo + off:hi + off]
        norm[lo:hi] += w
    return out / norm.reshape((f,) + (1,) * (arr.ndim - 1))


def frame_latencies(events):
    """pipeline.py:503-507: frame -> emit slot minus ingest slot."""
    ingest, emit = {}, {}
    for e in events:
        (ingest if e["event"] == "ingest" else emit)[e["frame"]] = e["slot"]
    return {f: emit[f] - ingest[f] for f in sorted(emit)}


def iou(a, b):
    """metrics.py:8-24 (two empty masks -> 1.0)."""
    a = np.asarray(a, dtype=bool)
    b = np.asarray(b, dtype=bool)
    union = np.sum(a | b)
    return 1.0 if union == 0 else float(np.sum(a & b) / union)


def mean_vertex_error(pred, gt, indices=None, center=True):
    """metrics.py:26-46: centre both clouds on their full means, select, then
    the mean Euclidean distance."""
    pred = np.asarray(pred, dtype=np.float64)
    gt = np.asarray(gt, dtype=np.float64)
    if pred.shape != gt.shape:
        raise ValueError("vertex array shapes differ")
    if center:
        pred = pred - pred.mean(axis=0)
        gt = gt - gt.mean(axis=0)
    if indices is not None:
        pred, gt = pred[indices], gt[indices]
    return float(np.mean(np.linalg.norm(pred - gt, axis=1)))


def umeyama(src, dst, with_scaling=True):
    """metrics.py:49-76: SVD of the cross-covariance with the determinant
    sign correction."""
    src = np.asarray(src, dtype=np.float64)
    dst = np.asarray(dst, dtype=np.float64)
    if src.shape != dst.shape or src.ndim != 2:
        raise ValueError("point sets must share shape (N,D)")
    n, d = src.shape
    if n < 3:
        raise ValueError("need at least 3 points to align")
    mu_s, mu_d = src.mean(axis=0), dst.mean(axis=0)
    xs, xd = src - mu_s, dst - mu_d
    u, s, vt = np.linalg.svd(xd.T @ xs / n)
    sign = np.ones(d)
    if np.linalg.det(u @ vt) < 0.0:
        sign[-1] = -1.0
    rot = (u * sign) @ vt
    if with_scaling:
        var_s = np.mean(np.sum(xs ** 2, axis=1))
        scale = float(np.sum(s * sign) / var_s) if var_s > 0.0 else 1.0
    else:
        scale = 1.0
    return scale, rot, mu_d - scale * rot @ mu_s


def aligned_joint_error(pred, gt, with_scaling=True):
    """metrics.py:79-83."""
    scale, rot, t = umeyama(pred, gt, with_scaling)
    return float(np.mean(np.linalg.norm(scale * pred @ rot.T + t - gt, axis=1)))


def sequence_errors(pred_vertices, gt_vertices, class_indices=None):
    """metrics.py:90-106."""
    per = [mean_vertex_error(p, g) for p, g in zip(pred_vertices, gt_vertices)]
    out = {"vertex_error": float(np.mean(per)), "vertex_error_per_frame": per}
    for name, idx in (class_indices or {}).items():
        out[f"vertex_error_{name}"] = float(np.mean([mean_vertex_error(p, g, indices=idx)
                                                     for p, g in zip(pred_vertices, gt_vertices)]))
    return out
