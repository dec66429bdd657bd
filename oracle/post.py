"""ORACLE (test infrastructure only): offline post-processing of sequences.

Restates reference `pipeline.py:308-325` (smooth_trajectory), `:365-375`
(_finalize's smoothing), `:503-507` (frame_latencies) and `metrics.py:8-24`
(iou) with plain numpy, in the reference's accumulation order.
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
