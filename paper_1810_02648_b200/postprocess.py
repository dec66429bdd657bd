"""Offline post-processing of tracked sequences on the device.

Mirrors reference `pipeline.py:308-325` (`smooth_trajectory`) and
`metrics.py:8-24` (`iou`, batched over frames).  Both go through the C-ABI
(`lc_smooth_trajectory`, `lc_mask_overlap`); the smoothing kernel
accumulates in the reference's order and is bit-identical to it.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L


def smooth_trajectory(values, stencil=(0.15, 0.7, 0.15), ctx: L.Context | None = None) -> np.ndarray:
    """Centred weighted average along axis 0, truncated and renormalised at
    the ends (reference pipeline.py:308-325)."""
    ctx = ctx or L.default_context()
    arr = np.ascontiguousarray(values, dtype=np.float64)
    st = np.ascontiguousarray(stencil, dtype=np.float64)
    if st.ndim != 1 or len(st) % 2 != 1:
        raise ValueError("stencil length must be odd")
    if arr.shape[0] == 0:
        return arr.copy()
    F = arr.shape[0]
    D = int(arr.size // F)
    out = np.empty_like(arr)
    L.check(ctx.lib.lc_smooth_trajectory(ctx.handle, F, D, L.ptr(arr), len(st), L.ptr(st), L.ptr(out)))
    return out


def iou_batch(masks_a, masks_b, ctx: L.Context | None = None) -> np.ndarray:
    """Per-frame intersection over union of two (F, H, W) mask stacks
    (metrics.iou; two empty masks count as 1.0)."""
    ctx = ctx or L.default_context()
    a = np.ascontiguousarray(masks_a, dtype=bool).view(np.uint8)
    b = np.ascontiguousarray(masks_b, dtype=bool).view(np.uint8)
    if a.shape != b.shape:
        raise ValueError("mask shapes differ")
    if a.ndim == 2:
        a, b = a[None], b[None]
    F = a.shape[0]
    HW = int(a[0].size)
    inter = np.zeros(F, dtype=np.uint64)
    uni = np.zeros(F, dtype=np.uint64)
    L.check(ctx.lib.lc_mask_overlap(ctx.handle, F, HW, L.ptr(a), L.ptr(b), L.ptr(inter), L.ptr(uni)))
    out = np.ones(F)
    nz = uni > 0
    out[nz] = inter[nz].astype(np.float64) / uni[nz].astype(np.float64)
    return out


def iou(mask_a, mask_b) -> float:
    return float(iou_batch(mask_a, mask_b)[0])
