"""Drop-in image-side primitives (reference imageproc.py:34-285,
rasterizer.py:71-120), computed on the GPU.

* `DistanceField(mask)`: exact nearest contour-pixel-centre queries through a
  device cell grid (reference: scipy cKDTree over the same points).
* `gaussian_pyramid(image, kernel_sizes)`: separable fp64 blur, scipy's
  `convolve1d(mode="nearest")` summation order.
* `render_depth / render_attributes / render_vertex_ids`: the two-pass device
  rasterizer reproducing the sequential "first strictly-smaller z" rule.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .device import camera_c

INTERFACE_OFFSET = 0.5
RAMP_HALF = 0.15


class DistanceField:
    """Distance field of a mask and its sampling conventions (imageproc.py:177-261)."""

    def __init__(self, mask, ctx: L.Context | None = None):
        self.ctx = ctx or L.default_context()
        self.mask = np.asarray(mask, dtype=bool)
        if self.mask.ndim != 2:
            raise ValueError("mask must be 2-D")
        self.shape = self.mask.shape
        m = L.u8c(self.mask)
        h = L.P()
        L.check(self.ctx.lib.lc_field_create(self.ctx.handle, m.shape[0], m.shape[1], L.ptr(m), C.byref(h)))
        self.handle = h

    def _query(self, pos, kind):
        pos = np.asarray(pos, dtype=np.float64)
        lead = pos.shape[:-1]
        q = L.f64c(pos.reshape(-1, 2))
        out = np.empty((len(q), 4))
        L.check(self.ctx.lib.lc_field_query(self.handle, len(q), L.ptr(q), kind, L.ptr(out)))
        return out.reshape(lead + (4,))

    @property
    def dt(self) -> np.ndarray:
        """Distance of every pixel centre to the nearest contour pixel centre
        (imageproc.py:182, euclidean_dt), computed on the device on first use."""
        if getattr(self, "_dt", None) is None:
            out = np.empty(self.shape)
            L.check(self.ctx.lib.lc_field_dt(self.handle, L.ptr(out)))
            self._dt = out
        return self._dt

    @property
    def n_contour(self) -> int:
        k = C.c_int32()
        L.check(self.ctx.lib.lc_field_n_contour(self.handle, C.byref(k)))
        return k.value

    def sample_value(self, pos):
        o = self._query(pos, 0)
        return o[..., 0], o[..., 3] != 0

    def sample_interface(self, pos):
        o = self._query(pos, 1)
        return o[..., 0], o[..., 3] != 0

    def sample_residual(self, pos):
        o = self._query(pos, 2)
        return o[..., 0], o[..., 1:3], o[..., 3] != 0

    def sample_gradient(self, pos):
        o = self._query(pos, 3)
        return o[..., 1:3], o[..., 3] != 0

    def side_direction(self, pos):
        return self._query(pos, 3)[..., 1:3]

    def inside(self, pos):
        return self._query(pos, 4)[..., 0] != 0

    def __del__(self):
        try:
            if self.handle:
                self.ctx.lib.lc_field_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def edt_squared(feature, ctx: L.Context | None = None) -> np.ndarray:
    """Exact squared Euclidean distance transform (imageproc.py:52-115)."""
    ctx = ctx or L.default_context()
    f = L.u8c(np.asarray(feature, dtype=bool))
    if f.ndim != 2:
        raise ValueError("feature image must be 2-D")
    out = np.empty(f.shape)
    L.check(ctx.lib.lc_edt_squared(ctx.handle, f.shape[0], f.shape[1], L.ptr(f), L.ptr(out)))
    return out


def euclidean_dt(mask, ctx: L.Context | None = None) -> np.ndarray:
    """Unsigned distance to the nearest contour pixel centre (imageproc.py:117-124)."""
    return DistanceField(mask, ctx).dt


def gaussian_pyramid(image, kernel_sizes=(15, 9, 3), ctx: L.Context | None = None):
    """Blur stack at full resolution, coarsest first (imageproc.py:276-285)."""
    ctx = ctx or L.default_context()
    img = L.f64c(image)
    shape = img.shape
    if img.ndim == 2:
        img = img[..., None]
    h, w, c = img.shape
    ks = np.ascontiguousarray(kernel_sizes, dtype=np.int32)
    for k in ks:
        if k < 1 or k % 2 == 0:
            raise ValueError(f"kernel size must be odd and positive, got {k}")
    taps = np.zeros((len(ks), 32))
    for i, k in enumerate(ks):
        if k <= 31:
            taps[i, :k] = L.gaussian_taps(int(k))
    out = np.empty((len(ks), h, w, c))
    L.check(ctx.lib.lc_gaussian_pyramid(ctx.handle, h, w, c, L.ptr(np.ascontiguousarray(img)), len(ks),
                                        L.ptr(ks), L.ptr(taps) if (ks <= 31).all() else None, L.ptr(out)))
    return [lvl.reshape(shape) for lvl in out]


def _render(cam, verts, tris, mode, attrs=None, ids=None, bg_attr=0.0, bg_id=-1, ctx=None):
    ctx = ctx or L.default_context()
    v = L.f64c(verts)
    t = L.i64c(tris)
    camc = camera_c(cam)
    z = np.empty((cam.height, cam.width))
    a_out = i_out = None
    a = i = None
    k = 0
    if mode == 1:
        a = L.f64c(attrs)
        if a.ndim == 1:
            a = a[:, None].copy()
        k = a.shape[1]
        a_out = np.empty((cam.height, cam.width, k))
    if mode == 2:
        i = L.i64c(ids)
        i_out = np.empty((cam.height, cam.width), dtype=np.int64)
    L.check(ctx.lib.lc_render(ctx.handle, C.byref(camc), len(v), L.ptr(v), len(t), L.ptr(t), mode,
                              L.ptr(a), k, L.ptr(i), float(bg_attr), int(bg_id), L.ptr(z), L.ptr(a_out),
                              L.ptr(i_out)))
    return z, a_out, i_out


def render_depth(cam, verts, tris, ctx=None):
    return _render(cam, verts, tris, 0, ctx=ctx)[0]


def render_mask(cam, verts, tris, ctx=None):
    return np.isfinite(render_depth(cam, verts, tris, ctx=ctx))


def render_attributes(cam, verts, tris, attrs, background=0.0, ctx=None):
    z, a, _ = _render(cam, verts, tris, 1, attrs=attrs, bg_attr=background, ctx=ctx)
    return a, z


def render_vertex_ids(cam, verts, tris, ids, background=-1, ctx=None):
    z, _, i = _render(cam, verts, tris, 2, ids=ids, bg_id=background, ctx=ctx)
    return i, z
