"""ORACLE (test infrastructure only): masks, distance fields, raster, pyramid.

Restates reference `imageproc.py:34-285` and `rasterizer.py:18-120`.  The two
numba kernels are in `oracle/csrc/oracle_raster.c` (built by
`oracle.build_oracle_lib()` into `oracle/_build/liboracle.so`); the cKDTree
and `convolve1d` calls are the reference's own third-party dependencies
(scipy 1.18.1, present in this image and on the GPU box).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

INTERFACE_OFFSET = 0.5   # imageproc.py:27
RAMP_HALF = 0.15         # imageproc.py:29
EDT_INF = 1e18

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None


def build_oracle_lib(force: bool = False) -> str:
    src = os.path.join(_HERE, "csrc", "oracle_raster.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def _clib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build_oracle_lib())
        P = ctypes.c_void_p
        _lib.oracle_raster.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, ctypes.c_int64,
                                       P, ctypes.c_int, P, P, P, P, ctypes.c_int]
        _lib.oracle_edt_squared.argtypes = [ctypes.c_int, ctypes.c_int, P, P]
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# rasterizer (rasterizer.py:71-120)

def _raster(cam, verts, tris, mode, attrs=None, ids=None, bg_attr=0.0, bg_id=-1):
    from .geometry import project
    pix, ok = project(cam, verts)
    pix = np.ascontiguousarray(pix)
    depth = np.ascontiguousarray(np.where(ok, np.asarray(verts)[:, 2], -1.0))
    tris = np.ascontiguousarray(tris, dtype=np.int64)
    zbuf = np.full((cam.height, cam.width), np.inf)
    k = 1
    a = np.zeros((1, 1))
    abuf = np.zeros(1)
    i = np.zeros(1, dtype=np.int64)
    ibuf = np.zeros(1, dtype=np.int64)
    if mode == 1:
        a = np.ascontiguousarray(attrs, dtype=np.float64)
        if a.ndim == 1:
            a = a[:, None]
        k = a.shape[1]
        abuf = np.full((cam.height, cam.width, k), bg_attr)
    elif mode == 2:
        i = np.ascontiguousarray(ids, dtype=np.int64)
        ibuf = np.full((cam.height, cam.width), bg_id, dtype=np.int64)
    _clib().oracle_raster(cam.height, cam.width, _ptr(pix), _ptr(depth), _ptr(tris), len(tris),
                          _ptr(a), k, _ptr(i), _ptr(zbuf), _ptr(abuf), _ptr(ibuf), mode)
    return zbuf, abuf, ibuf


def render_depth(cam, verts, tris):
    return _raster(cam, verts, tris, 0)[0]


def render_attributes(cam, verts, tris, attrs, background=0.0):
    zbuf, abuf, _ = _raster(cam, verts, tris, 1, attrs=attrs, bg_attr=background)
    return abuf, zbuf


def render_vertex_ids(cam, verts, tris, ids, background=-1):
    zbuf, _, ibuf = _raster(cam, verts, tris, 2, ids=ids, bg_id=background)
    return ibuf, zbuf


# ---------------------------------------------------------------------------
# masks, EDT (imageproc.py:34-124)

def contour_mask(mask):
    m = np.asarray(mask, dtype=bool)
    p = np.pad(m, 1, constant_values=False)
    interior = p[:-2, 1:-1] & p[2:, 1:-1] & p[1:-1, :-2] & p[1:-1, 2:]
    return m & ~interior


def edt_squared(feature):
    f = np.ascontiguousarray(feature, dtype=np.uint8)
    out = np.empty(f.shape)
    _clib().oracle_edt_squared(f.shape[0], f.shape[1], _ptr(f), _ptr(out))
    return out


def euclidean_dt(mask):
    c = contour_mask(mask)
    if not c.any():
        raise ValueError("mask has no foreground, distance transform undefined")
    return np.sqrt(edt_squared(c))


# ---------------------------------------------------------------------------
# bilinear sampling with analytic gradient (imageproc.py:127-174)

def sample_bilinear(image, pos):
    img = np.asarray(image, dtype=np.float64)
    flat = img.ndim == 2
    if flat:
        img = img[..., None]
    h, w = img.shape[0], img.shape[1]
    pos = np.asarray(pos, dtype=np.float64)
    x, y = pos[..., 0], pos[..., 1]
    clamped = (x < 0) | (x > w - 1) | (y < 0) | (y > h - 1)
    xc = np.clip(x, 0.0, w - 1.0)
    yc = np.clip(y, 0.0, h - 1.0)
    x0 = np.minimum(np.floor(xc).astype(np.int64), w - 2)
    y0 = np.minimum(np.floor(yc).astype(np.int64), h - 2)
    fx = (xc - x0)[..., None]
    fy = (yc - y0)[..., None]
    c00, c01 = img[y0, x0], img[y0, x0 + 1]
    c10, c11 = img[y0 + 1, x0], img[y0 + 1, x0 + 1]
    top = c00 * (1 - fx) + c01 * fx
    bot = c10 * (1 - fx) + c11 * fx
    val = top * (1 - fy) + bot * fy
    gx = ((c01 - c00) * (1 - fy) + (c11 - c10) * fy) * ((x >= 0) & (x <= w - 1))[..., None]
    gy = (bot - top) * ((y >= 0) & (y <= h - 1))[..., None]
    grad = np.stack([gx, gy], axis=-1)
    if flat:
        return val[..., 0], grad[..., 0, :], clamped
    return val, grad, clamped


# ---------------------------------------------------------------------------
# continuous distance field (imageproc.py:177-261)

class DistanceField:
    """Exact nearest contour-pixel-centre distance; cKDTree as in the reference."""

    def __init__(self, mask):
        from scipy.spatial import cKDTree
        self.mask = np.asarray(mask, dtype=bool)
        self.shape = self.mask.shape
        self.points = np.argwhere(contour_mask(self.mask))[:, ::-1].astype(np.float64)
        if len(self.points) == 0:
            raise ValueError("mask has no foreground, distance transform undefined")
        self.tree = cKDTree(self.points)

    def nearest(self, pos):
        pos = np.asarray(pos, dtype=np.float64)
        fin = np.isfinite(pos).all(axis=-1)
        q = np.where(fin[..., None], pos, 0.0)
        dist, idx = self.tree.query(q)
        feat = self.tree.data[idx]
        vec = (q - feat) / np.maximum(dist, 1e-12)[..., None]
        vec = vec * ((dist > 1e-12) & fin)[..., None]
        return dist * fin, vec, ~fin

    def sample_value(self, pos):
        d, _, c = self.nearest(pos)
        return d, c

    def sample_interface(self, pos):
        d, c = self.sample_value(pos)
        return np.maximum(d - INTERFACE_OFFSET, 0.0), c

    def sample_residual(self, pos):
        d, vec, c = self.nearest(pos)
        lo, hi = INTERFACE_OFFSET - RAMP_HALF, INTERFACE_OFFSET + RAMP_HALF
        t = np.clip(d - lo, 0.0, hi - lo)
        far = d >= hi
        res = np.where(far, d - INTERFACE_OFFSET, t * t / (4.0 * RAMP_HALF))
        slope = np.where(far, 1.0, t / (2.0 * RAMP_HALF))
        return res, vec * slope[..., None], c

    def sample_gradient(self, pos):
        _, vec, c = self.nearest(pos)
        return vec, c

    def side_direction(self, pos):
        return self.nearest(pos)[1]

    def inside(self, pos):
        pos = np.asarray(pos, dtype=np.float64)
        h, w = self.shape
        xi = np.round(pos[..., 0]).astype(np.int64)
        yi = np.round(pos[..., 1]).astype(np.int64)
        ok = (xi >= 0) & (xi < w) & (yi >= 0) & (yi < h)
        return ok & self.mask[np.clip(yi, 0, h - 1), np.clip(xi, 0, w - 1)]


# ---------------------------------------------------------------------------
# blur pyramid (imageproc.py:264-285)

def gaussian_kernel(size):
    if size < 1 or size % 2 == 0:
        raise ValueError(f"kernel size must be odd and positive, got {size}")
    if size == 1:
        return np.ones(1)
    sigma = (size - 1) / 6.0
    x = np.arange(size) - (size - 1) / 2.0
    k = np.exp(-0.5 * (x / sigma) ** 2)
    return k / k.sum()


def gaussian_pyramid(image, kernel_sizes=(15, 9, 3)):
    from scipy.ndimage import convolve1d
    img = np.asarray(image, dtype=np.float64)
    out = []
    for size in kernel_sizes:
        k = gaussian_kernel(size)
        out.append(convolve1d(convolve1d(img, k, axis=0, mode="nearest"), k, axis=1, mode="nearest"))
    return out
