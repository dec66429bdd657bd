"""The synthetic generator's random stream on the device.

The reference's generator (synthetic.py:170-203, restated in synthetic.py)
draws every frame's image noise (H*W*3 normals) and then its detection noise
and dropouts from one numpy Generator(PCG64).  `DeviceStream` draws the same
numbers on the GPU (csrc/lc_rng.cu: jump-ahead PCG64, numpy's ziggurat) and
keeps the numpy generator's state in step, so host and device draws can be
mixed and the stream continues exactly where numpy's would.

The ziggurat's tail samples (about 1 in 4000) use log1p, whose last bit may
differ between CUDA and the host libm numpy calls: the device lists them with
their draws and this module finishes them with math.log1p (the same libm
function numpy's npy_log1p is), checking that the device walked the same
number of draws.  A mismatch (never expected) raises.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib as L

MASK64 = (1 << 64) - 1
ZIG_R = 3.6541528853610088
ZIG_INV_R = 0.27366123732975828
TAIL_DRAWS = 31
_tables = None


def _zig_tables():
    global _tables
    if _tables is None:
        ki = np.zeros(256, dtype=np.uint64)
        wi = np.zeros(256)
        fi = np.zeros(256)
        L.check(L.load_library().lc_rng_tables(L.ptr(ki), L.ptr(wi), L.ptr(fi)))
        _tables = ([int(x) for x in ki], [float(x) for x in wi], [float(x) for x in fi])
    return _tables


def _dbl(u: int) -> float:
    return (u >> 11) * (1.0 / 9007199254740992.0)


def _walk(draws) -> tuple[float, int]:
    """random_standard_normal over the given draws (numpy/random/src/
    distributions/distributions.c): (value, draws consumed)."""
    ki, wi, fi = _zig_tables()
    p = 0
    while True:
        r = int(draws[p])
        p += 1
        idx = r & 0xFF
        r >>= 8
        sign = r & 1
        rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
        x = rabs * wi[idx]
        if sign:
            x = -x
        if rabs < ki[idx]:
            return x, p
        if idx == 0:
            while True:
                xx = -ZIG_INV_R * math.log1p(-_dbl(int(draws[p])))
                yy = -math.log1p(-_dbl(int(draws[p + 1])))
                p += 2
                if yy + yy > xx * xx:
                    return (-(ZIG_R + xx) if ((rabs >> 8) & 1) else ZIG_R + xx), p
        elif (fi[idx - 1] - fi[idx]) * _dbl(int(draws[p])) + fi[idx] < math.exp(-0.5 * x * x):
            return x, p + 1
        else:
            p += 1


class DeviceStream:
    """numpy Generator(PCG64) draws on the device, in step with `rng`."""

    def __init__(self, rng: np.random.Generator, ctx: L.Context | None = None):
        if not isinstance(rng.bit_generator, np.random.PCG64):
            raise ValueError("DeviceStream follows a PCG64 generator (np.random.default_rng)")
        self.rng = rng
        self.ctx = ctx or L.default_context()

    def _state(self):
        st = self.rng.bit_generator.state["state"]
        s, inc = st["state"], st["inc"]
        return (np.array([s >> 64, s & MASK64], dtype=np.uint64),
                np.array([inc >> 64, inc & MASK64], dtype=np.uint64))

    def normal_(self, out, loc: float, scale: float, add_clip: bool = False):
        """Fill the contiguous float64 device tensor `out` with
        rng.normal(loc, scale, out.shape) (add_clip: out = clip(out + noise,
        0, 1), the generator's image noise) and advance `rng` past the draws."""
        import torch
        if not (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.float64
                and out.is_contiguous()):
            raise ValueError("out must be a contiguous float64 CUDA tensor")
        n = out.numel()
        s, inc = self._state()
        max_tails = max(64, n // 256)
        tails = np.zeros(2 * max_tails, dtype=np.int64)
        draws = np.zeros(max_tails * TAIL_DRAWS, dtype=np.uint64)
        consumed, nt = C.c_int64(), C.c_int32()
        lib = self.ctx.lib
        L.check(lib.lc_rng_normal(self.ctx.handle, L.ptr(s), L.ptr(inc), float(loc), float(scale),
                                  out.data_ptr(), n, int(add_clip), C.byref(consumed), L.ptr(tails), L.ptr(draws),
                                  max_tails, C.byref(nt)))
        k = nt.value
        if k:
            idx = np.ascontiguousarray(tails[0:2 * k:2])
            want = tails[1:2 * k:2]
            vals = np.empty(k)
            if int(want.max()) > TAIL_DRAWS:   # (a tail sample of > 15 rejection rounds: never observed)
                raise RuntimeError("a ziggurat tail sample took more draws than the device records")
            for t in range(k):
                z, used = _walk(draws[t * TAIL_DRAWS:(t + 1) * TAIL_DRAWS])
                if used != int(want[t]):
                    raise RuntimeError("device ziggurat walk disagrees with libm on a tail sample")
                vals[t] = loc + scale * z
            if add_clip:
                orig = np.empty(k)
                L.check(lib.lc_rng_gather(self.ctx.handle, L.ptr(idx), k, out.data_ptr(), L.ptr(orig)))
                vals = np.clip(orig + vals, 0.0, 1.0)
            L.check(lib.lc_rng_scatter(self.ctx.handle, L.ptr(idx), L.ptr(vals), k, out.data_ptr()))
        self.rng.bit_generator.advance(consumed.value)
        return out

    def normal(self, loc: float, scale: float, size, device=None):
        import torch
        out = torch.empty(size, dtype=torch.float64, device=device or f"cuda:{self.ctx.device}")
        return self.normal_(out, loc, scale)

    def random(self, size, device=None):
        """rng.random(size) on the device."""
        import torch
        out = torch.empty(size, dtype=torch.float64, device=device or f"cuda:{self.ctx.device}")
        s, inc = self._state()
        L.check(self.ctx.lib.lc_rng_uniform(self.ctx.handle, L.ptr(s), L.ptr(inc), out.data_ptr(), out.numel()))
        self.rng.bit_generator.advance(out.numel())
        return out
