"""Test infrastructure (checker only, never shipped): a restatement of the
random stream the reference's synthetic generator draws from --
numpy.random.Generator(PCG64) (numpy 2.3, BSD-3-Clause; the reference calls
np.random.default_rng(seed).normal / .random in synthetic.py:170-203,
restated by paper_1810_02648_b200/synthetic.py).

* PCG64 (numpy/random/src/pcg64/pcg64.h): 128-bit LCG state,
  s <- s * 0x2360ed051fc65da44385df649fccf645 + inc, output XSL-RR of the new
  state: rotr64(hi ^ lo, s >> 122).
* next_double = (next_uint64 >> 11) * 2**-53.
* random_standard_normal (numpy/random/src/distributions/distributions.c):
  256-layer ziggurat with numpy's tables (tools/extract_ziggurat.py), the
  tail via log1p(-U), the wedge test fi[i-1]-fi[i] against exp(-x^2/2).
* normal(loc, scale) = loc + scale * standard_normal, elementwise in C order.

Pure-Python loops: for small cases (tests/test_rng.py checks it bit for bit
against numpy, slow paths included); the device kernels (csrc/lc_rng.cu)
follow the same steps and are checked against numpy on the GPU.
"""
import math
import os
import sys

MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
ZIG_R = 3.6541528853610088
ZIG_INV_R = 0.27366123732975828


def _tables():
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import extract_ziggurat
    t = extract_ziggurat.tables()
    return t["ki_double"], t["wi_double"], t["fi_double"]


class Pcg64:
    def __init__(self, state: int, inc: int):
        self.s = state & MASK128
        self.inc = inc & MASK128

    @classmethod
    def from_numpy(cls, bitgen):
        st = bitgen.state["state"]
        return cls(st["state"], st["inc"])

    def next64(self) -> int:
        self.s = (self.s * PCG_MULT + self.inc) & MASK128
        hi, lo = self.s >> 64, self.s & MASK64
        x = hi ^ lo
        r = self.s >> 122
        return ((x >> r) | (x << ((64 - r) & 63))) & MASK64

    def next_double(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def advance(self, delta: int):
        """Jump ahead by delta steps (the LCG's affine map, squared up)."""
        acc_mult, acc_plus = 1, 0
        cur_mult, cur_plus = PCG_MULT, self.inc
        while delta > 0:
            if delta & 1:
                acc_mult = (acc_mult * cur_mult) & MASK128
                acc_plus = (acc_plus * cur_mult + cur_plus) & MASK128
            cur_plus = ((cur_mult + 1) * cur_plus) & MASK128
            cur_mult = (cur_mult * cur_mult) & MASK128
            delta >>= 1
        self.s = (acc_mult * self.s + acc_plus) & MASK128


class Normal:
    def __init__(self, gen: Pcg64):
        self.g = gen
        self.ki, self.wi, self.fi = _tables()

    def standard(self) -> float:
        g, ki, wi, fi = self.g, self.ki, self.wi, self.fi
        while True:
            r = g.next64()
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * wi[idx]
            if sign:
                x = -x
            if rabs < ki[idx]:
                return x
            if idx == 0:
                while True:
                    xx = -ZIG_INV_R * math.log1p(-g.next_double())
                    yy = -math.log1p(-g.next_double())
                    if yy + yy > xx * xx:
                        return -(ZIG_R + xx) if ((rabs >> 8) & 1) else ZIG_R + xx
            else:
                if (fi[idx - 1] - fi[idx]) * g.next_double() + fi[idx] < math.exp(-0.5 * x * x):
                    return x

    def normal(self, loc: float, scale: float, n: int):
        return [loc + scale * self.standard() for _ in range(n)]
