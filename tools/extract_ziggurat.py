"""Extract numpy's normal-ziggurat tables (ki_double, wi_double, fi_double)
from the static library numpy ships for Cython users
(numpy/random/lib/libnpyrandom.a, object src_distributions_distributions.c.o)
and write paper_1810_02648_b200/csrc/lc_ziggurat_tables.h.  The device
generator (csrc/lc_rng.cu) draws Generator.normal with these tables, so its
noise is numpy's bit for bit (tests/test_rng.py checks the restatement
against numpy on CPU, tests/test_gpu_rng.py the device kernels).

  python tools/extract_ziggurat.py
"""
import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_1810_02648_b200", "csrc", "lc_ziggurat_tables.h")


def tables():
    lib = os.path.join(os.path.dirname(np.__file__), "random", "lib", "libnpyrandom.a")
    member = "src_distributions_distributions.c.o"
    tmp = tempfile.mkdtemp()
    subprocess.run(["ar", "x", lib, member], cwd=tmp, check=True)
    obj = os.path.join(tmp, member)
    syms = {}
    for line in subprocess.run(["nm", obj], capture_output=True, text=True, check=True).stdout.splitlines():
        p = line.split()
        if len(p) == 3 and p[2] in ("ki_double", "wi_double", "fi_double"):
            syms[p[2]] = int(p[0], 16)
    # file offset of .rodata
    sec = subprocess.run(["readelf", "-S", "-W", obj], capture_output=True, text=True, check=True).stdout
    off = None
    for line in sec.splitlines():
        if " .rodata " in line + " ":
            f = line.split()
            i = f.index(".rodata")
            off = int(f[i + 3], 16)
            break
    data = open(obj, "rb").read()
    out = {}
    for name, fmt in (("ki_double", "<256Q"), ("wi_double", "<256d"), ("fi_double", "<256d")):
        a = off + syms[name]
        out[name] = struct.unpack(fmt, data[a:a + 2048])
    return out


def main():
    t = tables()
    lines = ["// numpy's normal-ziggurat tables (numpy/random/src/distributions/ziggurat_constants.h,",
             "// BSD-3-Clause), extracted from numpy's libnpyrandom.a by tools/extract_ziggurat.py",
             f"// (numpy {np.__version__}).  Generated file.",
             "#pragma once", "#include <cstdint>", ""]
    lines.append("__device__ static const uint64_t lc_zig_ki[256] = {")
    lines += [", ".join(f"0x{v:016x}ULL" for v in t["ki_double"][i:i + 4]) + "," for i in range(0, 256, 4)]
    lines.append("};")
    for name, key in (("lc_zig_wi", "wi_double"), ("lc_zig_fi", "fi_double")):
        lines.append(f"__device__ static const double {name}[256] = {{")
        lines += [", ".join(float(v).hex() for v in t[key][i:i + 4]) + "," for i in range(0, 256, 4)]
        lines.append("};")
    open(OUT, "w").write("\n".join(lines) + "\n")
    print(f"wrote {OUT}")


if __name__ == "__main__":
    sys.exit(main())
