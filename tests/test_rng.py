"""CPU: the restated numpy Generator(PCG64) stream (oracle/rng.py) is numpy's,
bit for bit -- uint64 draws, doubles, jump-ahead and standard normals
(ziggurat fast path, wedge and tail), the random stream the reference's
synthetic generator draws its image noise and detections from."""
import numpy as np
import pytest

from oracle import rng as R


@pytest.mark.parametrize("seed", [0, 7, 12345])
def test_pcg64_uint64_and_double(seed):
    g = np.random.Generator(np.random.PCG64(seed))
    p = R.Pcg64.from_numpy(g.bit_generator)
    want = g.bit_generator.random_raw(1000)
    got = np.array([p.next64() for _ in range(1000)], dtype=np.uint64)
    assert np.array_equal(want, got)
    d = g.random(100)
    assert np.array_equal(d, np.array([p.next_double() for _ in range(100)]))


def test_pcg64_advance():
    g = np.random.Generator(np.random.PCG64(3))
    p = R.Pcg64.from_numpy(g.bit_generator)
    p.advance(123457)
    g.bit_generator.advance(123457)
    assert p.s == g.bit_generator.state["state"]["state"]
    assert p.next64() == int(g.bit_generator.random_raw())


@pytest.mark.parametrize("seed", [0, 1, 99])
def test_standard_normal_bit_exact(seed):
    g = np.random.Generator(np.random.PCG64(seed))
    n = R.Normal(R.Pcg64.from_numpy(g.bit_generator))
    want = g.normal(0.0, 0.02, 20000)
    got = np.array(n.normal(0.0, 0.02, 20000))
    assert np.array_equal(want, got)
    # the stream position after the draws is numpy's too
    assert n.g.s == g.bit_generator.state["state"]["state"]


def test_committed_device_tables_match_numpy():
    """csrc/lc_ziggurat_tables.h (the device's tables) is what
    tools/extract_ziggurat.py reads from the installed numpy."""
    import os
    import re
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "tools"))
    import extract_ziggurat
    t = extract_ziggurat.tables()
    src = open(os.path.join(root, "paper_1810_02648_b200", "csrc", "lc_ziggurat_tables.h")).read()
    ki = [int(x, 16) for x in re.findall(r"0x([0-9a-f]{16})ULL", src)]
    assert ki == list(t["ki_double"])
    fl = [float.fromhex(x) for x in re.findall(r"(-?0x[0-9a-f.]+p[-+]?\d+|0x0\.0p\+0)", src)]
    assert fl == list(t["wi_double"]) + list(t["fi_double"])
