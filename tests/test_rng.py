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
