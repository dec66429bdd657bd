"""CPU: the oracle reproduces the REAL reference bit for bit on the bench's
own workloads (tools/make_golden.py --bench): the bench's seed-0 stream at
x5k @1024² with directional=False over frames 0-24, and cfg4 (x20k @1024²,
4 GN x 8 PCG) over frames 0-2.  Free-running: the oracle's recursion must
give the reference's poses, vertex digests and per-iteration energies
exactly, which pins the checker the GPU parity tests
(tests/test_gpu_bench_parity.py) compare against."""

import numpy as np
import pytest

from helpers import scene_bench
from test_oracle_golden import check_digest, load


def _digest(v):
    return dict(sum=v.sum(axis=(1, 2)), sq=(v ** 2).sum(axis=(1, 2)), rows=v[:, ::97])


@pytest.mark.parametrize("name", ["ref_digest_x5k1024_dir0.npz", "ref_digest_x20k1024_cfg4.npz"])
def test_oracle_matches_reference_on_bench_workloads(name):
    from oracle import frame as OF
    from paper_1810_02648_b200.config import SequenceConfig
    g = load(name)
    preset, res, n, directional, seed, gn, pcg = g["meta"]
    actor, cam, frames = scene_bench(preset, int(res), int(n), int(seed))
    check_digest(g, frames)
    cfg = SequenceConfig(directional=bool(int(directional)))
    if gn != "None":
        cfg.nonrigid.gn_iterations = int(gn)
    if pcg != "None":
        cfg.nonrigid.pcg_iterations = int(pcg)
    st = OF.State()
    xs, vs, pe0, nre0, nrh = [], [], [], [], []
    for fr in frames:
        prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
        x, v, _, st, plogs, slogs = OF.solve_frame(prep, actor, cam, cfg, st)
        xs.append(x)
        vs.append(v)
        pe0.append([o["energy_before"] for o in plogs])
        nre0.append([o["energy_before"] for o in slogs])
        nrh.append([o["halvings"] for o in slogs])
    assert np.array_equal(np.stack(xs), g["poses"])
    d = _digest(np.stack(vs))
    for k in ("sum", "sq", "rows"):
        assert np.array_equal(d[k], g["v_" + k]), k
    for k, row in enumerate(pe0):
        assert np.array_equal(row, g["pose_e0"][k][:len(row)]), k
    assert np.array_equal(np.array(nre0), g["nr_e0"])
    assert np.array_equal(np.array(nrh), g["nr_halv"])
