"""Parity on exactly the workloads bench.py times.

* The bench's seed-0 stream (x5k @1024², directional=False, the bench's
  SequenceConfig), teacher-forced through frames 0-24: every frame starts
  from the oracle's TrackState; per-iteration energies and surface energy
  terms within 1e-4, identical decision traces, vertices within 1e-4 of the
  bbox diagonal.  Four identical streams in one launch (the bench's group
  shape) must agree bit for bit.
* cfg4 (x20k @1024², 4 GN x 8 PCG), whose default surface team is the
  16-CTA cluster, teacher-forced through frames 0-2.
* Every team-size instantiation of both solvers (1, 2, 4, 8, 16 CTAs per
  stream) on small @128 and standard @256.

The oracle is pinned to the real reference on these same workloads by
tests/test_oracle_bench_golden.py (digests of the reference's own runs).
"""

import numpy as np
import pytest

from helpers import bbox_diag, check_pose_strict, check_surface_strict, oracle_state_to_mirror, scene, scene_bench
from test_oracle_golden import check_digest, load

pytestmark = pytest.mark.gpu


def _stage2_jitter(prep, actor, cam, cfg, st, xo, slogs):
    """SURVEY §8c self-jitter screen: the oracle's own Stage II energies when
    its Stage I pose is perturbed at the rounding level (1e-14 relative).
    Returns the largest relative energy change; frames where the oracle moves
    by more than 1e-6 under that jitter are chaotic at the call level (a
    nearest-contour-pixel or prune decision sits on a boundary), and no
    non-bit-identical implementation can be held to 1e-4 there."""
    from oracle import frame as OF
    from oracle.surface import solve_surface
    n = actor.mesh.n_vertices
    disp = st.disp_rest if st.disp_rest is not None else np.zeros((n, 3))
    xj = xo * (1.0 + 1e-14)
    pb, v_init, _, _ = OF.stage2_problem(prep, actor, cam, cfg, st, xj, actor.mesh.rest_vertices + disp)
    _, logs, _ = solve_surface(pb, v_init)
    dev = 0.0
    for a, b in zip(logs, slogs):
        if a["halvings"] != b["halvings"] or a["rejected"] != b["rejected"]:
            return float("inf")
        for k in ("energy_before", "energy_after"):
            dev = max(dev, abs(a[k] - b[k]) / max(abs(b[k]), 1e-300))
    return dev


def _teacher_forced(actor, cam, frames, cfg, streams=1, ctx=None, check_streams_equal=True, screen=False,
                    pose_tol=1e-6):
    """Per-stage teacher forcing: tracker A solves the whole
    frame from the oracle's TrackState and its Stage I is checked against
    the oracle's; tracker B solves Stage II from the same state and the
    oracle's own Stage I pose (lc_tracker_set_pose), so the Stage II check
    does not inherit the ~1e-9 pose rounding that a single non-rigid solve
    amplifies ~1e6.  With `screen`, Stage II of frames that fail
    the oracle's self-jitter screen is reported, not asserted."""
    from oracle import frame as OF
    from paper_1810_02648_b200.device import Tracker
    A = Tracker(actor, cam, cfg, streams, ctx=ctx)
    B = Tracker(actor, cam, cfg, streams, ctx=ctx) if cfg.mode == "full" else None
    st = OF.State()
    diag = bbox_diag(actor)
    worst = 0.0
    skipped = []
    for fr in frames:
        prep = OF.prepare(fr.image, fr.mask, fr.detections, actor, cfg)
        xo, vo, _, st_new, plogs, slogs = OF.solve_frame(prep, actor, cam, cfg, st)
        stable = True
        if screen and B is not None:
            stable = _stage2_jitter(prep, actor, cam, cfg, st, xo, slogs) <= 1e-6
        for s in range(streams):
            A.set_state(s, oracle_state_to_mirror(st))
            A.set_frame(s, fr.image, fr.mask, fr.detections)
            if B is not None:
                B.set_state(s, oracle_state_to_mirror(st))
                B.set_frame(s, fr.image, fr.mask, fr.detections)
                B.set_pose(s, xo)
        A.step()
        if B is not None:
            B.step_stage(2)
        out0 = None
        for s in range(streams):
            x, v, _, rep = A.result(s)
            check_pose_strict(rep.pose, plogs, (fr.index, s))
            if pose_tol is not None:
                assert np.abs(x - xo).max() <= pose_tol, (fr.index, s, "pose", np.abs(x - xo).max())
            else:   # the north-star bound on the frame's output vertices (here the skinned surface)
                assert np.abs(v - vo).max() <= 1e-4 * diag, (fr.index, s, "vertices", np.abs(v - vo).max() / diag)
            if B is not None:
                _, vb, _, repb = B.result(s)
                if stable:
                    worst = max(worst, check_surface_strict(repb.nonrigid, slogs, vb, vo, diag, (fr.index, s)))
                else:
                    assert np.all(np.isfinite(vb))
                    if s == 0:
                        skipped.append((fr.index, float(np.abs(vb - vo).max() / diag)))
            if check_streams_equal:
                if out0 is None:
                    out0 = (x, v)
                else:
                    assert np.array_equal(out0[0], x) and np.array_equal(out0[1], v), (fr.index, s)
        st = st_new
    A.close()
    if B is not None:
        B.close()
    if skipped:
        print(f"Stage II frames failing the oracle's self-jitter screen (reported, not asserted): {skipped}")
    assert len(skipped) <= len(frames) // 4, f"too few screened frames: {skipped}"
    return worst


def test_bench_workload_teacher_forced_25_frames():
    from paper_1810_02648_b200.config import SequenceConfig
    actor, cam, frames = scene_bench("x5k", 1024, 25, seed=0)
    check_digest(load("ref_digest_x5k1024_dir0.npz"), frames)     # the reference's own inputs
    worst = _teacher_forced(actor, cam, frames, SequenceConfig(directional=False), streams=4, screen=True)
    print(f"x5k@1024 frames 0-24: worst vertex err / diag {worst:.2e}")


def test_reference_default_directional_teacher_forced():
    """The reference's default SequenceConfig() (directional silhouette rows,
    the configuration round 1 benchmarked) on the bench's seed-1 stream,
    frames 0-7, teacher-forced per stage: the directional side-sign path of
    both solvers and the snapping walk at x5k@1024^2."""
    from paper_1810_02648_b200.config import SequenceConfig
    actor, cam, frames = scene_bench("x5k", 1024, 8, seed=1)
    worst = _teacher_forced(actor, cam, frames, SequenceConfig(), streams=2, screen=True)
    print(f"x5k@1024 directional frames 0-7: worst vertex err / diag {worst:.2e}")


LONG = pytest.mark.skipif(not __import__("os").environ.get("LIVECAP_LONG_TESTS"),
                          reason="long sequence (minutes of CPU oracle); LIVECAP_LONG_TESTS=1")


@LONG
def test_cfg3_300_frames_teacher_forced():
    """full two-stage tracking over a 300-frame synthetic
    x5k@1024^2 sequence (the reference's default config), teacher-forced per
    stage at every frame (log: profiles/r02/long_sequences.txt)."""
    from paper_1810_02648_b200.config import SequenceConfig
    actor, cam, frames = scene_bench("x5k", 1024, 300, seed=0)
    worst = _teacher_forced(actor, cam, frames, SequenceConfig(), streams=1, screen=True)
    print(f"cfg3 x5k@1024 300 frames: worst vertex err / diag {worst:.2e}")


@LONG
def test_cfg2_pose_only_100_frames_teacher_forced():
    """the pose stage alone over a 100-frame sequence."""
    from paper_1810_02648_b200.config import SequenceConfig
    actor, cam, frames = scene_bench("x5k", 1024, 100, seed=0)
    # (without the surface the pose problem is weakly conditioned on some
    # frames: parameters agree to ~2e-6, so the check is the north-star bound
    # on the output vertices, with identical decisions and energies <= 1e-4)
    _teacher_forced(actor, cam, frames, SequenceConfig(mode="pose_only"), streams=1, pose_tol=None)
    print("cfg2 x5k@1024 100 frames pose-only: decisions identical, energies within 1e-4, vertices within 1e-4 diag")


def test_cfg4_x20k_teacher_forced():
    from paper_1810_02648_b200.config import SequenceConfig
    actor, cam, frames = scene_bench("x20k", 1024, 3, seed=0)
    check_digest(load("ref_digest_x20k1024_cfg4.npz"), frames)
    cfg = SequenceConfig(directional=False)
    cfg.nonrigid.gn_iterations, cfg.nonrigid.pcg_iterations = 4, 8
    worst = _teacher_forced(actor, cam, frames, cfg, streams=2, screen=True)
    print(f"x20k@1024 cfg4 frames 0-2: worst vertex err / diag {worst:.2e}")


@pytest.mark.parametrize("cs", [1, 2, 4, 8, 16])
@pytest.mark.parametrize("preset,res", [("small", 128), ("standard", 256)])
def test_every_team_size(cs, preset, res):
    from paper_1810_02648_b200 import _lib
    from paper_1810_02648_b200.config import SequenceConfig
    ctx = _lib.Context(0)
    ctx.set_team_sizes(pose=cs, surface=cs)
    actor, cam, frames = scene(preset, res, 3)
    _teacher_forced(actor, cam, frames, SequenceConfig(directional=False), streams=2, ctx=ctx)


def test_team_sizes_agree():
    """Teams of different sizes reduce in different orders (fp64 rounding
    only): a free-running run agrees within the parity bar (1e-4 of the bbox
    diagonal; the recursion amplifies rounding ~250x per frame)."""
    from paper_1810_02648_b200 import _lib
    from paper_1810_02648_b200.config import SequenceConfig
    from paper_1810_02648_b200.device import Tracker
    actor, cam, frames = scene("standard", 256, 3)
    res = {}
    for cs in (1, 4, 16):
        ctx = _lib.Context(0)
        ctx.set_team_sizes(pose=cs, surface=cs)
        tr = Tracker(actor, cam, SequenceConfig(directional=False), 1, ctx=ctx)
        out = []
        for fr in frames:
            tr.set_frame(0, fr.image, fr.mask, fr.detections)
            tr.step()
            out.append(tr.result(0, with_report=False)[1])
        res[cs] = np.stack(out)
        tr.close()
    diag = bbox_diag(actor)
    for cs in (4, 16):
        assert np.abs(res[cs][0] - res[1][0]).max() <= 1e-9 * diag     # frame 0: rounding only
        assert np.abs(res[cs] - res[1]).max() <= 1e-4 * diag


def test_team_size_validation():
    from paper_1810_02648_b200 import _lib
    ctx = _lib.Context(0)
    with pytest.raises(ValueError):
        ctx.set_team_sizes(pose=3)
